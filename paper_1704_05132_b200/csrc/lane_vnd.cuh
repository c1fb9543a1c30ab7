// lane_vnd.cuh -- lane-per-product resident VND for short horizons (T <= 63)
// in throughput-bound launches (BASELINE config 3: K = 100,000, T = 52).
// Included by remlot_b200.cu after k_vnd.
//
// k_vnd (warp per product) scores one pass's ~40 moves with the 32 lanes of
// a warp, so every pass ends with the warp waiting for its longest delta
// walk: at C3 only ~46% of the walk lane slots do work, and the per-pass
// base scan, move enumeration, ballots and argmin are paid by the whole
// warp (ncu r02: 31 warp instructions per evaluation).  Here every lane owns
// a whole product and runs the reference's loop (vnd.py:277-288 for one
// product) sequentially: moves in list_moves order (_kernels.py:188-258),
// each scored by the same closed-form delta walk (vnd_device.cuh), the
// first strict minimum kept with '<' (_kernels.py:315-317) -- no argmin
// reduction, no pass barrier.  The lanes of a warp are at different moves,
// passes and products; one loop iteration advances every busy lane by one
// segment of its walk (a base-plan walk that rewrites xc, or a move walk),
// and idle lanes pick their next move (or pass end / product) in a
// divergent control step that runs when enough lanes wait for it.
//
// Shared memory per lane: dr[t] = {cd[t], cr[t+1]} and xc[t] = {cpre[t],
// xin[t]} (t <= T), interleaved by lane (element t of lane l at t*32 + l),
// so every warp-wide access is bank-conflict free whatever t each lane
// reads.  Rows are two uint64 masks per lane (MaskReg) in registers.

namespace rl {

// One lane's rows in a warp's shared-memory block, element t at t*32 + lane.
// Packed (the host proved every product's sum D and sum R < 2^15): dr[t] is
// one 32-bit word cd | cr << 16 and xc is split into cpre (C) and a 16-bit
// xin, 10 bytes per period at int32 costs instead of 16 -- the lane kernel's
// occupancy is bounded by shared memory (T = 52: 13 instead of 8 warps/SM).
template <typename V, typename C, bool Packed>
struct LaneRows;

template <typename V, typename C>
struct LaneRows<V, C, false> {
    DR<V> *dr;
    XC<V, C> *xc;
    __host__ __device__ static size_t bytes(int T)
    {
        return align16((size_t)(T + 1) * 32 * sizeof(DR<V>)) +
               align16((size_t)(T + 1) * 32 * sizeof(XC<V, C>));
    }
    __device__ LaneRows(unsigned char *base, int T, int lane)
    {
        dr = (DR<V> *)base + lane;
        xc = (XC<V, C> *)(base + align16((size_t)(T + 1) * 32 * sizeof(DR<V>))) + lane;
    }
    __device__ DR<V> d(int t) const { return dr[t * 32]; }
    __device__ void set_d(int t, V cd, V cr) const { dr[t * 32] = DR<V>{cd, cr}; }
    __device__ XC<V, C> x(int t) const { return xc[t * 32]; }
    __device__ void set_x(int t, C c, V xv) const { xc[t * 32] = XC<V, C>{c, xv}; }
};

template <typename V, typename C>
struct LaneRows<V, C, true> {
    uint32_t *dr;
    C *cp;
    uint16_t *xi;
    __host__ __device__ static size_t bytes(int T)
    {
        return align16((size_t)(T + 1) * 32 * 4) + align16((size_t)(T + 1) * 32 * sizeof(C)) +
               align16((size_t)(T + 1) * 32 * 2);
    }
    __device__ LaneRows(unsigned char *base, int T, int lane)
    {
        dr = (uint32_t *)base + lane;
        base += align16((size_t)(T + 1) * 32 * 4);
        cp = (C *)base + lane;
        base += align16((size_t)(T + 1) * 32 * sizeof(C));
        xi = (uint16_t *)base + lane;
    }
    __device__ DR<V> d(int t) const
    {
        const uint32_t w = dr[t * 32];
        return DR<V>{V(w & 0xffffu), V(w >> 16)};
    }
    __device__ void set_d(int t, V cd, V cr) const
    {
        RL_ASSERT(cd >= 0 && cd < 32768 && cr >= 0 && cr < 32768);   // the 15-bit proof
        dr[t * 32] = (uint32_t)cd | (uint32_t)cr << 16;
    }
    __device__ XC<V, C> x(int t) const
    {
        XC<V, C> e;
        e.c = cp[t * 32];
        e.x = V(xi[t * 32]);
        return e;
    }
    __device__ void set_x(int t, C c, V xv) const
    {
        cp[t * 32] = c;
        xi[t * 32] = (uint16_t)xv;
    }
};

template <typename V, typename C, bool Packed>
__host__ __device__ inline size_t lane_slot_bytes(int T)
{
    return LaneRows<V, C, Packed>::bytes(T);
}

#ifndef RL_LANE_REFILL_MIN
#define RL_LANE_REFILL_MIN 8
#endif

#ifdef RL_WALK_STATS
// Diagnostic build (tools/lane_stats.py): [0] warp iterations, [1] walking
// lanes summed over iterations, [2] idle (waiting) lanes, [3] done lanes,
// [4] control steps, [5] lanes in control steps, [6] products, [7] cycles in
// load_product, [8] cycles in finish_product, [9] warp lifetimes in cycles.
__device__ unsigned long long g_lane_stats[16];
#endif

enum : int { LN_IDLE = 0, LN_WALK = 1, LN_DONE = 2 };
enum : int { LP_NEWPROD = 0, LP_MOVE = 1, LP_BASE_END = 2 };

template <typename V, typename C, bool Packed>
__global__ void __launch_bounds__(32) k_vnd_lane(InstView<V> in, const uint8_t *sm_in,
                                                 const uint8_t *sr_in, uint8_t *sm_out,
                                                 uint8_t *sr_out, int k_max, VndOut o,
                                                 int refill_min)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int T = in.T;
    const LaneRows<V, C, Packed> L(smem, T, lane);
    const uint64_t sent = 1ull << T, all = sent - 1;

    // product
    int64_t k = 0;
    ProductCosts<C> pc{};
    C K0 = 0, S = 0, S0 = 0;
    uint64_t M = 0, R = 0;
    int sweep = 0, nbh = 1, moves = 0;
    int64_t evals = 0;
    bool improved = false, first_base = false, feas = true;
    // pass: the moves still to score are the set bits of cL (N1/N2/N4
    // periods, N3 left shifts of the current row) and cR (N3 right shifts);
    // cL2/cR2 the R row's N3 shifts, scored after the M row's (list_moves
    // order, _kernels.py:188-258).  fm/fr: the move flips M/R bits.
    uint64_t cL = 0, cR = 0, cL2 = 0, cR2 = 0;
    int row = 0;
    bool is3 = false, fm = false, fr = false;
    C best = 0;
    int bid = -1;   // best move of the pass: t | dir << 6 | row << 7
    // walk
    int u = 0, b = 0, mid = 0;
    V X = 0, cdu = 0, cru = 0;
    C acc = 0;
    uint64_t pM = 0, pR = 0, pSR = 0;
    bool basewalk = false;

    int state = LN_IDLE, post = LP_NEWPROD;
#ifdef RL_WALK_STATS
    unsigned long long ls[10] = {};
    const long long t_start = clock64();
#endif

    // the candidate rows of move (t, dir) of the pass (row = its N3 row)
    auto move_rows = [&](int t, int dir, int mrow, uint64_t &xm, uint64_t &xr) {
        const uint64_t bt = 1ull << t;
        const uint64_t span = bt | (is3 ? (dir ? bt << 1 : bt >> 1) : 0);
        const bool m_ = is3 ? mrow == 0 : fm, r_ = is3 ? mrow == 1 : fr;
        xm = m_ ? span : 0;
        xr = r_ ? span : 0;
        return span;
    };
    // begin a walk of the base plan from its first setup (rewrites xc)
    auto start_base = [&]() {
        pM = M;
        pR = R;
        pSR = __brevll(M | R | sent);
        b = T;   // never "past the move": the walk runs to T
        basewalk = true;
        u = __clzll((long long)pSR);   // first setup >= 0
        acc = 0;
        X = 0;
        const DR<V> e = L.d(u);
        cdu = e.d;
        cru = e.r;
        post = LP_BASE_END;
        if (e.d != 0) {   // demand before the first setup (_kernels.py:58-60)
            feas = false;
            state = LN_IDLE;
        } else if (u >= T) {   // no setup and no demand: cost 0
            S = 0;
            L.set_x(T, S, V(0));
            state = LN_IDLE;
        } else {
            state = LN_WALK;
        }
    };
    // begin pass nbh at the current plan (cursor, move count, best = S)
    auto begin_pass = [&]() {
        row = 0;
        is3 = nbh == 3;
        fm = nbh == 1 || nbh == 4;
        fr = nbh == 2 || nbh == 4;
        cR = cL2 = cR2 = 0;
        if (nbh <= 2) {
            cL = all;
        } else if (nbh == 4) {
            cL = (M ^ R) & all;   // swaps where the rows differ
        } else {
            const RegMoveMasks q = reg_move_masks(MaskReg{M, R, T});
            cL = q.lm;
            cR = q.rm;
            cL2 = q.lr;
            cR2 = q.rr;
        }
        evals += __popcll(cL) + __popcll(cR) + __popcll(cL2) + __popcll(cR2);
        best = S;
        bid = -1;
    };
    // the pass after this one; false when the product reached its fixpoint
    auto advance_pass = [&]() -> bool {
        if (++nbh > k_max) {
            ++sweep;
            if (!improved)
                return false;
            improved = false;
            nbh = 1;
        }
        begin_pass();
        return true;
    };
    auto finish_product = [&]() {
        int ntot = 0;
        if (feas)
            for (int q = 1; q <= k_max; ++q)
                ntot += move_count(MaskReg{M, R, T}, q, T, lane);
        uint8_t *om = sm_out + k * T, *orr = sr_out + k * T;
        for (int t = 0; t < T; ++t) {
            om[t] = (uint8_t)((M >> t) & 1);
            orr[t] = (uint8_t)((R >> t) & 1);
        }
        o.start_cost[k] = feas ? (int64_t)(K0 + S0) : RL_INFEASIBLE;
        o.final_cost[k] = feas ? (int64_t)(K0 + S) : RL_INFEASIBLE;
        o.evals[k] = evals;
        o.ntot[k] = ntot;
        o.sweeps[k] = feas ? sweep : 1;
        o.moves[k] = moves;
    };
    auto load_product = [&]() {
        pc = load_costs<C>(in.cost6, in.K, k, T, in.one);
        const V *d = in.dem + k * T, *r = in.ret + k * T;
        const uint8_t *a = sm_in + k * T, *bb = sr_in + k * T;
        V cd = 0, cr = 0;
        C scd = 0, scr = 0;
        M = R = 0;
        for (int t = 0; t < T; ++t) {
            cr += r[t];
            L.set_d(t, cd, cr);
            cd += d[t];
            scd += C(cd);
            scr += C(cr);
            M |= (uint64_t)(a[t] != 0) << t;
            R |= (uint64_t)(bb[t] != 0) << t;
        }
        L.set_d(T, cd, V(0));
        K0 = pc.hr * scr - pc.hm * scd;
        sweep = 0;
        nbh = 1;
        moves = 0;
        evals = 0;
        improved = false;
        feas = true;
        first_base = true;
        start_base();
    };

    for (;;) {
        const unsigned idle = __ballot_sync(FULL, state == LN_IDLE);
        const unsigned walking = __ballot_sync(FULL, state == LN_WALK);
        if (!(idle | walking))
            break;
#ifdef RL_WALK_STATS
        ++ls[0];
        ls[1] += __popc(walking);
        ls[2] += __popc(idle);
        ls[3] += 32 - __popc(idle | walking);
        if (idle && (!walking || __popc(idle) >= refill_min)) {
            ++ls[4];
            ls[5] += __popc(idle);
        }
#endif
        // control step for the idle lanes, in batches (the branches cost the
        // warp's issue slots however few lanes take them)
        if (idle && (!walking || __popc(idle) >= refill_min)) {
            // phase 1 (rare, divergent): product loads, base-walk ends, pass
            // ends, N3 row switches -- until the lane walks, is done, or has
            // a move to score
            while (state == LN_IDLE && (post != LP_MOVE || !(cL | cR))) {
                if (post == LP_NEWPROD) {
                    k = o.k_lo + atomicAdd(o.queue, 1);
                    if (k >= o.k_hi) {
                        state = LN_DONE;
                        break;
                    }
#ifdef RL_WALK_STATS
                    const long long c0_ = clock64();
                    load_product();
                    ls[7] += clock64() - c0_;
                    ++ls[6];
#else
                    load_product();
#endif
                } else if (post == LP_BASE_END) {
                    post = LP_MOVE;
                    if (!feas) {   // skipped product (_kernels.py:289-290)
                        finish_product();
                        post = LP_NEWPROD;
                    } else if (first_base) {
                        first_base = false;
                        S0 = S;
                        begin_pass();
                    } else if (!advance_pass()) {
                        finish_product();
                        post = LP_NEWPROD;
                    }
                } else if (is3 && row == 0 && (cL2 | cR2)) {   // the R row's shifts
                    row = 1;
                    cL = cL2;
                    cR = cR2;
                } else if (bid >= 0) {   // pass end: apply the first strict minimum
                    uint64_t xm, xr;
                    move_rows(bid & 63, (bid >> 6) & 1, bid >> 7, xm, xr);
                    M ^= xm;
                    R ^= xr;
                    if (sweep < o.cap_sweeps)
                        atomicAdd(&o.trace_dec[(int64_t)sweep * k_max + nbh - 1],
                                  (unsigned long long)(int64_t)(S - best));
                    else
                        atomicExch(o.overflow, 1);
                    ++moves;
                    improved = true;
                    bid = -1;
                    start_base();   // S = best again once the walk ends
                } else if (!advance_pass()) {
                    finish_product();
                    post = LP_NEWPROD;
                }
            }
            __syncwarp();
            // phase 2 (every idle lane with a move): set up its next move's
            // delta walk, branch-free
            if (state == LN_IDLE) {
                const int t = __ffsll((long long)(cL | cR)) - 1;
                const uint64_t bt = 1ull << t;
                const int dir = (cL & bt) ? 0 : 1;   // left before right (_kernels.py:221-233)
                cL &= dir ? ~0ull : ~bt;
                cR &= dir ? ~bt : ~0ull;
                mid = t | dir << 6 | row << 7;
                uint64_t xm, xr;
                const uint64_t span = move_rows(t, dir, row, xm, xr);
                pM = M ^ xm;
                pR = R ^ xr;
                pSR = __brevll(pM | pR | sent);
                const int a = __ffsll((long long)span) - 1;
                b = 63 - __clzll((long long)span);
                basewalk = false;
                // the prefix before the base plan's last setup ahead of a is
                // the base's (xc); else the candidate's first setup
                const uint64_t below = (M | R) & ((1ull << a) - 1);
                const int p = 63 - __clzll((long long)below);   // -1 if none
                const XC<V, C> e = L.x((p < 0 ? 0 : p));
                u = p >= 0 ? p : __clzll((long long)pSR);
                acc = p >= 0 ? e.c : C(0);
                X = p >= 0 ? e.x : V(0);
                const DR<V> f = L.d(u);
                cdu = f.d;
                cru = f.r;
                // no setup ahead: demand before the first setup is infeasible
                // (not scored); no setup at all and no demand costs 0
                const bool dead = p < 0 && f.d != 0;
                const bool zero = !dead && u >= T;
                if (zero && acc < best) {
                    best = acc;
                    bid = mid;
                }
                state = dead || zero ? LN_IDLE : LN_WALK;
            }
        }
        __syncwarp();
        if (state == LN_WALK) {
            // one segment [u, v) of the walk (vnd_device.cuh walk_moves)
            RL_ASSERT(u >= 0 && u < T);
            const int v = (u + 1) + __clzll((long long)(pSR << (u + 1)));
            RL_ASSERT(v > u && v <= T);
            const bool mu = (pM >> u) & 1, ru = (pR >> u) & 1;
            const DR<V> ev = L.d(v);
            C c;
            V xr;
            const bool ok = seg_cost<V, C>(cdu, cru, ev.d, u, mu, ru, X, pc, c, xr);
            if (basewalk)
                L.set_x(u, acc, X);
            const XC<V, C> bv = L.x(v);   // v <= T; xc[T].c = S
            acc += c;
            X += xr;
            const bool past = v < T && v > b;
            const bool sync = past && X == bv.x;
            const C total = acc + (S - bv.c);
            const bool fin = v >= T || sync;
            if (!basewalk && ok && fin && total < best) {
                best = total;
                bid = mid;
            }
            u = v;
            cdu = ev.d;
            cru = ev.r;
            if (basewalk) {
                feas = feas && ok;
                if (!ok || v >= T) {
                    if (ok) {
                        S = acc;
                        L.set_x(T, S, V(0));
                    }
                    state = LN_IDLE;
                }
            } else if (!ok || fin) {
                state = LN_IDLE;
            }
        }
    }
#ifdef RL_WALK_STATS
    ls[9] = clock64() - t_start;
    if (lane == 0)
        for (int i = 0; i < 10; ++i)
            atomicAdd(&g_lane_stats[i], ls[i]);
#endif
}

}  // namespace rl
