// gvns_impl.cuh -- device shaking, W-worker rounds and the best-of join
// (reference gvns.py:88-221).  Included by remlot_b200.cu after the handle.
//
// A round (worker_round, gvns.py:147-174) runs W workers; worker w draws from
// Philox(SeedSequence((seed, round, w))) exactly like numpy (rng_device.cuh),
// flips k_eff = min(k, 2KT) distinct flat positions (gvns.py:93-122), and
// descends with VND.  Because products never interact and the VND of a plan
// is the per-product VND of its rows, a worker's
// result is F (the per-product VND image of the incumbent, computed once)
// with only its touched products re-descended.  So a round is:
//   k_shake           warp per worker: draws, touched rows, feasibility; lane 0
//                     runs the fallback when all 50 draws failed (gvns.py:124-137)
//   k_gvns_vnd        warp per (worker, touched product) [+ fallback plans]
//   k_gvns_join       block: min (cost, worker) join, accept, next strength
// with no host synchronisation; the incumbent and F stay resident.
//
// Speculative batches (rl_gvns_begin_batch / rl_gvns_run): rounds r0 ..
// r0+B-1 run as one launch of B x W worker slots, each round shaking the
// same incumbent with the strength it would have if no earlier round of the
// batch improved (the round's RNG streams depend only on (seed, round, w)).
// The join walks the rounds in order and stops at the first accepted one;
// the rounds after it are discarded and re-run from the new incumbent by the
// next batch, so the trajectory is exactly the sequential one.  Most rounds
// do not improve, and a batch costs about one round's latency.

struct GvnsArgs {
    int64_t K, KT, pop;
    int64_t w0;                       // global index of local worker 0 (sharded rounds)
    int T, NW, W, k_max, kcap, tcap, tsize, fb_slots;
    int Wr, B;                        // workers per round, rounds per batch (W = B x Wr slots)
    int shake_bytes;                  // per-worker shared scratch of k_shake (0: global)
    uint64_t seed;
    uint8_t *inc, *F, *init, *cand;   // 2KT bytes each: m rows then r rows
    int64_t *Fcost;                   // K
    int64_t *scal;                    // see GV_* below
    int64_t *pos;                     // W x kcap
    uint64_t *table;                  // W x tsize
    int64_t *tailidx;                 // W x pop (only when the tail shuffle is needed)
    int64_t *tp;                      // W x tcap touched products
    int *tn, *fb, *fbslot;            // W
    int *tasks;                       // W x tcap: compact (worker x tcap + j) VND tasks
    uint32_t *tw;                     // W x tcap x 2 x NW
    int64_t *tcost;                   // W x tcap
    PhiloxState *rng;                 // W
    uint8_t *fbplan;                  // fb_slots x 2KT
    int64_t *fbdiff;                  // fb_slots x pop
    int64_t *fbpcost;                 // fb_slots x K
    int *queue;
    int64_t *rbest;                   // B x 3: per batch round best (cost, global worker, slot)
    void *pfx;                        // K x 2(T+1) V: cd[0..T], cr[0..T] (prefix sums, shake test)
};

enum {
    GV_INC_COST = 0,
    GV_FTOT,
    GV_STRENGTH,
    GV_INC_IS_F,
    GV_BEST_COST,
    GV_BEST_W,
    GV_ACCEPTED,
    GV_FB_COUNT,
    GV_ERROR,
    GV_ROUND,     // rounds completed (the next batch starts here)
    GV_NB,        // rounds of the next batch (adaptive, <= B)
    GV_NTASK,     // compact VND tasks appended by k_shake (reset by the join)
    GV_FB_TRUNC,  // B - (first batch round whose fallback found no slot), 0 = none
    GV_LOCAL_NB,  // rounds of the last local batch (mode 2) with valid bests
    GV_MAXR,      // round cap of a device-resident run (max_rounds < 0 in the kernels)
    GV_TBUDGET,   // its wall-clock budget in ns
    GV_T0,        // %globaltimer at its start
    GV_FBCOST0,   // fb_slots entries follow
};

// Rounds of this launch: round_arg >= 0 names the first round (single-round
// calls), else the device counter does; at most GV_NB (the adaptive batch
// size: 1 after an accepted round, doubled up to B after a batch without
// one, so improving phases run round by round and stagnating phases
// speculate) and never past max_rounds.
__device__ inline int gv_batch(const GvnsArgs &g, int64_t round_arg, int64_t max_rounds,
                               int64_t &r0)
{
    r0 = round_arg >= 0 ? round_arg : g.scal[GV_ROUND];
    const int64_t cap = round_arg >= 0 ? g.B : g.scal[GV_NB];
    const int64_t left = (max_rounds < 0 ? g.scal[GV_MAXR] : max_rounds) - r0;
    return left <= 0 ? 0 : left < cap ? (int)left : (int)cap;
}

// Strength of batch round j if rounds 0..j-1 do not improve
// (next_strength, gvns.py:177-181, applied j times).
__device__ inline int64_t gv_strength(const GvnsArgs &g, int j)
{
    int64_t k = g.scal[GV_STRENGTH];
    for (int i = 0; i < j; ++i)
        k = k >= g.k_max ? 1 : k + 1;
    return k;
}

// Feasibility of a shaken product's rows over prefix sums cd[t] = sum_{i<t} D,
// cr[t] = sum_{i<t} R (closed form of DESIGN.md 3: x_R = min(seg, cr[u+1] -
// X) at sR setups) with the whole warp (k_shake): lane l
// owns periods [lL, lL + L); the cumulative remanufacturing X entering each
// lane's periods comes from a warp scan of the (min, +)-affine maps X ->
// min(X + seg, cr[u+1]) of its sR setups (as base_pass), then every lane
// checks its own segments.  A few hundred cycles instead of one dependent
// step per segment on lane 0.
template <typename V>
__device__ inline bool warp_row_feasible(const V *cd, const V *cr, int T, const uint32_t *row,
                                         int NW, int lane)
{
    auto next_setup = [&](int x) {   // first setup >= x, T if none
        if (x >= T)
            return T;
        int w = x >> 5;
        uint32_t bits = (row[w] | row[NW + w]) & (0xffffffffu << (x & 31));
        while (!bits && ++w < NW)
            bits = row[w] | row[NW + w];
        return bits ? min((w << 5) + __ffs(bits) - 1, T) : T;
    };
    const int L = (T + 31) >> 5;
    const int lo = min(lane * L, T), hi = min(lo + L, T);
    const V INF = VInf<V>::value;
    V A = 0, B = INF;
    for (int u = lo; u < hi; ++u) {
        if (!((row[NW + (u >> 5)] >> (u & 31)) & 1u))
            continue;   // only remanufacturing setups move X
        const V seg = cd[next_setup(u + 1)] - cd[u];
        A += seg;
        B = vmin<V>(B + seg, cr[u + 1]);
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const V a2 = __shfl_up_sync(FULL, A, off), b2 = __shfl_up_sync(FULL, B, off);
        if (lane >= off) {
            B = vmin<V>(b2 + A, B);
            A = a2 + A;
        }
    }
    const V pa = __shfl_up_sync(FULL, A, 1), pb = __shfl_up_sync(FULL, B, 1);
    V X = lane == 0 ? V(0) : vmin<V>(pa, pb);
    bool ok = true;
    for (int u = lo; u < hi; ++u) {
        const bool m = (row[u >> 5] >> (u & 31)) & 1u, r = (row[NW + (u >> 5)] >> (u & 31)) & 1u;
        if (!(m | r))
            continue;
        const V seg = cd[next_setup(u + 1)] - cd[u];
        const V xr = r ? vmin<V>(seg, cr[u + 1] - X) : V(0);
        ok &= !(seg - xr > 0 && !m);
        X += xr;
    }
    if (lane == 0)
        ok &= cd[next_setup(0)] <= 0;   // demand before the first setup (_kernels.py:58-60)
    return __all_sync(FULL, ok);
}

// Feasibility of one product's rows under row_cost (_kernels.py:58-82):
// no demand before the first setup, and every segment whose demand exceeds
// the remanufactured quantity has a manufacturing setup.
template <typename V, typename BitM, typename BitR>
__device__ inline bool row_feasible(const V *d, const V *r, int T, BitM bm, BitR br)
{
    int t = 0;
    V rec = 0;
    for (; t < T && !(bm(t) | br(t)); ++t) {
        if (d[t] > 0)
            return false;
        rec += r[t];
    }
    while (t < T) {
        const int u = t;
        int v = u + 1;
        V seg = d[u], ret = r[u];
        while (v < T && !(bm(v) | br(v))) {
            seg += d[v];
            ret += r[v];
            ++v;
        }
        const V avail = rec + r[u];
        const V xr = br(u) ? (seg < avail ? seg : avail) : V(0);
        if (seg - xr > 0 && !bm(u))
            return false;
        rec += ret - xr;
        t = v;
    }
    return true;
}

// gvns.py:124-137: flip the positions where the incumbent differs from the
// lot-for-lot start, in rng.shuffle order, until >= k_eff flips and the whole
// plan is feasible; else return the start.  Run by the worker's whole k_shake
// warp right after its 50 redraws failed (rare), with the worker's RNG state
// after them (g.rng[w]): the warp copies the plan and compacts the differing
// positions (ballot prefix sums keep them ascending, m rows then r rows like
// the reference), lane 0 runs the shuffle and the flip/feasibility walk.
template <typename V>
__device__ void shake_fallback(const InstView<V> &in, const GvnsArgs &g, int w, int lane)
{
    int slot = 0;
    if (lane == 0) {
        slot = (int)atomicAdd((unsigned long long *)&g.scal[GV_FB_COUNT], 1ull);
        if (slot >= g.fb_slots) {
            // slots ran out (speculative rounds of a batch share them): the
            // join truncates the batch before this worker's round, which is
            // re-run later with the slots to itself; fbslot = fb_slots is
            // never read
            g.fbslot[w] = g.fb_slots;
            atomicMax((unsigned long long *)&g.scal[GV_FB_TRUNC],
                      (unsigned long long)(g.B - w / g.Wr));
        } else {
            g.fbslot[w] = slot;
        }
    }
    slot = __shfl_sync(FULL, slot, 0);
    if (slot >= g.fb_slots)
        return;
    const int T = g.T;
    const int64_t KT = g.KT, K = g.K, KT2 = 2 * KT;
    uint8_t *plan = g.fbplan + (int64_t)slot * KT2;
    int64_t *diff = g.fbdiff + (int64_t)slot * g.pop;
    int64_t *bad = g.fbpcost + (int64_t)slot * K;   // infeasibility flags, then costs
    int64_t n = 0;
    for (int64_t base = 0; base < KT2; base += 32) {
        const int64_t p = base + lane;
        uint8_t v = 0;
        bool d = false;
        if (p < KT2) {
            v = g.inc[p];
            plan[p] = v;
            d = v != g.init[p];
        }
        const uint32_t bal = __ballot_sync(FULL, d);
        if (d)
            diff[n + __popc(bal & ((1u << lane) - 1u))] = p;
        n += __popc(bal);
    }
    for (int64_t k = lane; k < K; k += 32)
        bad[k] = 0;   // the incumbent is feasible
    __syncwarp();
    int done = 0;
    if (lane == 0) {
        Philox rng;
        rng.st = g.rng[w];
        rng.shuffle(diff, n);
        const int64_t strength = gv_strength(g, w / g.Wr);
        const int64_t k_eff = strength < g.pop ? strength : g.pop;
        int64_t nbad = 0;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t p = diff[i];
            plan[p] ^= 1;
            const int64_t k = (p % KT) / T;
            const uint8_t *pm = plan + k * T, *pr = plan + KT + k * T;
            const bool f = row_feasible<V>(in.dem + k * T, in.ret + k * T, T,
                                           [&](int q) { return pm[q] != 0; },
                                           [&](int q) { return pr[q] != 0; });
            nbad += (f ? 0 : 1) - bad[k];
            bad[k] = f ? 0 : 1;
            if (i + 1 >= k_eff && nbad == 0) {
                done = 1;
                break;
            }
        }
    }
    done = __shfl_sync(FULL, done, 0);
    if (!done)
        for (int64_t i = lane; i < KT2; i += 32)
            plan[i] = g.init[i];
    __syncwarp();
}

// Per-product prefix sums cd[t] = sum_{i<t} D, cr[t] = sum_{i<t} R (t <= T)
// for the shake's feasibility test, computed once per rl_gvns_begin (one
// warp per product) instead of for every touched product of every redraw.
template <typename V>
__global__ void k_gvns_prefix(InstView<V> in, V *pfx)
{
    const int lane = threadIdx.x & 31, T = in.T;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < in.K;
         k += nw) {
        V *cd = pfx + k * 2 * (T + 1), *cr = cd + T + 1;
        V cdc = 0, crc = 0;
        if (lane == 0) {
            cd[0] = 0;
            cr[0] = 0;
        }
        for (int base = 0; base < T; base += 32) {
            const int t = base + lane;
            V d = t < T ? in.dem[k * T + t] : V(0);
            V r = t < T ? in.ret[k * T + t] : V(0);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const V od = __shfl_up_sync(FULL, d, off), orr = __shfl_up_sync(FULL, r, off);
                if (lane >= off) {
                    d += od;
                    r += orr;
                }
            }
            d += cdc;
            r += crc;
            if (t < T) {
                cd[t + 1] = d;
                cr[t + 1] = r;
            }
            cdc = __shfl_sync(FULL, d, 31);
            crc = __shfl_sync(FULL, r, 31);
        }
    }
}

// One warp per worker: lane 0 runs the (inherently sequential) numpy-exact
// draw and the flips; the other lanes pull the touched products' rows
// (incumbent bits, demand, returns) into L1 with coalesced loads first, so
// lane 0's sequential feasibility walk hits the cache instead of DRAM/L2.
template <typename V>
__global__ void k_shake(InstView<V> in, GvnsArgs g, int64_t round_arg, int64_t max_rounds)
{
    extern __shared__ __align__(16) unsigned char shk[];
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // the per-round counters this kernel and the next ones use (fallback
    // slots, fallback plan costs, task list, VND queue) were reset by the
    // previous round's join (or rl_gvns_begin)
    if (w >= g.W)
        return;
    int64_t r0;
    const int nb = gv_batch(g, round_arg, max_rounds, r0);
    const int jr = w / g.Wr;   // batch round of this slot
    if (jr >= nb) {            // past the batch: no tasks, no fallback
        if (lane == 0) {
            g.tn[w] = 0;
            g.fb[w] = 0;
        }
        return;
    }
    Philox rng;
    if (lane == 0)
        rng.seed(g.seed, (uint64_t)(r0 + jr), (uint64_t)(g.w0 + w % g.Wr));
    const int64_t strength = gv_strength(g, jr);
    const int64_t k_eff = strength < g.pop ? strength : g.pop;   // gvns.py:113
    const int T = g.T, NW = g.NW;
    // the draw's scratch (Floyd table, positions, touched rows) lives in
    // shared memory when it fits: the sequential draw and feasibility walk
    // then wait on shared-memory instead of L2 latencies; the accepted
    // touched rows are copied out for k_gvns_vnd
    int64_t *P = g.pos + (int64_t)w * g.kcap;
    int64_t *tp = g.tp + (int64_t)w * g.tcap;
    uint32_t *tw = g.tw + (int64_t)w * g.tcap * 2 * NW;
    uint64_t *table = g.table + (int64_t)w * g.tsize;
    if (g.shake_bytes) {
        unsigned char *b = shk + (size_t)(threadIdx.x >> 5) * g.shake_bytes;
        table = (uint64_t *)b;
        b += align16((size_t)g.tsize * 8);
        P = (int64_t *)b;
        b += align16((size_t)g.kcap * 8);
        tp = (int64_t *)b;
        b += align16((size_t)g.tcap * 8);
        tw = (uint32_t *)b;
    }
    for (int attempt = 0; attempt < 50; ++attempt) {   // _SHAKE_REDRAWS (gvns.py:29, :114)
        int n = 0;
        if (lane == 0) {
            if (choice_uses_tail_shuffle(g.pop, k_eff))
                choice_tail(rng, g.pop, k_eff, P, g.tailidx + (int64_t)w * g.pop);
            else
                choice_floyd(rng, g.pop, k_eff, P, table);
            for (int64_t i = 0; i < k_eff; ++i) {   // distinct touched products
                RL_ASSERT(P[i] >= 0 && P[i] < g.pop);
                const int64_t k = (P[i] % g.KT) / T;
                int j = 0;
                while (j < n && tp[j] != k)
                    ++j;
                if (j == n)
                    tp[n++] = k;
            }
        }
        n = __shfl_sync(FULL, n, 0);
        __syncwarp();
        // rows of the touched products, product by product: incumbent bits
        // by ballot, the flips that fall on the product (_flip_flat,
        // gvns.py:93-98), prefix sums, the warp feasibility test; an
        // infeasible product ends the attempt (most redraws fail early)
        bool ok = true;
        for (int j = 0; j < n && ok; ++j) {
            const int64_t k = tp[j];
            const uint8_t *im = g.inc + k * T, *ir = g.inc + g.KT + k * T;
            uint32_t *row = tw + (int64_t)j * 2 * NW;
            for (int base = 0; base < T; base += 32) {
                const int t = base + lane;
                const uint32_t wm = __ballot_sync(FULL, t < T && im[t]);
                const uint32_t wr = __ballot_sync(FULL, t < T && ir[t]);
                if (lane == 0) {
                    row[base >> 5] = wm;
                    row[NW + (base >> 5)] = wr;
                }
            }
            if (lane == 0)
                for (int64_t i = 0; i < k_eff; ++i) {
                    const int64_t p = P[i];
                    const int64_t rem = p % g.KT;
                    if (rem / T != k)
                        continue;
                    const int t = (int)(rem % T);
                    row[(p < g.KT ? 0 : NW) + (t >> 5)] ^= 1u << (t & 31);
                }
            // the warp test over the product's prefix sums (k_gvns_prefix)
            const V *cd = (const V *)g.pfx + k * 2 * (T + 1);
            __syncwarp();
            ok = warp_row_feasible<V>(cd, cd + T + 1, T, row, NW, lane);
        }
        ok = __shfl_sync(FULL, (int)ok, 0);
        if (ok) {
            if (g.shake_bytes) {
                __syncwarp();   // lane 0 wrote the scratch
                for (int j = lane; j < n; j += 32)
                    g.tp[(int64_t)w * g.tcap + j] = tp[j];
                uint32_t *gw = g.tw + (int64_t)w * g.tcap * 2 * NW;
                for (int i = lane; i < n * 2 * NW; i += 32)
                    gw[i] = tw[i];
            }
            if (lane == 0) {
                g.tn[w] = n;
                g.fb[w] = 0;
                // compact task list: k_gvns_vnd's warps take only real tasks
                const int64_t b =
                    (int64_t)atomicAdd((unsigned long long *)&g.scal[GV_NTASK], (unsigned long long)n);
                for (int j = 0; j < n; ++j)
                    g.tasks[b + j] = w * g.tcap + j;
            }
            return;
        }
    }
    if (lane == 0) {
        g.tn[w] = 0;
        g.fb[w] = 1;
        g.rng[w] = rng.st;
    }
    __syncwarp();
    shake_fallback<V>(in, g, w, lane);
}


// VND of every (worker, touched product) task and of every product of the
// fallback plans; warps pull tasks from a queue.
template <typename V, typename C, typename Mask, bool Skip = true>
__global__ void __launch_bounds__(128) k_gvns_vnd(InstView<V> in, GvnsArgs g, int k_vnd_max)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = in.T, NW = g.NW;
    const int64_t n_norm = g.scal[GV_NTASK];
    int64_t nfb = g.scal[GV_FB_COUNT];
    nfb = nfb < g.fb_slots ? nfb : g.fb_slots;
    const int64_t n_tasks = n_norm + nfb * g.K;
    // warps beyond the round's task count leave before touching the queue
    // (the grid is sized for the worst case: every slot's tasks + fallbacks)
    if ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp >= n_tasks)
        return;
    Slot<V, C> s = carve<V, C>(smem + warp * slot_bytes<V, C>(T), T);
    if (lane == 0)
        mbar_init(s.bar);
    __syncwarp();
    uint32_t phase = 0;
    for (;;) {
        int64_t task = 0;
        if (lane == 0)
            task = atomicAdd(g.queue, 1);
        task = __shfl_sync(FULL, task, 0);
        if (task >= n_tasks)
            break;
        int64_t k;
        uint32_t *row = nullptr;
        uint8_t *plan = nullptr;
        int w = -1, j = -1, slot = -1;
        if (task < n_norm) {
            const int id = g.tasks[task];
            w = id / g.tcap;
            j = id % g.tcap;
            if (g.fb[w] || j >= g.tn[w])
                continue;
            k = g.tp[(int64_t)w * g.tcap + j];
            row = g.tw + ((int64_t)w * g.tcap + j) * 2 * NW;
        } else {
            slot = (int)((task - n_norm) / g.K);
            k = (task - n_norm) % g.K;
            plan = g.fbplan + (int64_t)slot * 2 * g.KT;
        }
        stage_begin(s, in, k, lane);
        const ProductCosts<C> pc = load_costs<C>(in.cost6, in.K, k, in.T, in.one);
        Mask mk;
        if (row) {
            // words -> plan bytes layout for load_rows: go through the slot's mv buffer
            uint8_t *tmp = (uint8_t *)s.mv;   // 2T+2 uint16 = 4T+4 bytes >= 2T
            for (int t = lane; t < T; t += 32) {
                tmp[t] = (row[t >> 5] >> (t & 31)) & 1u;
                tmp[T + t] = (row[NW + (t >> 5)] >> (t & 31)) & 1u;
            }
            __syncwarp();
            mk = load_rows(s, Mask{}, tmp, tmp + T, 0, T, lane);
        } else {
            mk = load_rows(s, Mask{}, plan, plan + g.KT, k, T, lane);
        }
        stage_end(s, in, k, lane, phase);
        const C K0 = build_prefix(s, T, pc, lane);
        C S0, S;
        VndStats st;
        vnd_product<V, C, Mask, Skip>(s, mk, T, pc, k_vnd_max, lane, S0, S, st, nullptr, 0,
                                      nullptr);
        const int64_t cost = (int64_t)(K0 + S);
        if (row) {
            __syncwarp();
            for (int q = lane; q < 2 * NW; q += 32)
                row[q] = 0;
            __syncwarp();
            for (int t = lane; t < T; t += 32) {
                if (mk.m(t))
                    atomicOr(&row[t >> 5], 1u << (t & 31));
                if (mk.r(t))
                    atomicOr(&row[NW + (t >> 5)], 1u << (t & 31));
            }
            if (lane == 0)
                g.tcost[(int64_t)w * g.tcap + j] = cost;
        } else {
            store_rows(mk, plan, plan + g.KT, k, T, lane);
            if (lane == 0) {
                g.fbpcost[(int64_t)slot * g.K + k] = cost;
                atomicAdd((unsigned long long *)&g.scal[GV_FBCOST0 + slot], (unsigned long long)cost);
            }
        }
        __syncwarp();
    }
}

// Candidate cost of worker slot w: F's total with its touched products'
// re-descended costs, or its fallback plan's cost.
__device__ inline long long gv_worker_cost(const GvnsArgs &g, int w)
{
    if (g.fb[w]) {
        const int slot = g.fbslot[w];
        return slot < g.fb_slots ? g.scal[GV_FBCOST0 + slot] : 0x7fffffffffffffffll;
    }
    long long c = g.scal[GV_FTOT];
    for (int j = 0; j < g.tn[w]; ++j) {
        c -= g.Fcost[g.tp[(int64_t)w * g.tcap + j]];
        c += g.tcost[(int64_t)w * g.tcap + j];
    }
    return c;
}

// Join (gvns.py:170-174: min cost, lowest worker on ties) and, in accept
// mode, the GVNS step (gvns.py:207-215): accept strict improvements, reset or
// advance the strength (next_strength, gvns.py:177-181).  mode 0 writes the
// winning candidate plan to g.cand (worker_round's return value).  A batch
// (B > 1, accept mode) joins each round with one warp and applies the steps
// in round order up to the first acceptance (GV_ROUND advances by the rounds
// used).
__global__ void k_gvns_join(GvnsArgs g, int mode, int64_t round_arg, int64_t max_rounds)
{
    __shared__ long long s_cost[32];
    __shared__ int s_w[32];
    __shared__ int s_accept, s_win, s_nb;
    int64_t r0;
    const int nb_all = gv_batch(g, round_arg, max_rounds, r0);
    if (threadIdx.x == 0) {
        // rounds from the first one with a fallback that found no slot on
        // are discarded (re-run by the next batch, like rounds after an
        // acceptance)
        const int64_t tr = g.scal[GV_FB_TRUNC];
        int nb = nb_all;
        if (tr > 0 && g.B - tr < nb)
            nb = (int)(g.B - tr);
        if (nb == 0 && nb_all > 0) {
            if (nb_all == 1)   // one round's fallbacks alone exceed the slots
                g.scal[GV_ERROR] = 1;
            else if (round_arg < 0)
                g.scal[GV_NB] = 1;   // re-run the first round alone
        }
        s_nb = nb;
        // k_gvns_vnd has consumed the round's tasks: per-round counters for
        // the next round (fallback plan costs are reset after the join reads
        // them)
        g.scal[GV_NTASK] = 0;
        g.scal[GV_FB_COUNT] = 0;
        g.scal[GV_FB_TRUNC] = 0;
        *g.queue = 0;
    }
    __syncthreads();
    const int nb = s_nb;
    if (nb == 0) {
        for (int i = threadIdx.x; i < g.fb_slots; i += blockDim.x)
            g.scal[GV_FBCOST0 + i] = 0;
        if (mode == 2 && threadIdx.x == 0)
            g.scal[GV_LOCAL_NB] = 0;
        return;
    }
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nwarps = (int)(blockDim.x >> 5);
    if (g.B == 1) {
        long long best = 0x7fffffffffffffffll;
        int bw = 0x7fffffff;
        for (int w = tid; w < g.W; w += blockDim.x) {
            const long long c = gv_worker_cost(g, w);
            if (c < best || (c == best && w < bw)) {
                best = c;
                bw = w;
            }
        }
        for (int off = 16; off; off >>= 1) {
            const long long oc = __shfl_xor_sync(FULL, best, off);
            const int ow = __shfl_xor_sync(FULL, bw, off);
            if (oc < best || (oc == best && ow < bw)) {
                best = oc;
                bw = ow;
            }
        }
        if (lane == 0) {
            s_cost[wid] = best;
            s_w[wid] = bw;
        }
        __syncthreads();
        if (tid == 0)
            for (int i = 1; i < nwarps; ++i)
                if (s_cost[i] < s_cost[0] || (s_cost[i] == s_cost[0] && s_w[i] < s_w[0])) {
                    s_cost[0] = s_cost[i];
                    s_w[0] = s_w[i];
                }
    } else {
        // warp per batch round (B <= 32): slots j*Wr .. j*Wr + Wr - 1
        for (int jr = wid; jr < nb; jr += nwarps) {
            long long best = 0x7fffffffffffffffll;
            int bw = 0x7fffffff;
            for (int q = lane; q < g.Wr; q += 32) {
                const int w = jr * g.Wr + q;
                const long long c = gv_worker_cost(g, w);
                if (c < best || (c == best && w < bw)) {
                    best = c;
                    bw = w;
                }
            }
            for (int off = 16; off; off >>= 1) {
                const long long oc = __shfl_xor_sync(FULL, best, off);
                const int ow = __shfl_xor_sync(FULL, bw, off);
                if (oc < best || (oc == best && ow < bw)) {
                    best = oc;
                    bw = ow;
                }
            }
            if (lane == 0) {
                s_cost[jr] = best;
                s_w[jr] = bw;
            }
        }
    }
    __syncthreads();
    if (mode == 2) {   // local batch of a sharded run: report, do not accept
        if (tid < nb) {
            g.rbest[3 * tid] = s_cost[tid];
            g.rbest[3 * tid + 1] = g.w0 + s_w[tid] % g.Wr;
            g.rbest[3 * tid + 2] = s_w[tid];
        }
        if (tid == 0)
            g.scal[GV_LOCAL_NB] = nb;
        // the fallback plan costs were read above; the plans stay for export
        __syncthreads();
        for (int i = tid; i < g.fb_slots; i += blockDim.x)
            g.scal[GV_FBCOST0 + i] = 0;
        return;
    }
    if (tid == 0) {
        int acc = 0, win = 0, used = nb;
        if (mode == 1) {
            int64_t k = g.scal[GV_STRENGTH];
            for (int jr = 0; jr < nb; ++jr) {
                win = jr;
                acc = s_cost[jr] < g.scal[GV_INC_COST];
                k = (acc || k >= g.k_max) ? 1 : k + 1;
                if (acc) {
                    used = jr + 1;
                    break;
                }
            }
            g.scal[GV_STRENGTH] = k;
        }
        g.scal[GV_BEST_COST] = s_cost[win];
        g.scal[GV_BEST_W] = g.w0 + s_w[win] % g.Wr;
        g.scal[GV_ROUND] = r0 + used;
        if (round_arg < 0)
            g.scal[GV_NB] = acc ? 1 : (2 * nb < g.B ? 2 * nb : g.B);
        s_accept = mode == 0 ? 1 : acc;
        s_win = win;
    }
    __syncthreads();
    for (int i = tid; i < g.fb_slots; i += blockDim.x)
        g.scal[GV_FBCOST0 + i] = 0;   // read (gv_worker_cost) before the barrier above
    const int win = s_win;
    if (!s_accept)
        return;
    const int w = s_w[win];
    const long long wcost = s_cost[win];
    // the candidate: F with the winner's touched rows, or its fallback plan
    uint8_t *dst = mode == 0 ? g.cand : g.inc;
    const int64_t KT2 = 2 * g.KT;
    if (g.fb[w]) {
        const uint8_t *src = g.fbplan + (int64_t)g.fbslot[w] * KT2;
        for (int64_t i = tid; i < KT2; i += blockDim.x) {
            dst[i] = src[i];
            if (mode == 1)
                g.F[i] = src[i];
        }
        if (mode == 1)
            for (int64_t k = tid; k < g.K; k += blockDim.x)
                g.Fcost[k] = g.fbpcost[(int64_t)g.fbslot[w] * g.K + k];
    } else {
        if (mode == 0 || !g.scal[GV_INC_IS_F])
            for (int64_t i = tid; i < KT2; i += blockDim.x)
                dst[i] = g.F[i];
        __syncthreads();
        const int NW = g.NW, T = g.T;
        const int n = g.tn[w];
        for (int64_t q = tid; q < (int64_t)n * T; q += blockDim.x) {
            const int j = (int)(q / T), t = (int)(q % T);
            const int64_t k = g.tp[(int64_t)w * g.tcap + j];
            const uint32_t *row = g.tw + ((int64_t)w * g.tcap + j) * 2 * NW;
            const uint8_t bm = (row[t >> 5] >> (t & 31)) & 1u, br = (row[NW + (t >> 5)] >> (t & 31)) & 1u;
            dst[k * T + t] = bm;
            dst[g.KT + k * T + t] = br;
            if (mode == 1) {
                g.F[k * T + t] = bm;
                g.F[g.KT + k * T + t] = br;
            }
        }
        if (mode == 1 && tid < n)
            g.Fcost[g.tp[(int64_t)w * g.tcap + tid]] = g.tcost[(int64_t)w * g.tcap + tid];
    }
    __syncthreads();
    if (mode == 1 && tid == 0) {
        g.scal[GV_INC_COST] = wcost;
        g.scal[GV_FTOT] = wcost;
        g.scal[GV_INC_IS_F] = 1;
        g.scal[GV_ACCEPTED] += 1;
    }
}

// ------------------------------------------------------------------ host

struct GvnsState {
    GvnsArgs a{};
    int k_vnd_max = 4;
    size_t tail_bytes = 0;
    void *blocks[24] = {};
    int nblocks = 0;
    // rl_gvns_run's batch (shake, VND tasks, join) as one CUDA graph: its
    // arguments are fixed between rl_gvns_begin calls except max_rounds
    cudaGraphExec_t graph = nullptr;
    int64_t graph_max = -1;
    int runs = 0;
    cudaGraphExec_t loop = nullptr;   // rl_gvns_run_until's device-resident loop
    int vbytes = 0;   // value width the shake scratch was sized for
};

static void gvns_free(GvnsState *gs)
{
    if (!gs)
        return;
    if (gs->graph)
        cudaGraphExecDestroy(gs->graph);
    if (gs->loop)
        cudaGraphExecDestroy(gs->loop);
    for (int i = 0; i < gs->nblocks; ++i)
        if (gs->blocks[i])
            cudaFree(gs->blocks[i]);
    delete gs;
}

template <typename P>
static cudaError_t gv_alloc(GvnsState *gs, P **p, size_t bytes)
{
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes > 0 ? bytes : 8);
    if (e == cudaSuccess) {
        gs->blocks[gs->nblocks++] = q;
        *p = (P *)q;
    }
    return e;
}

template <typename V, typename C, typename Mask>
static int gv_launch_vnd(rl_instance *h, GvnsState *gs)
{
    int grid, block;
    size_t smem;
    // the slack skip shortens the long delta walks of these latency-bound
    // tasks (variant bit 3 turns it off for A/B)
    const bool skip = h->skip_mode != 2;
    const void *fn = skip ? (const void *)k_gvns_vnd<V, C, Mask, true>
                          : (const void *)k_gvns_vnd<V, C, Mask, false>;
    int rc = launch_cfg<V, C>(h, fn,
                              (int64_t)gs->a.W * gs->a.tcap + (int64_t)gs->a.fb_slots * h->K,
                              grid, smem, block);
    if (rc)
        return rc;
    if (skip)
        k_gvns_vnd<V, C, Mask, true><<<grid, block, smem, h->stream>>>(view<V>(h), gs->a,
                                                                        gs->k_vnd_max);
    else
        k_gvns_vnd<V, C, Mask, false><<<grid, block, smem, h->stream>>>(view<V>(h), gs->a,
                                                                         gs->k_vnd_max);
    CKL();
    return 0;
}

template <typename V, typename C>
static int gv_launch_shake(rl_instance *h, GvnsState *gs, int64_t round_arg,
                           int64_t max_rounds)
{
    const int W = gs->a.W;
    k_shake<V><<<(W + 3) / 4, 128, 4 * (size_t)gs->a.shake_bytes, h->stream>>>(
        view<V>(h), gs->a, round_arg, max_rounds);
    CKL();
    return 0;
}

template <typename V, typename C>
static int gv_launch_prefix(rl_instance *h, GvnsState *gs)
{
    const int64_t warps = h->K < 148 * 64 ? h->K : 148 * 64;
    k_gvns_prefix<V><<<(unsigned)((warps + 7) / 8), 256, 0, h->stream>>>(view<V>(h),
                                                                         (V *)gs->a.pfx);
    CKL();
    return 0;
}

extern "C" int rl_gvns_begin_batch(rl_instance *h, int workers, int batch, int64_t worker_offset,
                                   int k_max, int k_vnd_max, uint64_t seed, const uint8_t *sm,
                                   const uint8_t *sr, int64_t *inc_cost)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !sm || !sr || workers < 1 || batch < 1 || batch > 32 ||
        (int64_t)workers * batch > (1 << 20) || worker_offset < 0 || k_max < 1 ||
        k_vnd_max < 1 || k_vnd_max > 4)
        return fail(RL_EINVAL,
                    "rl_gvns_begin: bad arguments (workers=%d batch=%d k_max=%d k_vnd_max=%d)",
                    workers, batch, k_max, k_vnd_max);
    const int slots = workers * batch;
    CK(cudaSetDevice(h->device));
    const int64_t K = h->K, KT = K * h->T, pop = 2 * KT;
    const int T = h->T, NW = (T + 31) / 32;
    const int64_t keff_max = k_max < pop ? k_max : pop;
    GvnsState *gs = h->gv;
    const bool reuse = gs && gs->a.Wr == workers && gs->a.B == batch && gs->a.k_max == k_max &&
                       gs->vbytes == h->vbytes;
    if (!reuse) {
        gvns_free(gs);
        h->gv = gs = new GvnsState();
        gs->vbytes = h->vbytes;
        GvnsArgs &a = gs->a;
        a.K = K;
        a.KT = KT;
        a.pop = pop;
        a.T = T;
        a.NW = NW;
        a.W = slots;
        a.Wr = workers;
        a.B = batch;
        a.k_max = k_max;
        a.kcap = (int)keff_max;
        a.tcap = (int)(keff_max < K ? keff_max : K);
        a.tsize = (int)(choice_table_mask(keff_max) + 1);
        {
            const size_t b = align16((size_t)a.tsize * 8) + align16((size_t)a.kcap * 8) +
                             align16((size_t)a.tcap * 8) + align16((size_t)a.tcap * 2 * NW * 4);
            a.shake_bytes = 4 * b <= 48 * 1024 ? (int)b : 0;
        }
        // fallback plans: enough slots for one round's workers (speculative
        // rounds past a slot overflow are truncated by the join) within a
        // 512 MB budget
        const double per_slot = (double)pop * (1 + 8) + 8.0 * K;
        int fbs = (int)(512.0 * (1 << 20) / per_slot);
        fbs = fbs < 1 ? 1 : fbs;
        fbs = fbs > slots ? slots : fbs;
        const int fcap = workers > 64 ? workers : 64;
        a.fb_slots = fbs > fcap ? fcap : fbs;
        if (const char *env = getenv("RL_GVNS_FB_SLOTS")) {   // test hook: fewer slots
            const int n = atoi(env);
            if (n >= 1 && n < a.fb_slots)
                a.fb_slots = n;
        }
        cudaError_t e = gv_alloc(gs, &a.inc, 4 * (size_t)pop);
        if (e == cudaSuccess) {
            a.F = a.inc + pop;
            a.init = a.F + pop;
            a.cand = a.init + pop;
            e = gv_alloc(gs, &a.Fcost, K * 8);
        }
        if (e == cudaSuccess) e = gv_alloc(gs, &a.scal, (GV_FBCOST0 + a.fb_slots) * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.pos, (size_t)slots * a.kcap * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.table, (size_t)slots * a.tsize * 8);
        if (e == cudaSuccess && choice_uses_tail_shuffle(pop, keff_max))
            e = gv_alloc(gs, &a.tailidx, (size_t)slots * pop * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.tp, (size_t)slots * a.tcap * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.tn, (size_t)slots * 3 * sizeof(int));
        if (e == cudaSuccess) {
            a.fb = a.tn + slots;
            a.fbslot = a.fb + slots;
            e = gv_alloc(gs, &a.tw, (size_t)slots * a.tcap * 2 * NW * 4);
        }
        if (e == cudaSuccess) e = gv_alloc(gs, &a.tcost, (size_t)slots * a.tcap * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.tasks, (size_t)slots * a.tcap * sizeof(int));
        if (e == cudaSuccess) e = gv_alloc(gs, &a.rng, (size_t)slots * sizeof(PhiloxState));
        if (e == cudaSuccess) e = gv_alloc(gs, &a.fbplan, (size_t)a.fb_slots * pop);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.fbdiff, (size_t)a.fb_slots * pop * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.fbpcost, (size_t)a.fb_slots * K * 8);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.queue, 16);
        if (e == cudaSuccess) e = gv_alloc(gs, &a.rbest, (size_t)batch * 3 * 8);
        if (e == cudaSuccess)
            e = gv_alloc(gs, (unsigned char **)&a.pfx, (size_t)K * 2 * (T + 1) * h->vbytes);
        if (e != cudaSuccess) {
            gvns_free(gs);
            h->gv = nullptr;
            return fail(RL_ECUDA, "rl_gvns_begin: %s", cudaGetErrorString(e));
        }
    }
    GvnsArgs &a = gs->a;
    a.seed = seed;
    a.w0 = worker_offset;
    if (gs->graph) {   // captured with the previous arguments
        cudaGraphExecDestroy(gs->graph);
        gs->graph = nullptr;
    }
    if (gs->loop) {
        cudaGraphExecDestroy(gs->loop);
        gs->loop = nullptr;
    }
    gs->runs = 0;
    gs->k_vnd_max = k_vnd_max;
    // incumbent, lot-for-lot start, and F = per-product VND image of the incumbent
    CK(cudaMemcpyAsync(a.inc, sm, KT, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(a.inc + KT, sr, KT, cudaMemcpyHostToDevice, h->stream));
    int rc = rl_initial_solution_device(h, a.init, a.init + KT, h->stream);
    if (rc)
        return rc;
    if ((rc = RL_DISPATCH(h, gv_launch_prefix, h, gs)))
        return rc;
    rc = rl_vnd_device(h, k_vnd_max, a.inc, a.inc + KT, a.F, a.F + KT, h->stream);
    if (rc)
        return rc;
    CK(cudaMemcpyAsync(a.Fcost, h->p64 + K, K * 8, cudaMemcpyDeviceToDevice, h->stream));
    int64_t sum[16];
    CK(cudaMemcpyAsync(sum, h->summary, sizeof sum, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (sum[1] == RL_INFEASIBLE)
        return fail(RL_EINVAL, "rl_gvns_begin: the incumbent plan is infeasible");
    int64_t scal[GV_FBCOST0] = {};
    scal[GV_INC_COST] = sum[1];
    scal[GV_FTOT] = sum[0];
    scal[GV_STRENGTH] = 1;
    scal[GV_INC_IS_F] = 0;
    scal[GV_ROUND] = 0;
    scal[GV_NB] = 1;
    scal[GV_NTASK] = 0;
    CK(cudaMemsetAsync(a.scal, 0, (GV_FBCOST0 + a.fb_slots) * sizeof(int64_t), h->stream));
    CK(cudaMemsetAsync(a.queue, 0, 16, h->stream));
    CK(cudaMemcpyAsync(a.scal, scal, sizeof scal, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (inc_cost)
        *inc_cost = sum[1];
    return 0;
}

extern "C" int rl_gvns_begin(rl_instance *h, int workers, int64_t worker_offset, int k_max,
                             int k_vnd_max, uint64_t seed, const uint8_t *sm, const uint8_t *sr,
                             int64_t *inc_cost)
{
    RL_GUARD(h);
    return rl_gvns_begin_batch(h, workers, 1, worker_offset, k_max, k_vnd_max, seed, sm, sr,
                               inc_cost);
}

extern "C" int rl_gvns_set_strength(rl_instance *h, int64_t strength)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || strength < 1)
        return fail(RL_EINVAL, "rl_gvns_set_strength: bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(&h->gv->a.scal[GV_STRENGTH], &strength, 8, cudaMemcpyHostToDevice,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

// shake -> fallback -> VND tasks -> join of one batch (round_arg < 0: at the
// device round counter), enqueued on the handle's stream
static int gv_launch_round(rl_instance *h, int64_t round_arg, int64_t max_rounds, int mode)
{
    GvnsState *gs = h->gv;
    int rc = RL_DISPATCH(h, gv_launch_shake, h, gs, round_arg, max_rounds);
    if (rc)
        return rc;
    if ((rc = RL_DISPATCH_M(h, gv_launch_vnd, h, gs)))
        return rc;
    k_gvns_join<<<1, 1024, 0, h->stream>>>(gs->a, mode, round_arg, max_rounds);
    CKL();
    return 0;
}

extern "C" int rl_gvns_round(rl_instance *h, int64_t round_index, int accept)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || round_index < 0)
        return fail(RL_EINVAL, "rl_gvns_round: call rl_gvns_begin first");
    CK(cudaSetDevice(h->device));
    return gv_launch_round(h, round_index, round_index + 1, accept ? 1 : 0);
}

extern "C" int rl_gvns_run(rl_instance *h, int64_t max_rounds)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || max_rounds < 0)
        return fail(RL_EINVAL, "rl_gvns_run: call rl_gvns_begin_batch first");
    CK(cudaSetDevice(h->device));
    GvnsState *gs = h->gv;
    if (gs->graph && gs->graph_max == max_rounds) {
        CK(cudaGraphLaunch(gs->graph, h->stream));
        h->launches += 3;
        return 0;
    }
    if (gs->runs++ == 0)   // first batch launched plainly (sets kernel attributes)
        return gv_launch_round(h, -1, max_rounds, 1);
    if (gs->graph) {
        cudaGraphExecDestroy(gs->graph);
        gs->graph = nullptr;
    }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = h->launches;
    const int rc = gv_launch_round(h, -1, max_rounds, 1);
    const cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    h->launches = l0;
    if (rc) {
        if (e == cudaSuccess)
            cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess)
        return fail(RL_ECUDA, "rl_gvns_run: capture: %s", cudaGetErrorString(e));
    const cudaError_t ei = cudaGraphInstantiate(&gs->graph, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        gs->graph = nullptr;
        return fail(RL_ECUDA, "rl_gvns_run: graph: %s", cudaGetErrorString(ei));
    }
    gs->graph_max = max_rounds;
    CK(cudaGraphLaunch(gs->graph, h->stream));
    h->launches += 3;
    return 0;
}

extern "C" int rl_gvns_state(rl_instance *h, int which, uint8_t *sm, uint8_t *sr, int64_t *info)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || !info)
        return fail(RL_EINVAL, "rl_gvns_state: bad arguments");
    CK(cudaSetDevice(h->device));
    GvnsArgs &a = h->gv->a;
    int64_t scal[GV_FBCOST0];
    CK(cudaMemcpyAsync(scal, a.scal, sizeof scal, cudaMemcpyDeviceToHost, h->stream));
    const uint8_t *src = which == 0 ? a.inc : a.cand;
    if (sm)
        CK(cudaMemcpyAsync(sm, src, a.KT, cudaMemcpyDeviceToHost, h->stream));
    if (sr)
        CK(cudaMemcpyAsync(sr, src + a.KT, a.KT, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (scal[GV_ERROR])
        return fail(RL_ECUDA, "gvns: more shake fallbacks in one round than slots (%d)",
                    a.fb_slots);
    info[0] = scal[GV_INC_COST];
    info[1] = scal[GV_STRENGTH];
    info[2] = scal[GV_BEST_COST];
    info[3] = scal[GV_BEST_W];
    info[4] = scal[GV_ACCEPTED];
    info[5] = scal[GV_FB_COUNT];
    info[6] = scal[GV_ROUND];
    return 0;
}

// Sharded rounds (BASELINE config 5): each rank runs a
// contiguous block of workers; the job joins the per-rank bests and every rank
// adopts the global winner.  rl_gvns_candidate copies this rank's best
// candidate (after rl_gvns_round(accept = 0)) to a device buffer (2KT bytes,
// m rows then r rows) and returns (cost, global worker) on the host;
// rl_gvns_import makes a plan (a VND fixpoint) the incumbent and its own F.
extern "C" int rl_gvns_candidate(rl_instance *h, uint8_t *d_plan, int64_t *best)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || !best)
        return fail(RL_EINVAL, "rl_gvns_candidate: bad arguments");
    CK(cudaSetDevice(h->device));
    GvnsArgs &a = h->gv->a;
    int64_t scal[GV_FBCOST0];
    if (d_plan)
        CK(cudaMemcpyAsync(d_plan, a.cand, 2 * a.KT, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync(scal, a.scal, sizeof scal, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (scal[GV_ERROR])
        return fail(RL_ECUDA, "gvns: more shake fallbacks in one round than slots (%d)",
                    a.fb_slots);
    best[0] = scal[GV_BEST_COST];
    best[1] = scal[GV_BEST_W];
    return 0;
}

extern "C" int rl_gvns_import(rl_instance *h, const uint8_t *d_plan, int64_t cost)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || !d_plan)
        return fail(RL_EINVAL, "rl_gvns_import: bad arguments");
    CK(cudaSetDevice(h->device));
    GvnsArgs &a = h->gv->a;
    CK(cudaMemcpyAsync(a.inc, d_plan, 2 * a.KT, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync(a.F, d_plan, 2 * a.KT, cudaMemcpyDeviceToDevice, h->stream));
    const size_t kt = (size_t)a.KT;
    CK(cudaMemcpyAsync(h->plan, d_plan, 2 * kt, cudaMemcpyDeviceToDevice, h->stream));
    int rc = RL_DISPATCH_M(h, do_costs, h, (int64_t)0, h->K, a.Fcost);
    if (rc)
        return rc;
    int64_t scal[4] = {cost, cost, 0, 1};   // inc cost, Ftot, (strength kept), inc_is_F
    CK(cudaMemcpyAsync(&a.scal[GV_INC_COST], &scal[0], 16, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(&a.scal[GV_INC_IS_F], &scal[3], 8, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

// ---- device-resident GVNS loop (rl_gvns_run_until)
__device__ inline int64_t gv_now_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

__global__ void k_gvns_t0(GvnsArgs g) { g.scal[GV_T0] = gv_now_ns(); }

// The loop condition, evaluated after every batch (gvns.py:200-206 checks
// the clock and the round cap before every round): another batch while the
// round cap is not reached, the budget not spent and no error raised.
__global__ void k_gvns_cond(GvnsArgs g, cudaGraphConditionalHandle hnd)
{
    const bool go = g.scal[GV_ROUND] < g.scal[GV_MAXR] &&
                    gv_now_ns() - g.scal[GV_T0] <= g.scal[GV_TBUDGET] && !g.scal[GV_ERROR];
    cudaGraphSetConditional(hnd, go ? 1u : 0u);
}

// gvns()'s whole loop (gvns.py:200-215) on the device: one graph launch runs
// speculative batches (shake, VND tasks, join + acceptance) inside a
// conditional WHILE node until max_rounds rounds are done or budget_ns of
// device time (%globaltimer) has passed, the check made between batches; the
// host waits once.  The graph is built on the first call after a begin
// and replayed with new caps (read from the device scalars).  Synchronous.
extern "C" int rl_gvns_run_until(rl_instance *h, int64_t max_rounds, int64_t budget_ns)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || max_rounds < 0)
        return fail(RL_EINVAL, "rl_gvns_run_until: call rl_gvns_begin_batch first");
    CK(cudaSetDevice(h->device));
    GvnsState *gs = h->gv;
    if (!gs->loop) {
        if (gs->runs++ == 0) {   // kernel attributes are set by a plain launch first
            int64_t zero = 0;
            CK(cudaMemcpyAsync(&gs->a.scal[GV_MAXR], &zero, 8, cudaMemcpyHostToDevice, h->stream));
            int rc = gv_launch_round(h, -1, -1, 1);   // no rounds (cap 0): sets attributes only
            if (rc)
                return rc;
        }
        cudaGraph_t g = nullptr;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hnd;
        cudaGraphNode_t t0node, loop;
        cudaError_t e = cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault);
        cudaGraph_t body = nullptr;
        if (e == cudaSuccess) {
            cudaKernelNodeParams kp = {};
            void *args[] = {(void *)&gs->a};
            kp.func = (void *)k_gvns_t0;
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(1);
            kp.kernelParams = args;
            e = cudaGraphAddKernelNode(&t0node, g, nullptr, 0, &kp);
        }
        if (e == cudaSuccess) {
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = hnd;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            e = cudaGraphAddNode(&loop, g, &t0node, 1, &cp);
            if (e == cudaSuccess)
                body = cp.conditional.phGraph_out[0];
        }
        if (e == cudaSuccess)
            e = cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
            cudaGraphDestroy(g);
            return fail(RL_ECUDA, "rl_gvns_run_until: graph: %s", cudaGetErrorString(e));
        }
        const int64_t l0 = h->launches;
        int rc = gv_launch_round(h, -1, -1, 1);
        if (!rc) {
            k_gvns_cond<<<1, 1, 0, h->stream>>>(gs->a, hnd);
            rc = cudaGetLastError() == cudaSuccess ? 0 : fail(RL_ECUDA, "k_gvns_cond launch");
        }
        cudaGraph_t cap = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(h->stream, &cap);
        h->launches = l0;
        if (rc || ec != cudaSuccess) {
            cudaGraphDestroy(g);
            return rc ? rc : fail(RL_ECUDA, "rl_gvns_run_until: capture: %s", cudaGetErrorString(ec));
        }
        e = cudaGraphInstantiate(&gs->loop, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            gs->loop = nullptr;
            return fail(RL_ECUDA, "rl_gvns_run_until: instantiate: %s", cudaGetErrorString(e));
        }
    }
    int64_t caps[2] = {max_rounds, budget_ns < 0 ? 0 : budget_ns};
    CK(cudaMemcpyAsync(&gs->a.scal[GV_MAXR], caps, sizeof caps, cudaMemcpyHostToDevice, h->stream));
    CK(cudaGraphLaunch(gs->loop, h->stream));
    h->launches += 5;   // t0, and per batch shake, VND, join, condition (counted once)
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

// Candidate of batch round jr of the last local batch (mode 2): F with the
// round's best worker's touched rows, or its fallback plan (one block).
__global__ void k_gvns_export(GvnsArgs g, int jr, uint8_t *dst)
{
    const int w = (int)g.rbest[3 * jr + 2];
    RL_ASSERT(w >= 0 && w < g.W && (!g.fb[w] || g.fbslot[w] < g.fb_slots));
    const int tid = threadIdx.x;
    const int64_t KT2 = 2 * g.KT;
    if (g.fb[w]) {
        const uint8_t *src = g.fbplan + (int64_t)g.fbslot[w] * KT2;
        for (int64_t i = tid; i < KT2; i += blockDim.x)
            dst[i] = src[i];
        return;
    }
    for (int64_t i = tid; i < KT2; i += blockDim.x)
        dst[i] = g.F[i];
    __syncthreads();
    const int NW = g.NW, T = g.T, n = g.tn[w];
    for (int64_t q = tid; q < (int64_t)n * T; q += blockDim.x) {
        const int j = (int)(q / T), t = (int)(q % T);
        const int64_t k = g.tp[(int64_t)w * g.tcap + j];
        const uint32_t *row = g.tw + ((int64_t)w * g.tcap + j) * 2 * NW;
        dst[k * T + t] = (row[t >> 5] >> (t & 31)) & 1u;
        dst[g.KT + k * T + t] = (row[NW + (t >> 5)] >> (t & 31)) & 1u;
    }
}

// Sharded replicas in speculative batches (sharded.sharded_gvns): rounds
// round0 .. round0 + nb - 1 (nb <= the begin's batch) with this rank's
// worker block, each shaking the incumbent with the strength it has if the
// rounds before it do not improve (strength set by rl_gvns_set_strength);
// no acceptance.  out[3j .. 3j+2] = round j's best (cost, global worker,
// local slot); *n_out = rounds with valid bests (fewer when fallback slots
// ran out: the rest are re-run by the caller).  Synchronous.
extern "C" int rl_gvns_run_local(rl_instance *h, int64_t round0, int nb, int64_t *out,
                                 int64_t *n_out)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || round0 < 0 || nb < 1 || nb > h->gv->a.B || !out || !n_out)
        return fail(RL_EINVAL, "rl_gvns_run_local: bad arguments");
    CK(cudaSetDevice(h->device));
    int rc = gv_launch_round(h, round0, round0 + nb, 2);
    if (rc)
        return rc;
    GvnsArgs &a = h->gv->a;
    int64_t scal[GV_FBCOST0];
    CK(cudaMemcpyAsync(scal, a.scal, sizeof scal, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(out, a.rbest, (size_t)nb * 3 * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (scal[GV_ERROR])
        return fail(RL_ECUDA, "gvns: more shake fallbacks in one round than slots (%d)",
                    a.fb_slots);
    *n_out = scal[GV_LOCAL_NB];
    return 0;
}

// Copy the candidate of round jr of the last local batch to device memory
// d_plan (2KT bytes: m rows then r rows).  Synchronous.
extern "C" int rl_gvns_export(rl_instance *h, int jr, uint8_t *d_plan)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !h->gv || jr < 0 || jr >= h->gv->a.B || !d_plan)
        return fail(RL_EINVAL, "rl_gvns_export: bad arguments");
    CK(cudaSetDevice(h->device));
    k_gvns_export<<<1, 1024, 0, h->stream>>>(h->gv->a, jr, d_plan);
    CKL();
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

// Test hook: the numpy-exact RNG on the device (raw draws, choice, shuffle).
__global__ void k_rng_probe(uint64_t seed, uint64_t round, uint64_t worker, int64_t pop,
                            int64_t size, int64_t shuffle_n, int64_t *out, uint64_t *table,
                            int64_t *idx)
{
    Philox g;
    g.seed(seed, round, worker);
    for (int i = 0; i < 4; ++i)
        out[i] = (int64_t)g.next64();
    if (choice_uses_tail_shuffle(pop, size))
        choice_tail(g, pop, size, out + 4, idx);
    else
        choice_floyd(g, pop, size, out + 4, table);
    int64_t *sh = out + 4 + size;
    for (int64_t i = 0; i < shuffle_n; ++i)
        sh[i] = 3 * i + 1;
    g.shuffle(sh, shuffle_n);
    out[4 + size + shuffle_n] = (int64_t)g.next64();
}

extern "C" int rl_rng_probe(uint64_t seed, uint64_t round, uint64_t worker, int64_t pop,
                            int64_t size, int64_t shuffle_n, int64_t *out)
{
    (void)cudaGetLastError();
    if (!out || pop < 1 || size < 0 || size > pop || shuffle_n < 0 || size > (1 << 20) ||
        shuffle_n > (1 << 20) || (choice_uses_tail_shuffle(pop, size) && pop > ((int64_t)1 << 26)))
        return fail(RL_EINVAL, "rl_rng_probe: bad arguments");
    const int64_t n_out = 4 + size + shuffle_n + 1;
    const uint64_t tsize = choice_table_mask(size) + 1;
    const bool tail = choice_uses_tail_shuffle(pop, size);
    int64_t *d;
    CK(cudaMalloc(&d, (n_out + tsize + (tail ? pop : 1)) * 8));
    k_rng_probe<<<1, 1>>>(seed, round, worker, pop, size, shuffle_n, d, (uint64_t *)(d + n_out),
                          d + n_out + tsize);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpy(out, d, n_out * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess)
        return fail(RL_ECUDA, "rl_rng_probe: %s", cudaGetErrorString(e));
    return 0;
}
