// vnd_packed.cuh -- two products per warp, lockstep sweeps (T <= 64).
//
// One product's pass has only ~40 moves at T = 52, so a warp-wide walk queue
// over one product idles lanes while the longest walk finishes (ncu: ~58%
// SIMT efficiency in k_vnd).  Here a warp owns two products (lane groups
// 0-15 and 16-31), runs their sweeps in lockstep (same neighborhood at the
// same time) and feeds the moves of BOTH products into one walk queue.
// Per-group work (staging, prefix sums, base pass, move enumeration) runs on
// 16 lanes per product with width-16 shuffles; the walk queue, the argmin
// reductions and the (register) row updates are warp-wide.  A product that
// finishes its VND (a sweep without improvement) is replaced at the sweep
// boundary by the next product from the global queue.  Each product follows
// exactly its solo trajectory (products never interact), so results equal
// k_vnd's bit for bit; the GPU tests run both kernels.
#pragma once

namespace rl {

constexpr unsigned HALF_LO = 0x0000ffffu;

__device__ inline uint64_t shfl64(uint64_t v, int src)
{
    const uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src);
    const uint32_t hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src);
    return (uint64_t)lo | ((uint64_t)hi << 32);
}

// prefix sums of the staged rows, 16 lanes per product; returns K0
template <typename V, typename C>
__device__ inline C build_prefix16(const Slot<V, C> &s, int T, const ProductCosts<C> &pc, int q,
                                   unsigned gm)
{
    V carry_d = 0, carry_r = 0;
    C sum_cd = 0, sum_cr = 0;
    if (q == 0) {
        s.cd[0] = 0;
        s.cr[0] = 0;
    }
    for (int base = 0; base < T; base += 16) {
        const int t = base + q;
        V d = t < T ? s.stage[t] : V(0);
        V r = t < T ? s.stage[T + t] : V(0);
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) {
            const V od = __shfl_up_sync(gm, d, off, 16), orr = __shfl_up_sync(gm, r, off, 16);
            if (q >= off) {
                d += od;
                r += orr;
            }
        }
        d += carry_d;
        r += carry_r;
        if (t < T) {
            s.cd[t + 1] = d;
            s.cr[t + 1] = r;
            sum_cd += C(d);
            sum_cr += C(r);
        }
        carry_d = __shfl_sync(gm, d, 15, 16);
        carry_r = __shfl_sync(gm, r, 15, 16);
    }
#pragma unroll
    for (int off = 8; off; off >>= 1) {
        sum_cd += __shfl_xor_sync(gm, sum_cd, off, 16);
        sum_cr += __shfl_xor_sync(gm, sum_cr, off, 16);
    }
    __syncwarp(gm);
    return pc.hr * sum_cr - pc.hm * sum_cd;
}

// group-aware staging completion (TMA, or plain loads on 16 lanes)
template <typename V, typename C>
__device__ inline void stage_end16(const Slot<V, C> &s, const InstView<V> &in, int64_t k, int q,
                                   uint32_t &phase, unsigned gm)
{
    if (tma_ok(in, k)) {
        mbar_wait(s.bar, phase);
        phase ^= 1;
    } else {
        const V *d = in.dem + k * (int64_t)in.T, *r = in.ret + k * (int64_t)in.T;
        for (int t = q; t < in.T; t += 16) {
            s.stage[t] = d[t];
            s.stage[in.T + t] = r[t];
        }
    }
    __syncwarp(gm);
}

// base pass of each group's own product on its 16 lanes (cf. base_pass)
template <typename V, typename C>
__device__ inline bool base_pass16(const Slot<V, C> &s, const MaskReg &mk, int T,
                                   const ProductCosts<C> &pc, int q, unsigned gmask, C &S)
{
    const int L = (T + 15) >> 4;
    const int lo = q * L, hi = min(lo + L, T);
    const V INF = VInf<V>::value;
    V A = 0, B = INF;
    for (int u = lo; u < hi; ++u) {
        if (!mk.r(u))
            continue;
        const int v = mk.next(u + 1);
        const V seg = s.cd[v] - s.cd[u];
        A += seg;
        B = vmin<V>(B + seg, s.cr[u + 1]);
    }
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        const V a2 = __shfl_up_sync(FULL, A, off, 16), b2 = __shfl_up_sync(FULL, B, off, 16);
        if (q >= off) {
            B = vmin<V>(b2 + A, B);
            A = a2 + A;
        }
    }
    const V pa = __shfl_up_sync(FULL, A, 1, 16), pb = __shfl_up_sync(FULL, B, 1, 16);
    V X = q == 0 ? V(0) : vmin<V>(pa, pb);
    C local = 0;
    bool ok = true;
    for (int u = lo; u < hi; ++u) {
        const bool m = mk.m(u), r = mk.r(u);
        if (!(m | r))
            continue;
        const int v = mk.next(u + 1);
        s.xin[u] = X;
        s.cpre[u] = local;
        C c;
        V xr;
        ok &= seg_cost<V, C>(s.cd, s.cr, T, u, v, m, r, X, pc, c, xr);
        local += c;
        X += xr;
    }
    C incl = local;
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        const C o = __shfl_up_sync(FULL, incl, off, 16);
        if (q >= off)
            incl += o;
    }
    const C excl = incl - local;
    if (excl != C(0))
        for (int u = lo; u < hi; ++u)
            if (mk.m(u) | mk.r(u))
                s.cpre[u] += excl;
    S = __shfl_sync(FULL, incl, 15, 16);
    const int f = mk.next(0);
    ok = ok && s.cd[f] == 0;
    const bool feas = (__ballot_sync(FULL, !ok) & gmask) == 0;
    __syncwarp();
    return feas;
}

// canonical move slots of each group's own product -> s.mv; returns the count
__device__ inline int enumerate16(uint16_t *mv, const MaskReg &mk, int nbh, int T, int q, int g,
                                  bool active)
{
    if (!active)
        return 0;   // group-uniform
    if (nbh <= 2)
        return T;
    const int nslots = nbh == 3 ? 4 * T : T;
    int n = 0;
    for (int base = 0; base < nslots; base += 16) {
        const int slot = base + q;
        const bool ok = slot < nslots && slot_valid(mk, nbh, slot, T);
        const unsigned bal = (__ballot_sync(HALF_LO << (16 * g), ok) >> (16 * g)) & HALF_LO;
        if (ok)
            mv[n + __popc(bal & ((1u << q) - 1))] = (uint16_t)slot;
        n += __popc(bal);
    }
    return n;
}

__device__ inline int move_count16(const MaskReg &mk, int nbh, int T, int q, int g)
{
    if (nbh <= 2)
        return T;
    const int nslots = nbh == 3 ? 4 * T : T;
    int n = 0;
    for (int base = 0; base < nslots; base += 16) {
        const int slot = base + q;
        n += __popc((__ballot_sync(HALF_LO << (16 * g),
                                   slot < nslots && slot_valid(mk, nbh, slot, T)) >>
                     (16 * g)) & HALF_LO);
    }
    return n;
}

template <typename V, typename C>
__global__ void __launch_bounds__(128, 4) k_vnd_pack2(InstView<V> in, const uint8_t *sm_in,
                                                      const uint8_t *sr_in, uint8_t *sm_out,
                                                      uint8_t *sr_out, int k_max, VndOut o)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = in.T;
    const int g = lane >> 4, q = lane & 15;
    const unsigned gmask = HALF_LO << (16 * g);
    const size_t sb = slot_bytes<V, C>(T);
    unsigned char *wbase = smem + (size_t)warp * 2 * sb;
    const Slot<V, C> s0 = carve<V, C>(wbase, T);
    const Slot<V, C> so = carve<V, C>(wbase + g * sb, T);   // own group's slot
    if (q == 0)
        mbar_init(so.bar);
    __syncwarp();
    uint32_t phase = 0;
    const int64_t NONE = o.k_hi;

    // lockstep state of both products, warp-uniform (held by every lane)
    int64_t kk[2] = {NONE, NONE}, evals[2] = {0, 0};
    int sweeps[2] = {0, 0}, moves[2] = {0, 0};
    bool feas[2] = {false, false}, want[2] = {true, true}, dirty[2] = {false, false};
    C S[2] = {0, 0}, S0[2] = {0, 0}, K0[2] = {0, 0};
    MaskReg mk[2] = {MaskReg{0, 0, T}, MaskReg{0, 0, T}};
    ProductCosts<C> pco{};   // own group's product
    ProductCosts<C> pcs[2];  // both, for the walks
    pcs[0] = pco;
    pcs[1] = pco;

    // each group prefetches its next product's rows (TMA) into its stage
    int64_t nxt = 0;
    if (q == 0)
        nxt = o.k_lo + atomicAdd(o.queue, 1);
    nxt = __shfl_sync(FULL, nxt, 16 * g);
    if (nxt < o.k_hi)
        stage_begin(so, in, nxt, q);

    for (;;) {
        // ---------------- sweep boundary: (re)load finished groups
        if (want[0] | want[1]) {
            const bool w_own = want[g];
            int64_t k_own = kk[g];
            uint64_t M = 0, R = 0;
            C K0o = 0;
            if (w_own) {
                k_own = nxt;
                const bool ld = k_own < o.k_hi;
                if (ld) {
                    stage_end16(so, in, k_own, q, phase, gmask);
                    pco = load_costs<C>(in.cost6, in.K, k_own);
                    const uint8_t *a = sm_in + k_own * (int64_t)T, *b = sr_in + k_own * (int64_t)T;
                    for (int base = 0; base < T; base += 16) {
                        const int t = base + q;
                        const unsigned bm = (__ballot_sync(gmask, t < T && a[t]) >> (16 * g)) & HALF_LO;
                        const unsigned br = (__ballot_sync(gmask, t < T && b[t]) >> (16 * g)) & HALF_LO;
                        M |= (uint64_t)bm << base;
                        R |= (uint64_t)br << base;
                    }
                    K0o = build_prefix16(so, T, pco, q, gmask);
                    int64_t n2 = 0;
                    if (q == 0)
                        n2 = o.k_lo + atomicAdd(o.queue, 1);
                    nxt = __shfl_sync(gmask, n2, 16 * g);
                    if (nxt < o.k_hi)
                        stage_begin(so, in, nxt, q);
                }
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t kh = __shfl_sync(FULL, k_own, 16 * h);
                const uint64_t Mh = shfl64(M, 16 * h), Rh = shfl64(R, 16 * h);
                const C K0h = __shfl_sync(FULL, K0o, 16 * h);
                if (want[h]) {
                    kk[h] = kh;
                    mk[h] = MaskReg{Mh, Rh, T};
                    K0[h] = K0h;
                    sweeps[h] = 0;
                    moves[h] = 0;
                    evals[h] = 0;
                }
                pcs[h].km = __shfl_sync(FULL, pco.km, 16 * h);
                pcs[h].kr = __shfl_sync(FULL, pco.kr, 16 * h);
                pcs[h].hm = __shfl_sync(FULL, pco.hm, 16 * h);
                pcs[h].hr = __shfl_sync(FULL, pco.hr, 16 * h);
                pcs[h].pm = __shfl_sync(FULL, pco.pm, 16 * h);
                pcs[h].pr = __shfl_sync(FULL, pco.pr, 16 * h);
            }
            if (kk[0] >= NONE && kk[1] >= NONE)
                break;
            C So;
            const bool fo = base_pass16(so, mk[g], T, pco, q, gmask, So);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const C Sh = __shfl_sync(FULL, So, 16 * h);
                const bool fh = __shfl_sync(FULL, (int)fo, 16 * h);
                if (want[h]) {
                    S[h] = S0[h] = Sh;
                    feas[h] = fh && kk[h] < NONE;
                    want[h] = false;
                    dirty[h] = false;
                }
            }
        }

        // ---------------- one lockstep sweep of both products
        bool improved[2] = {false, false};
        for (int nbh = 1; nbh <= k_max; ++nbh) {
            if (dirty[0] | dirty[1]) {
                C So;
                const bool fo = base_pass16(so, mk[g], T, pco, q, gmask, So);
                (void)fo;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const C Sh = __shfl_sync(FULL, So, 16 * h);
                    if (dirty[h])
                        S[h] = Sh;
                    dirty[h] = false;
                }
            }
            const bool act_own = feas[g];
            const int n_own = enumerate16(so.mv, mk[g], nbh, T, q, g, act_own);
            __syncwarp();
            const int n0 = __shfl_sync(FULL, n_own, 0), n1 = __shfl_sync(FULL, n_own, 16);
            const int n = n0 + n1;
            const bool dense = nbh <= 2;
            C best[2] = {S[0], S[1]};
            int key[2] = {0x7fffffff, 0x7fffffff};
            // ---- walk queue over both products' moves
            const unsigned lt = (1u << lane) - 1;
            int idx = lane, next = 32;
            bool pend = idx < n, act = false;
            int gw = 0, slot = 0, u = 0, bb = 0;
            V X = 0;
            C acc = 0, Sw = 0;
            ProductCosts<C> pcw = pcs[0];
            PatchedReg nw;
            const V *cd = s0.cd, *cr = s0.cr, *xin = s0.xin;
            const C *cpre = s0.cpre;
            while (__any_sync(FULL, pend | act)) {
                if (pend) {
                    pend = false;
                    gw = idx >= n0;
                    const int i = gw ? idx - n0 : idx;
                    const size_t off = gw ? sb : 0;
                    cd = (const V *)((const char *)s0.cd + off);
                    cr = (const V *)((const char *)s0.cr + off);
                    xin = (const V *)((const char *)s0.xin + off);
                    cpre = (const C *)((const char *)s0.cpre + off);
                    const uint16_t *mv = (const uint16_t *)((const char *)s0.mv + off);
                    slot = dense ? i : mv[i];
                    const MaskReg mw = gw ? mk[1] : mk[0];
                    pcw = gw ? pcs[1] : pcs[0];
                    Sw = gw ? S[1] : S[0];
                    const MoveDesc d = slot_move(mw, nbh, slot, T);
                    int a;
                    nw = patch_of<V, C, MaskReg>(mw, d, a, bb);
                    u = mw.prev(a);
                    if (u < 0) {
                        u = nw.next(0);
                        acc = 0;
                        X = 0;
                        act = cd[u] == 0;
                    } else {
                        acc = cpre[u];
                        X = xin[u];
                        act = true;
                    }
                    if (act && u >= T) {
                        act = false;
                        if (acc < (gw ? best[1] : best[0])) {
                            if (gw) { best[1] = acc; key[1] = slot; }
                            else { best[0] = acc; key[0] = slot; }
                        }
                    }
                }
                if (act) {
                    const int v = nw.next(u + 1);
                    C c;
                    V xr;
                    if (!seg_cost<V, C>(cd, cr, T, u, v, nw.m(u), nw.r(u), X, pcw, c, xr)) {
                        act = false;
                    } else {
                        acc += c;
                        X += xr;
                        u = v;
                        bool done = v >= T;
                        if (!done && v > bb && X == xin[v]) {
                            acc += Sw - cpre[v];
                            done = true;
                        }
                        if (done) {
                            act = false;
                            if (gw) {
                                if (acc < best[1]) { best[1] = acc; key[1] = slot; }
                            } else {
                                if (acc < best[0]) { best[0] = acc; key[0] = slot; }
                            }
                        }
                    }
                }
                const bool idle = !(pend | act);
                const unsigned m = __ballot_sync(FULL, idle);
                if (idle) {
                    idx = next + __popc(m & lt);
                    pend = idx < n;
                }
                next += __popc(m);
            }
            // ---- per-product argmin, apply, trace
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                C bh = best[h];
                int kh = key[h];
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    const C ob = __shfl_xor_sync(FULL, bh, off);
                    const int ok = __shfl_xor_sync(FULL, kh, off);
                    if (ob < bh || (ob == bh && ok < kh)) {
                        bh = ob;
                        kh = ok;
                    }
                }
                evals[h] += h ? n1 : n0;
                if (kh != 0x7fffffff) {
                    const MoveDesc d = slot_move(mk[h], nbh, kh, T);
                    mk[h].set(d.p0, d.m0, d.r0, lane);
                    if (d.p1 >= 0)
                        mk[h].set(d.p1, d.m1, d.r1, lane);
                    if (lane == 0) {
                        if (sweeps[h] < o.cap_sweeps)
                            atomicAdd(&o.trace_dec[(int64_t)sweeps[h] * k_max + nbh - 1],
                                      (unsigned long long)(int64_t)(S[h] - bh));
                        else
                            atomicExch(o.overflow, 1);
                    }
                    S[h] = bh;
                    dirty[h] = true;
                    improved[h] = true;
                    ++moves[h];
                }
            }
        }
        // ---------------- sweep end: finished products write out
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (kk[h] < NONE) {
                ++sweeps[h];
                if (!improved[h])
                    want[h] = true;
            }
        }
        if (want[g] && kk[g] < NONE) {
            int ntot = 0;
            if (feas[g])
                for (int nbh = 1; nbh <= k_max; ++nbh)
                    ntot += move_count16(mk[g], nbh, T, q, g);
            const int64_t k = kk[g];
            uint8_t *a = sm_out + k * (int64_t)T, *b = sr_out + k * (int64_t)T;
            for (int t = q; t < T; t += 16) {
                a[t] = mk[g].m(t);
                b[t] = mk[g].r(t);
            }
            if (q == 0) {
                o.start_cost[k] = feas[g] ? (int64_t)(K0[g] + S0[g]) : RL_INFEASIBLE;
                o.final_cost[k] = feas[g] ? (int64_t)(K0[g] + S[g]) : RL_INFEASIBLE;
                o.evals[k] = evals[g];
                o.ntot[k] = ntot;
                o.sweeps[k] = sweeps[g];
                o.moves[k] = moves[g];
            }
        }
        __syncwarp();
        if (want[0] & want[1] && kk[0] >= NONE && kk[1] >= NONE)
            break;
    }
}

}  // namespace rl
