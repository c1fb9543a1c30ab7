// vnd_device.cuh -- per-product device machinery of the VND hot path.
//
// One warp owns one product at a time (north_star: "one warp or CTA per
// product").  The product's T-period slice lives in shared memory:
//
//   stage[2T]   demand row, returns row (V), landed by a 1-D TMA bulk copy
//   cd[T+1]     cd[t] = sum_{i<t} D[i]       (V)
//   cr[T+1]     cr[t] = sum_{i<t} R[i]       (V)
//   xin[T]      cumulative remanufactured quantity entering setup u (V)
//   slk[T]      remanufacturing slack CR[u] - xin[u] - seg(u) at sR setups (V)
//   lm[17]      T <= 63: masks of sR setups with slack < 2^j (j < 16), slack < 0
//   cpre[T]     sum of segment costs before setup u (C)
//   bm[NW],br[NW]  setup bit rows (uint32 words; used when T > 64)
//   mv[2T+2]    compacted move slots of the current neighborhood (uint16)
//
// For T <= 63 the setup rows live in registers instead (two warp-uniform
// uint64 masks, class MaskReg): "next/previous setup" are single bit scans
// and a candidate move's rows are built with two masked ORs.  For longer
// horizons MaskSmem scans the shared-memory words.
//
// Cost model (the reference's row_cost, _kernels.py:46-97, re-derived in
// closed form; DESIGN.md section 3 has the derivation):
//   cost = K0 + sum over segments [u,v) of
//          k_R[x_R>0] + k_M[x_M>0] + p_R x_R + p_M x_M + (T-u)(h_M seg - h_R x_R)
//   K0   = h_R * sum_t CR[t] - h_M * sum_t CD[t]
//   seg  = cd[v]-cd[u];  x_R = sR[u] ? min(seg, cr[u+1]-X) : 0;  x_M = seg-x_R
//   infeasible if x_M>0 and !sM[u], or demand before the first setup.
// X (cumulative remanufacturing) evolves as X' = sR[u] ? min(X+seg, CR[u]) : X,
// a (min,+)-affine map, so the base pass is a warp scan and a candidate
// move is scored by re-walking only the segments it touches (delta walk)
// until its X re-synchronises with the base plan, then adding the base
// plan's suffix.  All arithmetic is exact integer: C is int32 only when the
// host proved every plan's cost < 2^31 (wrapping arithmetic is then exact
// for the final values), else int64.
#pragma once
#include <cstdint>
#include <type_traits>
#ifdef RL_DEBUG_CHECKS
#include <cassert>
#define RL_ASSERT(x) assert(x)
#else
#define RL_ASSERT(x) ((void)0)
#endif

namespace rl {

constexpr unsigned FULL = 0xffffffffu;

template <typename V> struct VInf;
template <> struct VInf<int32_t> { static constexpr int32_t value = 1 << 29; };
template <> struct VInf<int64_t> { static constexpr int64_t value = (int64_t)1 << 61; };

template <typename C>
struct ProductCosts {
    C km, kr, hm, hr, pm, pr;
};

template <typename V, typename C>
struct Slot {
    V *stage, *cd, *cr, *xin, *slk;
    C *cpre;
    int16_t *nx, *pv;   // T > 63: next setup >= t / last setup < t of the base plan
    uint32_t *bm, *br;
    uint16_t *mv;
    uint64_t *lm;
    uint64_t *bar;
};

constexpr int kSlackLevels = 16;
// The slack-level skip (scan_pass) shortens long delta walks, which pays
// when the descent is latency-bound (few products per SM, GVNS tasks) and
// costs ~7% extra instructions when it is throughput-bound; the host picks
// per launch.   // lm[j] = {sR setups: slack < 2^j}, lm[16] = {slack < 0}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename V, typename C>
__host__ __device__ inline size_t slot_bytes(int T)
{
    const int NW = (T + 31) >> 5;
    size_t b = 0;
    b += align16(2 * (size_t)T * sizeof(V));     // stage
    b += align16((size_t)(T + 1) * sizeof(V));   // cd
    b += align16((size_t)(T + 1) * sizeof(V));   // cr
    b += align16((size_t)T * sizeof(V));         // xin
    b += align16((size_t)(T <= 63 ? T : 0) * sizeof(V));   // slk (register-mask path only)
    b += align16((size_t)T * sizeof(C));         // cpre
    b += 2 * align16((size_t)(T > 63 ? T + 1 : 0) * sizeof(int16_t));   // nx, pv
    b += align16(2 * (size_t)NW * sizeof(uint32_t));
    b += align16((size_t)(2 * T + 2) * sizeof(uint16_t));
    b += align16((kSlackLevels + 1) * 8);        // lm
    b += 16;                                     // mbarrier
    return b;
}

template <typename V, typename C>
__device__ inline Slot<V, C> carve(unsigned char *base, int T)
{
    const int NW = (T + 31) >> 5;
    Slot<V, C> s;
    unsigned char *p = base;
    s.stage = (V *)p; p += align16(2 * (size_t)T * sizeof(V));
    s.cd = (V *)p;    p += align16((size_t)(T + 1) * sizeof(V));
    s.cr = (V *)p;    p += align16((size_t)(T + 1) * sizeof(V));
    s.xin = (V *)p;   p += align16((size_t)T * sizeof(V));
    s.slk = (V *)p;   p += align16((size_t)(T <= 63 ? T : 0) * sizeof(V));
    s.cpre = (C *)p;  p += align16((size_t)T * sizeof(C));
    s.nx = (int16_t *)p; p += align16((size_t)(T > 63 ? T + 1 : 0) * sizeof(int16_t));
    s.pv = (int16_t *)p; p += align16((size_t)(T > 63 ? T + 1 : 0) * sizeof(int16_t));
    s.bm = (uint32_t *)p;
    s.br = s.bm + NW; p += align16(2 * (size_t)NW * sizeof(uint32_t));
    s.mv = (uint16_t *)p; p += align16((size_t)(2 * T + 2) * sizeof(uint16_t));
    s.lm = (uint64_t *)p; p += align16((kSlackLevels + 1) * 8);
    s.bar = (uint64_t *)p;
    return s;
}

// ---------------------------------------------------------------- TMA bulk

__device__ inline uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ inline void mbar_init(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ inline void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ inline void mbar_wait(uint64_t *bar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// 1-D TMA: global -> this CTA's shared memory, completion on an mbarrier.
__device__ inline void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Issue the staging copy of product k's demand/returns rows (lane 0 only).
template <typename V>
__device__ inline void stage_issue(V *stage, const V *dem, const V *ret, int64_t k, int T,
                                   uint64_t *bar)
{
    const uint32_t bytes = (uint32_t)(T * sizeof(V));
    mbar_expect_tx(bar, 2 * bytes);
    tma_load_1d(stage, dem + k * (int64_t)T, bytes, bar);
    tma_load_1d(stage + T, ret + k * (int64_t)T, bytes, bar);
}

template <typename V>
__device__ inline V vmin(V a, V b) { return a < b ? a : b; }

// ------------------------------------------------------------- bit rows

__device__ inline bool wbit(const uint32_t *w, int t) { return (w[t >> 5] >> (t & 31)) & 1u; }

// Setup rows held in shared memory words (T > 63).  Next/previous-setup
// queries read per-period tables (nx, pv) that base_pass rebuilds whenever
// the rows change, so they are one shared-memory load each.
struct MaskSmem {
    uint32_t *bm, *br;
    int16_t *nx, *pv;
    int T;
    __device__ bool m(int t) const { return wbit(bm, t); }
    __device__ bool r(int t) const { return wbit(br, t); }
    __device__ bool setup(int t) const { return wbit(bm, t) | wbit(br, t); }
    // smallest setup period >= x (T if none); needs fresh tables
    __device__ int next(int x) const
    {
        RL_ASSERT(x >= 0);
        return x >= T ? T : nx[x];
    }
    // largest setup period < x (-1 if none); needs fresh tables
    __device__ int prev(int x) const
    {
        RL_ASSERT(x <= T);
        return x <= 0 ? -1 : pv[x];
    }
    __device__ void set(int t, bool mv, bool rv, int lane)
    {
        if (lane == 0) {
            const uint32_t b = 1u << (t & 31);
            bm[t >> 5] = mv ? (bm[t >> 5] | b) : (bm[t >> 5] & ~b);
            br[t >> 5] = rv ? (br[t >> 5] | b) : (br[t >> 5] & ~b);
        }
    }
    __device__ void sync() const { __syncwarp(); }
    __device__ uint64_t R_mask() const { return 0; }   // unused (no skip for T > 63)
    // rebuild nx/pv from the bit rows (lane chunks + warp min/max scans)
    __device__ void build_tables(int lane) const
    {
        const int L = (T + 31) >> 5;
        const int lo = lane * L, hi = min(lo + L, T);
        int first = T, last = -1;
        for (int t = lo; t < hi; ++t)
            if (setup(t)) {
                first = min(first, t);
                last = t;
            }
        int sf = first, pl = last;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_down_sync(FULL, sf, off), q = __shfl_up_sync(FULL, pl, off);
            if (lane + off < 32)
                sf = min(sf, o);
            if (lane >= off)
                pl = max(pl, q);
        }
        int run = __shfl_down_sync(FULL, sf, 1);
        if (lane == 31)
            run = T;
        for (int t = hi - 1; t >= lo; --t) {
            if (setup(t))
                run = t;
            nx[t] = (int16_t)run;
        }
        run = __shfl_up_sync(FULL, pl, 1);
        if (lane == 0)
            run = -1;
        for (int t = lo; t < hi; ++t) {
            pv[t] = (int16_t)run;
            if (setup(t))
                run = t;
        }
        if (lane == 31) {
            nx[T] = (int16_t)T;
            pv[T] = (int16_t)pl;
        }
        __syncwarp();
    }
};

// The rows of a candidate move: base rows with periods a <= b rewritten.
struct PatchedSmem {
    MaskSmem base;
    int a, b;
    bool ma, ra, mb, rb;
    __device__ bool m(int t) const { return t == a ? ma : t == b ? mb : base.m(t); }
    __device__ bool r(int t) const { return t == a ? ra : t == b ? rb : base.r(t); }
    __device__ int next(int x) const
    {
        int t = base.next(x);
        while (t < base.T && (t == a || t == b) && !(m(t) | r(t)))
            t = base.next(t + 1);
        if (x <= a && a < t && (ma | ra))
            t = a;
        else if (x <= b && b < t && (mb | rb))
            t = b;
        return t;
    }
};

// Setup rows in two warp-uniform registers (T <= 63: bit T is a sentinel
// "setup" so a next-setup query is one bit scan with no empty case).
struct MaskReg {
    uint64_t M, R;
    int T;
    __device__ bool m(int t) const { return (M >> t) & 1; }
    __device__ bool r(int t) const { return (R >> t) & 1; }
    // smallest set bit >= x of S (which carries the sentinel bit T), x <= T
    __device__ static int next_of(uint64_t S, int x, int)
    {
        return x + __ffsll((long long)(S >> x)) - 1;
    }
    __device__ uint64_t sentinel() const { return 1ull << T; }
    __device__ int next(int x) const { return next_of(M | R | sentinel(), x, T); }
    __device__ uint64_t R_mask() const { return R; }
    __device__ int prev(int x) const
    {
        const uint64_t w = (M | R) & ((1ull << x) - 1);   // x <= T <= 63
        return w ? 63 - __clzll((long long)w) : -1;
    }
    __device__ void set(int t, bool mv, bool rv, int)
    {
        const uint64_t b = 1ull << t;
        M = mv ? (M | b) : (M & ~b);
        R = rv ? (R | b) : (R & ~b);
    }
    __device__ void sync() const {}
};

struct PatchedReg {
    uint64_t M, R, SR;   // SR = bit-reversed (M | R | sentinel)
    PatchedReg() = default;
    __device__ PatchedReg(const MaskReg &base, int a, int b, bool ma, bool ra, bool mb, bool rb)
    {
        const uint64_t ba = 1ull << a, bb = 1ull << b, clr = ~(ba | bb);
        M = (base.M & clr) | (ma ? ba : 0) | (mb ? bb : 0);
        R = (base.R & clr) | (ra ? ba : 0) | (rb ? bb : 0);
        SR = __brevll(M | R | base.sentinel());
    }
    __device__ bool m(int t) const { return (M >> t) & 1; }
    __device__ bool r(int t) const { return (R >> t) & 1; }
    // period t is bit 63-t of SR: shifting left by x drops periods < x and
    // the leading one is the first setup >= x (count leading zeros)
    __device__ int next(int x) const { return x + __clzll((long long)(SR << x)); }
};

template <typename Mask> struct PatchOf;
template <> struct PatchOf<MaskSmem> {
    using type = PatchedSmem;
    __device__ static PatchedSmem make(const MaskSmem &b, int a, int bb, bool ma, bool ra,
                                       bool mb, bool rb)
    {
        return PatchedSmem{b, a, bb, ma, ra, mb, rb};
    }
};
template <> struct PatchOf<MaskReg> {
    using type = PatchedReg;
    __device__ static PatchedReg make(const MaskReg &b, int a, int bb, bool ma, bool ra, bool mb,
                                      bool rb)
    {
        return PatchedReg(b, a, bb, ma, ra, mb, rb);
    }
};

// Plan row bytes (bool K x T, plan.py:22-29) -> bit rows.
template <typename V, typename C>
__device__ inline MaskSmem load_rows(const Slot<V, C> &s, MaskSmem, const uint8_t *sm,
                                     const uint8_t *sr, int64_t k, int T, int lane)
{
    const uint8_t *a = sm + k * (int64_t)T, *b = sr + k * (int64_t)T;
    for (int base = 0; base < T; base += 32) {
        const int t = base + lane;
        const uint32_t wm = __ballot_sync(FULL, t < T && a[t]);
        const uint32_t wr = __ballot_sync(FULL, t < T && b[t]);
        if (lane == 0) {
            s.bm[base >> 5] = wm;
            s.br[base >> 5] = wr;
        }
    }
    __syncwarp();
    return MaskSmem{s.bm, s.br, s.nx, s.pv, T};
}

template <typename V, typename C>
__device__ inline MaskReg load_rows(const Slot<V, C> &, MaskReg, const uint8_t *sm,
                                    const uint8_t *sr, int64_t k, int T, int lane)
{
    const uint8_t *a = sm + k * (int64_t)T, *b = sr + k * (int64_t)T;
    uint64_t M = 0, R = 0;
    for (int base = 0; base < T; base += 32) {
        const int t = base + lane;
        M |= (uint64_t)__ballot_sync(FULL, t < T && a[t]) << base;
        R |= (uint64_t)__ballot_sync(FULL, t < T && b[t]) << base;
    }
    return MaskReg{M, R, T};
}

template <typename Mask>
__device__ inline void store_rows(const Mask &mk, uint8_t *sm, uint8_t *sr, int64_t k, int T,
                                  int lane)
{
    uint8_t *a = sm + k * (int64_t)T, *b = sr + k * (int64_t)T;
    for (int t = lane; t < T; t += 32) {
        a[t] = mk.m(t);
        b[t] = mk.r(t);
    }
}

// Cost of one segment [u, v) entered with cumulative remanufacturing X.
// Follows _kernels.py:66-95 (seg :70-72, avail :73, x_r :74-76, x_m and
// infeasibility :77-82, setup :83-86, unit :87, holding :88-95 summed).
template <typename V, typename C>
__device__ inline bool seg_cost(const V *cd, const V *cr, int T, int u, int v, bool m, bool r,
                                V X, const ProductCosts<C> &pc, C &c, V &xr)
{
    RL_ASSERT(0 <= u && u < v && v <= T);
    const V seg = cd[v] - cd[u];
    const V avail = cr[u + 1] - X;
    xr = r ? vmin(seg, avail) : V(0);
    const V xm = seg - xr;
    // computed unconditionally (no branch): callers discard c when infeasible
    c = (xr > 0 ? pc.kr : C(0)) + (xm > 0 ? pc.km : C(0)) + pc.pr * C(xr) + pc.pm * C(xm) +
        C(T - u) * (pc.hm * C(seg) - pc.hr * C(xr));
    return !(xm > 0 && !m);
}

// ------------------------------------------------------------ staging

// Prefix sums of the staged rows into cd/cr; returns K0 (warp-uniform).
template <typename V, typename C>
__device__ inline C build_prefix(const Slot<V, C> &s, int T, const ProductCosts<C> &pc, int lane)
{
    V carry_d = 0, carry_r = 0;
    C sum_cd = 0, sum_cr = 0;   // sum_t CD[t], sum_t CR[t] (inclusive prefixes)
    if (lane == 0) {
        s.cd[0] = 0;
        s.cr[0] = 0;
    }
    for (int base = 0; base < T; base += 32) {
        const int t = base + lane;
        V d = t < T ? s.stage[t] : V(0);
        V r = t < T ? s.stage[T + t] : V(0);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            V od = __shfl_up_sync(FULL, d, off), orr = __shfl_up_sync(FULL, r, off);
            if (lane >= off) {
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
        carry_d = __shfl_sync(FULL, d, 31);
        carry_r = __shfl_sync(FULL, r, 31);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        sum_cd += __shfl_xor_sync(FULL, sum_cd, off);
        sum_cr += __shfl_xor_sync(FULL, sum_cr, off);
    }
    __syncwarp();
    return pc.hr * sum_cr - pc.hm * sum_cd;
}

// Plain coalesced staging (fallback when TMA alignment does not hold).
template <typename V, typename C>
__device__ inline void stage_plain(const Slot<V, C> &s, const V *dem, const V *ret, int64_t k,
                                   int T, int lane)
{
    const V *d = dem + k * (int64_t)T, *r = ret + k * (int64_t)T;
    for (int t = lane; t < T; t += 32) {
        s.stage[t] = d[t];
        s.stage[T + t] = r[t];
    }
    __syncwarp();
}

// --------------------------------------------------------- base pass

// Evaluate the current plan: fills xin/cpre at every setup period, returns
// feasibility and S = sum of segment costs (warp-uniform).  Lane l owns the
// periods [l*L, l*L+L).  Step 1 composes the (min,+) maps of its setups,
// a warp scan gives every lane its entering X, step 2 walks the segments.
template <typename V, typename C, typename Mask, bool Skip = false>
__device__ inline bool base_pass(const Slot<V, C> &s, const Mask &mk, int T,
                                 const ProductCosts<C> &pc, int lane, C &S)
{
    if constexpr (std::is_same<Mask, MaskSmem>::value)
        mk.build_tables(lane);
    const int L = (T + 31) >> 5;
    const int lo = lane * L, hi = min(lo + L, T);
    const V INF = VInf<V>::value;
    V A = 0, B = INF;
    for (int u = lo; u < hi; ++u) {
        if (!mk.r(u))
            continue;   // only remanufacturing setups move X
        const int v = mk.next(u + 1);
        const V seg = s.cd[v] - s.cd[u];
        A += seg;
        B = vmin<V>(B + seg, s.cr[u + 1]);
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        V a2 = __shfl_up_sync(FULL, A, off), b2 = __shfl_up_sync(FULL, B, off);
        if (lane >= off) {
            B = vmin<V>(b2 + A, B);
            A = a2 + A;
        }
    }
    V pa = __shfl_up_sync(FULL, A, 1), pb = __shfl_up_sync(FULL, B, 1);
    V X = lane == 0 ? V(0) : vmin<V>(pa, pb);

    constexpr bool kSkip = Skip && std::is_same<Mask, MaskReg>::value;
    C local = 0;
    bool ok = true;
    for (int u = lo; u < hi; ++u) {
        const bool m = mk.m(u), r = mk.r(u);
        if (kSkip)
            s.slk[u] = INF;
        if (!(m | r))
            continue;
        const int v = mk.next(u + 1);
        s.xin[u] = X;
        s.cpre[u] = local;
        if (kSkip && r)
            s.slk[u] = s.cr[u + 1] - X - (s.cd[v] - s.cd[u]);
        C c;
        V xr;
        ok &= seg_cost<V, C>(s.cd, s.cr, T, u, v, m, r, X, pc, c, xr);
        local += c;
        X += xr;
    }
    C incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        C o = __shfl_up_sync(FULL, incl, off);
        if (lane >= off)
            incl += o;
    }
    const C excl = incl - local;
    if (excl != C(0))
        for (int u = lo; u < hi; ++u)
            if (mk.m(u) | mk.r(u))
                s.cpre[u] += excl;
    S = __shfl_sync(FULL, incl, 31);
    const int f = mk.next(0);
    ok = ok && s.cd[f] == 0;   // demand before the first setup (_kernels.py:58-60)
    const bool feas = __all_sync(FULL, ok);
    if (kSkip) {
        // slack-level masks for the delta-walk skip (scan_pass): lane l owns
        // periods l and l + 32, so each ballot yields one 32-bit half
        __syncwarp();
        const V s0 = lane < T ? s.slk[lane] : INF;
        const V s1 = lane + 32 < T ? s.slk[lane + 32] : INF;
        uint64_t mine = 0;
#pragma unroll
        for (int j = 0; j <= kSlackLevels; ++j) {
            const V lim = j < kSlackLevels ? (V(1) << j) : V(0);
            const uint64_t mk2 = (uint64_t)__ballot_sync(FULL, s0 < lim) |
                                 ((uint64_t)__ballot_sync(FULL, s1 < lim) << 32);
            if (lane == j)
                mine = mk2;
        }
        if (lane <= kSlackLevels)
            s.lm[lane] = mine;
    }
    __syncwarp();
    return feas;
}

// ------------------------------------------------------- move scoring

// A move in reference form (list_moves, _kernels.py:188-258): period p0
// (and p1 >= 0 for shifts) with the new bits of both rows there.
struct MoveDesc {
    int p0, p1;
    bool m0, r0, m1, r1;
};

// Canonical move slots of neighborhood nbh.  N1/N2/N4: slot t.  N3: slot
// row*2T + 2t + dir (row 0 = manufacturing, dir 0 = left).  The slot number
// is monotone in the reference's enumeration index, so it is the tie key.
template <typename Mask>
__device__ inline bool slot_valid(const Mask &mk, int nbh, int slot, int T)
{
    if (nbh == 1 || nbh == 2)
        return slot < T;
    if (nbh == 4)
        return slot < T && mk.m(slot) != mk.r(slot);
    if (slot >= 4 * T)
        return false;
    const bool rrow = slot >= 2 * T;
    const int t = (slot - (rrow ? 2 * T : 0)) >> 1;
    auto row = [&](int q) { return rrow ? mk.r(q) : mk.m(q); };
    if (!row(t))
        return false;
    return (slot & 1) ? (t + 1 < T && !row(t + 1)) : (t > 0 && !row(t - 1));
}

template <typename Mask>
__device__ inline MoveDesc slot_move(const Mask &mk, int nbh, int slot, int T)
{
    MoveDesc d;
    if (nbh != 3) {
        const int t = slot;
        const bool m = mk.m(t), r = mk.r(t);
        d.p0 = t;
        d.p1 = -1;
        d.m0 = nbh == 1 ? !m : nbh == 2 ? m : r;
        d.r0 = nbh == 1 ? r : nbh == 2 ? !r : m;
        d.m1 = d.r1 = false;
        return d;
    }
    const bool rrow = slot >= 2 * T;
    const int t = (slot - (rrow ? 2 * T : 0)) >> 1;
    const int t1 = (slot & 1) ? t + 1 : t - 1;
    d.p0 = t;
    d.p1 = t1;
    d.m0 = rrow ? mk.m(t) : false;
    d.r0 = rrow ? false : mk.r(t);
    d.m1 = rrow ? mk.m(t1) : true;
    d.r1 = rrow ? true : mk.r(t1);
    return d;
}

struct PassResult {
    bool improved;
    int slot;     // winning canonical slot
    int n_moves;  // candidates scored (list_moves count)
};

// Per-lane state of one delta walk.  A move rewrites periods a <= b; its
// cost is the base plan's prefix up to the last setup before a (cpre, xin),
// the re-walked segments, and -- once past b the walk's X equals the base
// plan's X at a setup -- the base plan's suffix.
template <typename V, typename C, typename Mask>
struct Walk {
    typename PatchOf<Mask>::type nw;
    int u, b, slot;
    V X;
    C acc;
};

template <typename V, typename C, typename Mask>
__device__ inline typename PatchOf<Mask>::type patch_of(const Mask &mk, const MoveDesc &d, int &a,
                                                        int &b)
{
    if (d.p1 < 0) {
        a = b = d.p0;
        return PatchOf<Mask>::make(mk, d.p0, d.p0, d.m0, d.r0, d.m0, d.r0);
    }
    if (d.p1 < d.p0) {
        a = d.p1;
        b = d.p0;
        return PatchOf<Mask>::make(mk, d.p1, d.p0, d.m1, d.r1, d.m0, d.r0);
    }
    a = d.p0;
    b = d.p1;
    return PatchOf<Mask>::make(mk, d.p0, d.p1, d.m0, d.r0, d.m1, d.r1);
}

// One neighborhood pass over the warp's product (scan_products body,
// _kernels.py:280-325): enumerate, score every move, keep the strict
// minimum with the earliest slot on ties.  best_out = winning S.
//
// Moves are scored by delta walks of data-dependent length, so the lanes
// run a warp-level work queue over walk *steps*: a lane whose walk ends
// takes the next unscored move, and every loop iteration advances every
// busy lane by one segment.  Each lane still scores its moves in
// increasing slot order, so a strict '<' keeps the earliest on ties.
// Move list of neighborhood nbh for the warp's product: N1/N2 are dense
// (slot = index, returns T), N3/N4 are compacted into s.mv.
template <typename V, typename C, typename Mask>
__device__ inline int enumerate_moves(const Slot<V, C> &s, const Mask &mk, int nbh, int T,
                                      int lane)
{
    if (nbh <= 2)
        return T;
    const int nslots = nbh == 3 ? 4 * T : T;
    int n = 0;
    for (int base = 0; base < nslots; base += 32) {
        const int slot = base + lane;
        const bool ok = slot < nslots && slot_valid(mk, nbh, slot, T);
        const uint32_t bal = __ballot_sync(FULL, ok);
        if (ok)
            s.mv[n + __popc(bal & ((1u << lane) - 1))] = (uint16_t)slot;
        n += __popc(bal);
    }
    __syncwarp();
    return n;
}

// lexicographic (cost, slot) minimum over the warp
template <typename C>
__device__ inline void warp_argmin(C &best, int &key)
{
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const C ob = __shfl_xor_sync(FULL, best, off);
        const int ok = __shfl_xor_sync(FULL, key, off);
        if (ob < best || (ob == best && ok < key)) {
            best = ob;
            key = ok;
        }
    }
}

// Score the moves i = wi, wi + nw, wi + 2 nw, ... (< n) of the current list
// on this warp (nw warps share a product in the CTA variant); per-lane
// results in best/key (initialise best = S, key = INT_MAX).
template <typename V, typename C, typename Mask, bool Skip = false>
__device__ inline void walk_moves(const Slot<V, C> &s, const Mask &mk, int T,
                                  const ProductCosts<C> &pc, C S, int nbh, int n, int lane,
                                  int wi, int nw, C &best, int &key)
{
    const bool dense = nbh <= 2;
    const unsigned lt = (1u << lane) - 1;
    Walk<V, C, Mask> w;
    int idx = lane, next = 32;
    int gi = idx * nw + wi;
    bool pend = gi < n, act = false;
    while (__any_sync(FULL, pend | act)) {
        if (pend) {
            pend = false;
            RL_ASSERT(gi < n && gi < 4 * T);
            w.slot = dense ? gi : s.mv[gi];
            const MoveDesc d = slot_move(mk, nbh, w.slot, T);
            int a;
            w.nw = patch_of<V, C, Mask>(mk, d, a, w.b);
            const int p = mk.prev(a);
            const int pp = p < 0 ? 0 : p;
            const int u0 = p < 0 ? w.nw.next(0) : p;
            w.u = u0;
            w.acc = p < 0 ? C(0) : s.cpre[pp];
            w.X = p < 0 ? V(0) : s.xin[pp];
            // no setup before the move: demand ahead of the first setup is infeasible
            act = p >= 0 || s.cd[u0] == 0;
            if (act && u0 >= T) {   // no setup at all and no demand: cost 0
                act = false;
                if (w.acc < best) {
                    best = w.acc;
                    key = w.slot;
                }
            }
        }
        if (act) {
            int u = w.u;
            bool done = false;
            if (Skip && std::is_same<Mask, MaskReg>::value) {
                // Past the move (u > b) the rows equal the base plan's and
                // only the entering X differs (delta != 0).  A segment then
                // costs what it costs in the base plan unless it starts at an
                // sR setup whose slack < max(delta, 0) (its min(seg, avail)
                // changes).  Jump to the next setup in the slack-level mask
                // that bounds that set (false positives are merely evaluated
                // exactly) and add the base cost of the skipped segments.
                const bool ph2 = u > w.b;
                const V delta = w.X - s.xin[u];
                const int j = delta <= 1 ? 0 : 64 - __clzll((long long)(uint64_t)(delta - 1));
                const uint64_t cand = (delta < 0 ? s.lm[kSlackLevels]
                                       : j < kSlackLevels ? s.lm[j] : mk.R_mask()) | (1ull << T);
                const int q = ph2 ? MaskReg::next_of(cand, u, T) : u;
                const int qq = q < T ? q : u;
                const C skipped = (q < T ? s.cpre[qq] : S) - s.cpre[u];
                if (ph2) {
                    w.acc += skipped;
                    w.X = s.xin[qq] + delta;
                }
                done = q >= T;
                u = qq;
            }
            // one segment of the walk, branch-free (every busy lane issues the
            // same instructions): cost, resync test, finish, argmin update
            const int v = w.nw.next(u + 1);
            C c;
            V xr;
            const bool ok = seg_cost<V, C>(s.cd, s.cr, T, u, v, w.nw.m(u), w.nw.r(u), w.X, pc, c,
                                           xr);
            const int vv = v < T ? v : T - 1;
            const V xv = s.xin[vv];
            const C cv = s.cpre[vv];
            const C acc = done ? w.acc : w.acc + c;
            const V X = w.X + xr;
            const bool sync = !done && v < T && v > w.b && X == xv;
            const bool fin = done || v >= T || sync;
            const C total = sync ? acc + (S - cv) : acc;
            const bool take = (done || ok) && fin && total < best;
            best = take ? total : best;
            key = take ? w.slot : key;
            act = !done && ok && !fin;
            w.acc = acc;
            w.X = X;
            w.u = v;
        }
        const bool idle = !(pend | act);
        const unsigned m = __ballot_sync(FULL, idle);
        if (idle) {
            idx = next + __popc(m & lt);
            gi = idx * nw + wi;
            pend = gi < n;
        }
        next += __popc(m);
    }
}

template <typename V, typename C, typename Mask, bool Skip = false>
__device__ inline PassResult scan_pass(const Slot<V, C> &s, const Mask &mk, int T,
                                       const ProductCosts<C> &pc, C S, int nbh, int lane,
                                       C &best_out)
{
    const int n = enumerate_moves(s, mk, nbh, T, lane);
    C best = S;
    int key = 0x7fffffff;
    walk_moves<V, C, Mask, Skip>(s, mk, T, pc, S, nbh, n, lane, 0, 1, best, key);
    warp_argmin(best, key);
    PassResult res;
    res.improved = key != 0x7fffffff;
    res.slot = key;
    res.n_moves = n;
    best_out = best;
    return res;
}

// Write the winning move into the rows (apply_scan, _kernels.py:335-342).
template <typename Mask>
__device__ inline void apply_slot(Mask &mk, int nbh, int slot, int T, int lane)
{
    const MoveDesc d = slot_move(mk, nbh, slot, T);
    mk.sync();
    mk.set(d.p0, d.m0, d.r0, lane);
    if (d.p1 >= 0)
        mk.set(d.p1, d.m1, d.r1, lane);
    mk.sync();
}

// Move count of one neighborhood at the current plan (used to credit the
// lockstep passes a product sits out after reaching its fixpoint).
template <typename Mask>
__device__ inline int move_count(const Mask &mk, int nbh, int T, int lane)
{
    if (nbh <= 2)
        return T;
    const int nslots = nbh == 3 ? 4 * T : T;
    int n = 0;
    for (int base = 0; base < nslots; base += 32) {
        const int slot = base + lane;
        n += __popc(__ballot_sync(FULL, slot < nslots && slot_valid(mk, nbh, slot, T)));
    }
    return n;
}

}  // namespace rl
