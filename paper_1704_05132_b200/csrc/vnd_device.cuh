// vnd_device.cuh -- per-product device machinery of the VND hot path.
//
// One warp owns one product at a time (north_star: "one warp or CTA per
// product").  The product's T-period slice lives in shared memory:
//
//   stage[2T]   demand row, returns row (V), landed by a 1-D TMA bulk copy
//               into the xc area (consumed by the prefix sums before xc is built)
//   dr[T+1]     {cd[t], cr[t+1]}: cd[t] = sum_{i<t} D[i], cr[t+1] = sum_{i<=t} R[i]
//               (V pairs: one 8/16-byte load gives a segment's demand prefix
//               and the returns available at its setup)
//   xc[T]       {cpre[u], xin[u]} at setups u: sum of segment costs before u
//               (C) and cumulative remanufactured quantity entering u (V)
//   slk[T]      remanufacturing slack CR[u] - xin[u] - seg(u) at sR setups (V)
//   lm[18]      T <= 63: masks of sR setups with slack < 2^j (j < 16), all sR, slack < 0
//   bm[NW],br[NW],bs[NW]  setup bit rows and their union (uint32 words; T > 63)
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

#ifdef RL_WALK_STATS
// Diagnostic build only (tools/walk_stats.py): [0] passes, [1] loop
// iterations, [2] moves, [3] walk steps, [4] sum of per-pass longest walk,
// [5] sum of per-pass busiest lane's steps, [8..71] walk-length histogram,
// [72..135] per-pass iterations histogram (both clamped to 63),
// [136 + nbh] passes, [144 + nbh] improving passes, [152 + nbh] moves of
// neighborhood nbh (vnd_product).
__device__ unsigned long long g_walk_stats[160];
#endif

template <typename V> struct VInf;
template <> struct VInf<int32_t> { static constexpr int32_t value = 1 << 29; };
template <> struct VInf<int64_t> { static constexpr int64_t value = (int64_t)1 << 61; };

// a0 = p_M + T h_M, b0 = p_R - p_M - T h_R: a segment [u, v) costs
// seg (a0 - u h_M) + x_R (b0 + u h_R) plus its setup charges (seg_cost)
template <typename C>
struct ProductCosts {
    C km, kr, hm, hr, pm, pr, a0, b0;
    // 1 and -1 the compiler cannot see through (derived from the horizon):
    // x * one + y issues as an IMAD on the FMA pipe instead of an IADD3 on
    // the ALU pipe, which bounds the int32 walk (ncu: ALU 83%, FMA 21%)
    C one, mone;
};

template <typename V>
struct alignas(2 * sizeof(V)) DR {
    V d, r;   // cd[t], cr[t+1]
};

template <typename V, typename C>
struct alignas(2 * sizeof(C)) XC {
    C c;      // cpre[u]
    V x;      // xin[u]
};

// {cpre, xin} per period: one interleaved array when both have the same
// width (one 8/16-byte load per query), two arrays for int32 X with int64
// costs (12 bytes per period instead of a padded 16: the long-horizon
// kernel's shared memory per warp bounds its occupancy).
template <typename V, typename C, bool Split = (sizeof(V) != sizeof(C))>
struct XCStore {
    XC<V, C> *p;
    __host__ __device__ static size_t bytes(int T) { return (size_t)T * sizeof(XC<V, C>); }
    __device__ void carve(unsigned char *b, int) { p = (XC<V, C> *)b; }
    __device__ XC<V, C> operator[](int i) const { return p[i]; }
    __device__ void set(int i, V x, C c) const
    {
        p[i].x = x;
        p[i].c = c;
    }
    __device__ void add_c(int i, C d) const { p[i].c += d; }
    __device__ void *base() const { return p; }
};
template <typename V, typename C>
struct XCStore<V, C, true> {
    C *c;
    V *x;
    __host__ __device__ static size_t bytes(int T)
    {
        return ((size_t)T * sizeof(C) + 15) / 16 * 16 + (size_t)T * sizeof(V);
    }
    __device__ void carve(unsigned char *b, int T)
    {
        c = (C *)b;
        x = (V *)(b + ((size_t)T * sizeof(C) + 15) / 16 * 16);
    }
    __device__ XC<V, C> operator[](int i) const
    {
        XC<V, C> e;
        e.c = c[i];
        e.x = x[i];
        return e;
    }
    __device__ void set(int i, V xv, C cv) const
    {
        x[i] = xv;
        c[i] = cv;
    }
    __device__ void add_c(int i, C d) const { c[i] += d; }
    __device__ void *base() const { return c; }
};

// {cd[t], cr[t+1]} per period.  SB = stored bytes per value: sizeof(V)
// stores DR<V> pairs; SB = 2 (int32 values with every product's sum D and sum
// R below 2^16, proved at upload) stores the two 16-bit halves of one word
// (the long-horizon kernel's occupancy is bounded by shared memory).
template <typename V, int SB>
struct DRStore {
    DR<V> *p;
    __host__ __device__ static size_t bytes(int n) { return (size_t)n * sizeof(DR<V>); }
    __device__ void carve(unsigned char *b) { p = (DR<V> *)b; }
    __device__ DR<V> operator[](int i) const { return p[i]; }
    __device__ void set_d(int i, V v) const { p[i].d = v; }
    __device__ void set_r(int i, V v) const { p[i].r = v; }
};
template <typename V>
struct DRStore<V, 2> {
    uint32_t *p;
    __host__ __device__ static size_t bytes(int n) { return (size_t)n * 4; }
    __device__ void carve(unsigned char *b) { p = (uint32_t *)b; }
    __device__ DR<V> operator[](int i) const
    {
        // two zero-extending 16-bit loads: no unpack on the ALU pipe
        // (measured C4 -2.5% against one 32-bit load and two ALU ops)
        const uint16_t *q = reinterpret_cast<const uint16_t *>(p + i);
        return DR<V>{V(q[0]), V(q[1])};
    }
    __device__ void set_d(int i, V v) const
    {
        RL_ASSERT(v >= 0 && v < 65536);   // the upload's 16-bit proof
        ((uint16_t *)p)[2 * i] = (uint16_t)v;
    }
    __device__ void set_r(int i, V v) const
    {
        RL_ASSERT(v >= 0 && v < 65536);
        ((uint16_t *)p)[2 * i + 1] = (uint16_t)v;
    }
};

// {cpre, xin} with a 16-bit xin (SB = 2; xin <= sum R < 2^16)
template <typename V, typename C>
struct XCStore16 {
    C *c;
    uint16_t *x;
    __host__ __device__ static size_t bytes(int T)
    {
        return ((size_t)T * sizeof(C) + 15) / 16 * 16 + (size_t)T * 2;
    }
    __device__ void carve(unsigned char *b, int T)
    {
        c = (C *)b;
        x = (uint16_t *)(b + ((size_t)T * sizeof(C) + 15) / 16 * 16);
    }
    __device__ XC<V, C> operator[](int i) const
    {
        XC<V, C> e;
        e.c = c[i];
        e.x = V(x[i]);
        return e;
    }
    __device__ void set(int i, V xv, C cv) const
    {
        RL_ASSERT(xv >= 0 && xv < 65536);
        x[i] = (uint16_t)xv;
        c[i] = cv;
    }
    __device__ void add_c(int i, C d) const { c[i] += d; }
    __device__ void *base() const { return c; }
};
template <typename V, typename C, int SB> struct XCStoreOf { using type = XCStore<V, C>; };
template <typename V, typename C> struct XCStoreOf<V, C, 2> { using type = XCStore16<V, C>; };

template <typename V, typename C, int SB = (int)sizeof(V)>
struct Slot {
    V *stage, *slk;
    DRStore<V, SB> dr;
    typename XCStoreOf<V, C, SB>::type xc;
    uint16_t *nx;       // T > 63: next setup >= t of the base plan and its kind
    uint32_t *bm, *br, *bs;
    uint16_t *mv;
    uint64_t *lm;
    uint64_t *bar;
};

#ifndef RL_WORD_ENUM_MIN_T
#define RL_WORD_ENUM_MIN_T 128
#endif
// Walk steps per queue iteration (between the ballot / refill control):
// register rows 2 (measured C3 17.6 -> 16.7 ms, T=63 12.2 -> 11.6, C2 0.59 ->
// 0.57, GVNS +3-5%; 3: C2 and GVNS slower, 4: +3-9%), shared-memory rows 2
// (after the incremental re-base: C4 114.5 -> 112.6-114.5 ms, T=200 -2%,
// K=100 T=520 (CTA per product) 12.0 -> 10.5 ms; within noise at C4 with
// the full base pass; 4: +11%).  A lane whose walk ends in the first step
// issues the second one discarded, like an idle lane.
#ifndef RL_WALK_STEPS_REG
#define RL_WALK_STEPS_REG 2
#endif
#ifndef RL_WALK_STEPS_SMEM
#define RL_WALK_STEPS_SMEM 2
#endif
#ifndef RL_DENSE_PREV_TABLE
#define RL_DENSE_PREV_TABLE 1
#endif
#ifndef RL_REFILL_MIN_SMEM   // shared-memory rows, two walk steps per iteration: measured
#define RL_REFILL_MIN_SMEM 12   // C4 8 / 12 / 16 / 24: 109.8-111.3 / 109.5-110.4 / 110.6-111.9 / 120 ms
#endif
#ifndef RL_REFILL_MIN
#define RL_REFILL_MIN 16   // measured: 1 -> 20.1, 8 -> 19.1, 16 -> 18.8, 24 -> 18.9 ms at C3
#endif
constexpr int kSlackLevels = 16;   // lm[j] = slack < 2^j (j < 16), lm[16] = all sR, lm[17] = slack < 0
// The slack-level skip (scan_pass) shortens long delta walks, which pays
// when the descent is latency-bound (few products per SM, GVNS tasks) and
// costs ~7% extra instructions when it is throughput-bound; the host picks
// per launch.

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename V, typename C, int SB = (int)sizeof(V)>
__host__ __device__ inline size_t slot_bytes(int T)
{
    const int NW = (T + 31) >> 5;
    size_t b = 0;
    b += align16(DRStore<V, SB>::bytes(T + 1));                      // dr
    b += align16(XCStoreOf<V, C, SB>::type::bytes(T + 1));          // xc (+ the end entry xc[T])
    b += align16((size_t)(T <= 63 ? T : 0) * sizeof(V));   // slk (register-mask path only)
    b += align16((size_t)(T > 63 ? T + 1 : 0) * sizeof(int16_t));   // nx
    b += align16(3 * (size_t)NW * sizeof(uint32_t));
    b += align16((size_t)(2 * T + 2) * sizeof(uint16_t));
    b += align16((T <= 63 ? kSlackLevels + 2 : 0) * 8);   // lm (register-mask skip only)
    b += 16;                                     // mbarrier
    return b;
}

template <typename V, typename C, int SB = (int)sizeof(V)>
__device__ inline Slot<V, C, SB> carve(unsigned char *base, int T)
{
    const int NW = (T + 31) >> 5;
    Slot<V, C, SB> s;
    unsigned char *p = base;
    s.dr.carve(p); p += align16(DRStore<V, SB>::bytes(T + 1));
    s.xc.carve(p, T + 1); p += align16(XCStoreOf<V, C, SB>::type::bytes(T + 1));
    // the staged demand/returns rows (2T x V <= the xc area) are consumed by
    // build_prefix before base_pass first writes xc
    s.stage = (V *)s.xc.base();
    static_assert(SB == 2 ? sizeof(C) + 2 >= 2 * sizeof(V) : sizeof(C) + sizeof(V) >= 2 * sizeof(V),
                  "stage must fit in xc");
    s.slk = (V *)p;   p += align16((size_t)(T <= 63 ? T : 0) * sizeof(V));
    s.nx = (uint16_t *)p; p += align16((size_t)(T > 63 ? T + 1 : 0) * sizeof(uint16_t));
    s.bm = (uint32_t *)p;
    s.br = s.bm + NW;
    s.bs = s.br + NW; p += align16(3 * (size_t)NW * sizeof(uint32_t));
    s.mv = (uint16_t *)p; p += align16((size_t)(2 * T + 2) * sizeof(uint16_t));
    s.lm = (uint64_t *)p; p += align16((T <= 63 ? kSlackLevels + 2 : 0) * 8);
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

// smallest j with 2^j >= x (0 for x <= 1)
__device__ inline int ceil_log2(int32_t x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }
__device__ inline int ceil_log2(int64_t x)
{
    return x <= 1 ? 0 : 64 - __clzll((long long)(x - 1));
}

// ------------------------------------------------------------- bit rows

__device__ inline bool wbit(const uint32_t *w, int t) { return (w[t >> 5] >> (t & 31)) & 1u; }

// Setup rows held in shared memory words (T > 63).  Next-setup queries (one
// per walk step) read a per-period table that base_pass rebuilds whenever
// the rows change: nx[t] = first setup >= t (bits 0-13) and its type (bits
// 14-15: 1 = manufacturing, 2 = remanufacturing), so a walk step learns the
// next segment's start and setup kind from one 16-bit load.
// Previous-setup queries (one per move) scan the words.
constexpr int kTypeShift = 14;
constexpr int kPeriodMask = (1 << kTypeShift) - 1;   // T <= 16000 < 2^14

struct MaskSmem {
    uint32_t *bm, *br, *bs;   // bs = bm | br (one load per setup query)
    uint16_t *nx;
    int T;
    __device__ bool m(int t) const { return wbit(bm, t); }
    __device__ bool r(int t) const { return wbit(br, t); }
    __device__ bool setup(int t) const { return wbit(bs, t); }
    // smallest setup period >= x (T if none); needs fresh tables
    __device__ int next(int x) const
    {
        RL_ASSERT(x >= 0);
        return x >= T ? T : (nx[x] & kPeriodMask);
    }
    // kind (m | r << 1) of setup period t (t must be a setup); fresh tables
    __device__ int setup_type(int t) const { return nx[t] >> kTypeShift; }
    // largest setup period < x (-1 if none)
    __device__ int prev(int x) const
    {
        RL_ASSERT(x <= T);
        if (x <= 0)
            return -1;
        int w = (x - 1) >> 5;
        uint32_t bits = bs[w] & (0xffffffffu >> (31 - ((x - 1) & 31)));
        while (!bits && w > 0) {
            --w;
            bits = bs[w];
        }
        return bits ? (w << 5) + 31 - __clz(bits) : -1;
    }
    __device__ void set(int t, bool mv, bool rv, int lane)
    {
        if (lane == 0) {
            const uint32_t b = 1u << (t & 31);
            const uint32_t wm = mv ? (bm[t >> 5] | b) : (bm[t >> 5] & ~b);
            const uint32_t wr = rv ? (br[t >> 5] | b) : (br[t >> 5] & ~b);
            bm[t >> 5] = wm;
            br[t >> 5] = wr;
            bs[t >> 5] = wm | wr;
        }
    }
    __device__ void sync() const { __syncwarp(); }
    __device__ uint64_t R_mask() const { return 0; }   // unused (no skip for T > 63)
    // rebuild nx from the bit rows (lane chunks + a warp min scan)
    __device__ void build_tables(int lane) const
    {
        const int L = (T + 31) >> 5;
        const int lo = lane * L, hi = min(lo + L, T);
        // first setup in [lo, hi): scan the chunk's words
        int first = T;
        if (lo < hi) {
            int w = lo >> 5;
            const int wl = (hi - 1) >> 5;
            uint32_t bits = bs[w] & (0xffffffffu << (lo & 31));
            while (!bits && w < wl) {
                ++w;
                bits = bs[w];
            }
            const int f = bits ? (w << 5) + __ffs(bits) - 1 : T;
            first = f < hi ? f : T;
        }
        int sf = first;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_down_sync(FULL, sf, off);
            if (lane + off < 32)
                sf = min(sf, o);
        }
        int run = __shfl_down_sync(FULL, sf, 1);
        if (lane == 31)
            run = T;
        // the first setup >= hi (a lane's successor chunk) and its kind
        int ty = run < T ? (int)m(run) | (int)r(run) << 1 : 0;
        // descending over the chunk, one pair of word loads per 32 periods
        for (int t = hi - 1; t >= lo;) {
            const int w = t >> 5;
            const uint32_t mw = bm[w], rw = br[w];
            const int tl = max(lo, w << 5);
            for (; t >= tl; --t) {
                const int k = (int)((mw >> (t & 31)) & 1u) | (int)((rw >> (t & 31)) & 1u) << 1;
                if (k) {
                    run = t;
                    ty = k;
                }
                nx[t] = (uint16_t)(run | ty << kTypeShift);
            }
        }
        if (lane == 31)
            nx[T] = (uint16_t)T;
        __syncwarp();
    }
};

// The rows of a candidate move: base rows with periods a <= b rewritten
// (ta, tb = the new kinds m | r << 1 there).
struct PatchedSmem {
    MaskSmem base;
    int a, b, ta, tb;
    // First setup >= x (T if none) and its kind, for the queries of a delta
    // walk (walk_moves): x = 0 when the base plan has no setup before a, else
    // x > prev(a).  The base plan then has no setup in [x, a), and none
    // strictly between a and b (b = a, or b = a + 1 for N3 shifts), so for
    // x <= b the answer is a (if set and x <= a), else b (if set), else the
    // first base setup after b; past b it is the table entry.  x <= T
    // (nx[T] = T is the end entry).
    __device__ int next_t(int x, int &ty) const
    {
        RL_ASSERT(x > b || (base.nx[x] & kPeriodMask) >= a);   // no base setup in [x, a)
        const int e = base.nx[x > b ? x : b + 1];
        int t = e & kPeriodMask;
        ty = e >> kTypeShift;
        if (x <= b) {
            if (tb) {
                t = b;
                ty = tb;
            }
            if (x <= a && ta) {
                t = a;
                ty = ta;
            }
        }
        return t;
    }
    __device__ int next(int x) const
    {
        int ty;
        return next_t(x, ty);
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
    __device__ static uint64_t sentinel_of(int T) { return 1ull << T; }
    __device__ int next(int x) const { return next_of(M | R | sentinel(), x, T); }
    __device__ uint64_t R_mask() const { return R; }
    __device__ int setup_type(int t) const { return (int)m(t) | (int)r(t) << 1; }
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
    __device__ int next_t(int x, int &ty) const
    {
        const int t = next(x);
        ty = (int)m(t) | (int)r(t) << 1;   // 0 at the sentinel T
        return t;
    }
};

template <typename Mask> struct PatchOf;
template <> struct PatchOf<MaskSmem> {
    using type = PatchedSmem;
    __device__ static PatchedSmem make(const MaskSmem &b, int a, int bb, bool ma, bool ra,
                                       bool mb, bool rb)
    {
        return PatchedSmem{b, a, bb, (int)ma | (int)ra << 1, (int)mb | (int)rb << 1};
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
template <typename V, typename C, int SB>
__device__ inline MaskSmem load_rows(const Slot<V, C, SB> &s, MaskSmem, const uint8_t *sm,
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
            s.bs[base >> 5] = wm | wr;
        }
    }
    __syncwarp();
    return MaskSmem{s.bm, s.br, s.bs, s.nx, T};
}

template <typename V, typename C, int SB>
__device__ inline MaskReg load_rows(const Slot<V, C, SB> &, MaskReg, const uint8_t *sm,
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

// Cost of one segment [u, v) entered with cumulative remanufacturing X, from
// cdu = cd[u], cru = cr[u+1], cdv = cd[v].  Follows _kernels.py:66-95 (seg
// :70-72, avail :73, x_r :74-76, x_m and infeasibility :77-82, setup :83-86,
// unit :87, holding :88-95 summed): p_M x_M + p_R x_R + (T-u)(h_M seg - h_R
// x_R) regrouped as seg (a0 - u h_M) + x_R (b0 + u h_R).
template <typename V, typename C>
__device__ inline bool seg_cost(V cdu, V cru, V cdv, int u, bool m, bool r, V X,
                                const ProductCosts<C> &pc, C &c, V &xr)
{
    const V seg = cdv - cdu;
    const V avail = cru - X;
    xr = r ? vmin(seg, avail) : V(0);
    const V xm = seg - xr;
    // computed unconditionally (no branch): callers discard c when infeasible;
    // a chain of multiply-adds (FMA pipe) rather than a three-input add
    if constexpr (sizeof(C) == 4) {
        C acc = xr > 0 ? pc.kr : C(0);
        acc = C(seg) * (pc.a0 - C(u) * pc.hm) + acc;
        acc = C(xr) * (pc.b0 + C(u) * pc.hr) + acc;
        c = (xm > 0 ? pc.km : C(0)) * pc.one + acc;
    } else {
        c = (xr > 0 ? pc.kr : C(0)) + (xm > 0 ? pc.km : C(0)) +
            C(seg) * (pc.a0 - C(u) * pc.hm) + C(xr) * (pc.b0 + C(u) * pc.hr);
    }
    return !(xm > 0 && !m);
}

// int32 values with int64 costs: the host selects this pair only when every
// coefficient (p_M + T h_M, p_R + p_M + T h_R, k_M, k_R) is below 2^30
// (prepare / k_check_narrow, coef_bound), so a0 - u h_M and b0 + u h_R are
// exact in int32 and the two products are 32 x 32 -> 64 multiply-adds.
template <>
__device__ inline bool seg_cost<int32_t, int64_t>(int32_t cdu, int32_t cru, int32_t cdv, int u,
                                                  bool m, bool r, int32_t X,
                                                  const ProductCosts<int64_t> &pc, int64_t &c,
                                                  int32_t &xr)
{
    const int32_t seg = cdv - cdu;
    const int32_t avail = cru - X;
    xr = r ? vmin(seg, avail) : 0;
    const int32_t xm = seg - xr;
    const int32_t ca = (int32_t)pc.a0 - u * (int32_t)pc.hm;
    const int32_t cb = (int32_t)pc.b0 + u * (int32_t)pc.hr;
    const int32_t setup = (xr > 0 ? (int32_t)pc.kr : 0) + (xm > 0 ? (int32_t)pc.km : 0);
    c = (int64_t)seg * ca + (int64_t)xr * cb + setup;
    return !(xm > 0 && !m);
}

// ------------------------------------------------------------ staging

// Prefix sums of the staged rows into cd/cr; returns K0 (warp-uniform).
template <typename V, typename C, int SB>
__device__ inline C build_prefix(const Slot<V, C, SB> &s, int T, const ProductCosts<C> &pc, int lane)
{
    V carry_d = 0, carry_r = 0;
    C sum_cd = 0, sum_cr = 0;   // sum_t CD[t], sum_t CR[t] (inclusive prefixes)
    if (lane == 0) {
        s.dr.set_d(0, V(0));
        s.dr.set_r(T, V(0));   // cr[T+1]: never used, kept defined
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
            s.dr.set_d(t + 1, d);
            s.dr.set_r(t, r);
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
template <typename V, typename C, int SB>
__device__ inline void stage_plain(const Slot<V, C, SB> &s, const V *dem, const V *ret, int64_t k,
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

// Slack-level masks for the delta-walk skip (scan_pass) from the slk row
// base_pass wrote: lane l owns periods l and l + 32, so each ballot yields
// one 32-bit half.
template <typename V, typename C, int SB, typename Mask>
__device__ inline void build_slack_masks(const Slot<V, C, SB> &s, const Mask &mk, int T, int lane)
{
    const V INF = VInf<V>::value;
    __syncwarp();
    const V s0 = lane < T ? s.slk[lane] : INF;
    const V s1 = lane + 32 < T ? s.slk[lane + 32] : INF;
    uint64_t mine = 0;
#pragma unroll
    for (int j = 0; j <= kSlackLevels + 1; ++j) {
        if (j == kSlackLevels) {
            if (lane == j)
                mine = mk.R_mask();   // any delta >= 2^16: every sR setup
            continue;
        }
        const V lim = j < kSlackLevels ? (V(1) << j) : V(0);
        const uint64_t mk2 = (uint64_t)__ballot_sync(FULL, s0 < lim) |
                             ((uint64_t)__ballot_sync(FULL, s1 < lim) << 32);
        if (lane == j)
            mine = mk2;
    }
    if (lane <= kSlackLevels + 1)
        s.lm[lane] = mine;
}

// base_pass for register rows (T <= 63: lane l owns periods lL and lL + 1,
// L = 1 or 2).  The same two steps and scans as the general form, with
// each owned period's setup kind, next setup and rows read once into
// registers (step 2 reuses step 1's), next-setup queries by one clz on the
// bit-reversed rows, and each xc entry written once after the cost scan
// (no read-modify-write fix-up).
template <typename V, typename C, bool Skip, int SB>
__device__ inline bool base_pass_reg(const Slot<V, C, SB> &s, const MaskReg &mk, int T,
                                     const ProductCosts<C> &pc, int lane, C &S)
{
    const int L = (T + 31) >> 5;
    const uint64_t SRv = __brevll(mk.M | mk.R | mk.sentinel());
    const V INF = VInf<V>::value;
    bool su[2], mu[2], ru[2];
    int vv[2];
    V ed[2], er[2], cdv[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int u = lane * L + j;
        const bool valid = j < L && u < T;
        mu[j] = valid && mk.m(u);
        ru[j] = valid && mk.r(u);
        su[j] = mu[j] | ru[j];
        vv[j] = 0;
        ed[j] = er[j] = cdv[j] = 0;
        if (su[j]) {
            vv[j] = u + 1 + __clzll((long long)(SRv << (u + 1)));   // first setup > u (<= T)
            const DR<V> e = s.dr[u];
            ed[j] = e.d;
            er[j] = e.r;
            cdv[j] = s.dr[vv[j]].d;
        }
        if (Skip && valid)
            s.slk[u] = INF;
    }
    V A = 0, B = INF;
#pragma unroll
    for (int j = 0; j < 2; ++j)
        if (ru[j]) {   // only remanufacturing setups move X
            const V seg = cdv[j] - ed[j];
            A += seg;
            B = vmin<V>(B + seg, er[j]);
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
    C local = 0;
    bool ok = true;
    V xin[2];
    C cin[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        xin[j] = X;
        cin[j] = local;
        if (su[j]) {
            if (Skip && ru[j])
                s.slk[lane * L + j] = er[j] - X - (cdv[j] - ed[j]);
            C c;
            V xr;
            ok &= seg_cost<V, C>(ed[j], er[j], cdv[j], lane * L + j, mu[j], ru[j], X, pc, c, xr);
            local += c;
            X += xr;
        }
    }
    C incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        C o = __shfl_up_sync(FULL, incl, off);
        if (lane >= off)
            incl += o;
    }
    const C excl = incl - local;
#pragma unroll
    for (int j = 0; j < 2; ++j)
        if (su[j])
            s.xc.set(lane * L + j, xin[j], cin[j] + excl);
    S = __shfl_sync(FULL, incl, 31);
    if (lane == 0)
        s.xc.set(T, V(0), S);   // end entry: a walk reaching T adds S - S
    const int f = __clzll((long long)SRv);   // first setup (T if none)
    ok = ok && s.dr[f].d == 0;   // demand before the first setup (_kernels.py:58-60)
    return __all_sync(FULL, ok);
}

// Evaluate the current plan: fills xin/cpre at every setup period, returns
// feasibility and S = sum of segment costs (warp-uniform).  Lane l owns the
// periods [l*L, l*L+L).  Step 1 composes the (min,+) maps of its setups,
// a warp scan gives every lane its entering X, step 2 walks the segments.
template <typename V, typename C, typename Mask, bool Skip = false, int SB = 4>
__device__ inline bool base_pass(const Slot<V, C, SB> &s, const Mask &mk, int T,
                                 const ProductCosts<C> &pc, int lane, C &S)
{
    if constexpr (std::is_same<Mask, MaskSmem>::value)
        mk.build_tables(lane);
#ifndef RL_BASE_REG_GENERIC
    if constexpr (std::is_same<Mask, MaskReg>::value) {
        const bool feas = base_pass_reg<V, C, Skip, SB>(s, mk, T, pc, lane, S);
        if (Skip)
            build_slack_masks(s, mk, T, lane);
        __syncwarp();
        return feas;
    }
#endif
    const int L = (T + 31) >> 5;
    const int lo = lane * L, hi = min(lo + L, T);
    const V INF = VInf<V>::value;
    constexpr bool kSmem = std::is_same<Mask, MaskSmem>::value;
    V A = 0, B = INF;
    if constexpr (kSmem) {
        // setup to setup through the next-setup table (one 16-bit load per
        // setup instead of two bit-row loads per period)
        int e = lo < hi ? mk.nx[lo] : hi;
        for (int u = e & kPeriodMask; u < hi;) {
            const int e2 = mk.nx[u + 1], v = e2 & kPeriodMask;
            if ((e >> kTypeShift) & 2) {   // only remanufacturing setups move X
                const DR<V> d = s.dr[u];
                const V seg = s.dr[v].d - d.d;
                A += seg;
                B = vmin<V>(B + seg, d.r);
            }
            u = v;
            e = e2;
        }
    } else {
        for (int u = lo; u < hi; ++u) {
            if (!mk.r(u))
                continue;   // only remanufacturing setups move X
            const int v = mk.next(u + 1);
            const DR<V> e = s.dr[u];
            const V seg = s.dr[v].d - e.d;
            A += seg;
            B = vmin<V>(B + seg, e.r);
        }
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
    if constexpr (kSmem) {
        int e = lo < hi ? mk.nx[lo] : hi;
        for (int u = e & kPeriodMask; u < hi;) {
            const int e2 = mk.nx[u + 1], v = e2 & kPeriodMask;
            const int ty = e >> kTypeShift;
            const DR<V> d = s.dr[u];
            const V cdv = s.dr[v].d;
            s.xc.set(u, X, local);
            C c;
            V xr;
            ok &= seg_cost<V, C>(d.d, d.r, cdv, u, ty & 1, ty >> 1, X, pc, c, xr);
            local += c;
            X += xr;
            u = v;
            e = e2;
        }
    } else {
        for (int u = lo; u < hi; ++u) {
            const bool m = mk.m(u), r = mk.r(u);
            if (kSkip)
                s.slk[u] = INF;
            if (!(m | r))
                continue;
            const int v = mk.next(u + 1);
            const DR<V> e = s.dr[u];
            const V cdv = s.dr[v].d;
            s.xc.set(u, X, local);
            if (kSkip && r)
                s.slk[u] = e.r - X - (cdv - e.d);
            C c;
            V xr;
            ok &= seg_cost<V, C>(e.d, e.r, cdv, u, m, r, X, pc, c, xr);
            local += c;
            X += xr;
        }
    }
    C incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        C o = __shfl_up_sync(FULL, incl, off);
        if (lane >= off)
            incl += o;
    }
    const C excl = incl - local;
    if (excl != C(0)) {
        if constexpr (kSmem) {
            for (int u = lo < hi ? mk.nx[lo] & kPeriodMask : hi; u < hi;
                 u = mk.nx[u + 1] & kPeriodMask)
                s.xc.add_c(u, excl);
        } else {
            for (int u = lo; u < hi; ++u)
                if (mk.m(u) | mk.r(u))
                    s.xc.add_c(u, excl);
        }
    }
    S = __shfl_sync(FULL, incl, 31);
    if (lane == 0)
        s.xc.set(T, V(0), S);   // end entry: a walk reaching T adds S - S
    const int f = mk.next(0);
    ok = ok && s.dr[f].d == 0;   // demand before the first setup (_kernels.py:58-60)
    const bool feas = __all_sync(FULL, ok);
    if (kSkip)
        build_slack_masks(s, mk, T, lane);
    __syncwarp();
    return feas;
}

// Incremental base pass for shared-memory rows after the applied move
// rewrote periods a <= b (vnd_product).  The new plan equals the old one
// before p = prev(a) and, past the first setup v > b where the re-walked X
// equals the old entering X, everywhere except for a constant shift of the
// prefix costs -- the resynchronisation the delta walk uses.  So: rebuild
// nx on [p+1, b], re-walk the move's segments from p writing their
// {xin, cpre}, add the cost shift to the setups past the resync point (or
// end the walk at T).  Identical values to a full base_pass (tested: the
// C4 pins, the long-horizon fuzz and GVNS goldens).  S: the winning total.
template <typename V, typename C, int SB>
__device__ inline void rebase_smem(const Slot<V, C, SB> &s, const MaskSmem &mk, int T,
                                   const ProductCosts<C> &pc, int lane, C &S, int a, int b)
{
    const int p = mk.prev(a);
    {   // next-setup table on [p + 1, b]: a, b (if setups now) or nx[b + 1]
        const int eb1 = mk.nx[b + 1];
        const int ka = (int)mk.m(a) | (int)mk.r(a) << 1, kb = (int)mk.m(b) | (int)mk.r(b) << 1;
        __syncwarp();
        for (int t = p + 1 + lane; t <= b; t += 32) {
            int e = eb1;
            if (kb)
                e = b | kb << kTypeShift;
            if (ka && t <= a)
                e = a | ka << kTypeShift;
            mk.nx[t] = (uint16_t)e;
        }
        __syncwarp();
    }
    int u;
    V X;
    C acc;
    if (p >= 0) {   // the prefix before p is unchanged
        const XC<V, C> e = s.xc[p];
        u = p;
        X = e.x;
        acc = e.c;
    } else {
        u = mk.nx[0] & kPeriodMask;
        X = 0;
        acc = 0;
    }
    const C S_old = s.xc[T].c;
    bool resync = false;
    int vs = T;
    C delta = 0;
    while (u < T) {
        const int ty = mk.nx[u] >> kTypeShift;   // u is a setup: its own entry
        const int v = mk.nx[u + 1] & kPeriodMask;
        const DR<V> d = s.dr[u];
        const V cdv = s.dr[v].d;
        if (lane == 0)
            s.xc.set(u, X, acc);
        C c;
        V xr;
        seg_cost<V, C>(d.d, d.r, cdv, u, ty & 1, ty >> 1, X, pc, c, xr);
        acc += c;
        X += xr;
        if (v > b && v < T) {
            const XC<V, C> o = s.xc[v];   // past the move: a setup of both plans
            if (X == o.x) {
                resync = true;
                vs = v;
                delta = acc - o.c;
                break;
            }
        }
        u = v;
    }
    __syncwarp();
    C S_new = acc;
    if (resync) {
        S_new = S_old + delta;
        if (delta != C(0))
            for (int t = vs + lane; t < T; t += 32)
                if (mk.setup(t))
                    s.xc.add_c(t, delta);
    }
    RL_ASSERT(S_new == S);
    S = S_new;
    if (lane == 0)
        s.xc.set(T, V(0), S);
    __syncwarp();
}

// The same incremental base pass for register rows (the throughput kernel;
// the slack-skip kernel rebuilds its slack rows in a full base_pass): the
// rows are already the new plan's, next setups by clz on the bit-reversed
// rows, and each lane shifts the prefix costs of its own periods.
template <typename V, typename C, int SB>
__device__ inline void rebase_reg(const Slot<V, C, SB> &s, const MaskReg &mk, int T,
                                  const ProductCosts<C> &pc, int lane, C &S, int a, int b)
{
    const uint64_t SRv = __brevll(mk.M | mk.R | mk.sentinel());
    const int p = mk.prev(a);
    int u;
    V X;
    C acc;
    if (p >= 0) {   // the prefix before p is unchanged
        const XC<V, C> e = s.xc[p];
        u = p;
        X = e.x;
        acc = e.c;
    } else {
        u = __clzll((long long)SRv);   // first setup (T if none)
        X = 0;
        acc = 0;
    }
    const C S_old = s.xc[T].c;
    bool resync = false;
    int vs = T;
    C delta = 0;
    while (u < T) {
        const int v = u + 1 + __clzll((long long)(SRv << (u + 1)));
        const DR<V> d = s.dr[u];
        const V cdv = s.dr[v].d;
        if (lane == 0)
            s.xc.set(u, X, acc);
        C c;
        V xr;
        seg_cost<V, C>(d.d, d.r, cdv, u, mk.m(u), mk.r(u), X, pc, c, xr);
        acc += c;
        X += xr;
        if (v > b && v < T) {
            const XC<V, C> o = s.xc[v];   // past the move: a setup of both plans
            if (X == o.x) {
                resync = true;
                vs = v;
                delta = acc - o.c;
                break;
            }
        }
        u = v;
    }
    __syncwarp();
    C S_new = acc;
    if (resync) {
        S_new = S_old + delta;
        if (delta != C(0)) {
            const int L = (T + 31) >> 5;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int t = lane * L + j;
                if (j < L && t < T && t >= vs && (mk.m(t) | mk.r(t)))
                    s.xc.add_c(t, delta);
            }
        }
    }
    RL_ASSERT(S_new == S);
    S = S_new;
    if (lane == 0)
        s.xc.set(T, V(0), S);
    __syncwarp();
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
// Register rows (T <= 63): the N3/N4 validity masks are bit operations on
// the rows (N3 row x: left shifts x & ~(x << 1) minus period 0, right shifts
// x & ~(x >> 1) below T - 1; N4: M ^ R), so each lane places its periods t
// and t + 32 with prefix popcounts in one round (slot order = row*2T + 2t +
// dir, the reference's list_moves order).
struct RegMoveMasks {
    uint64_t lm, rm, lr, rr;   // N3 left/right shifts of the M and R rows
};
__device__ inline RegMoveMasks reg_move_masks(const MaskReg &mk)
{
    const int T = mk.T;
    const uint64_t all = (1ull << T) - 1, nolast = (1ull << (T - 1)) - 1;
    RegMoveMasks r;
    r.lm = mk.M & ~(mk.M << 1) & all & ~1ull;
    r.rm = mk.M & ~(mk.M >> 1) & nolast;
    r.lr = mk.R & ~(mk.R << 1) & all & ~1ull;
    r.rr = mk.R & ~(mk.R >> 1) & nolast;
    return r;
}

template <typename V, typename C, int SB>
__device__ inline int enumerate_moves(const Slot<V, C, SB> &s, const MaskReg &mk, int nbh, int T,
                                      int lane)
{
    if (nbh <= 2)
        return T;
    int n;
    if (nbh == 4) {
        const uint64_t x = (mk.M ^ mk.R) & ((1ull << T) - 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            if (t < T && ((x >> t) & 1))
                s.mv[__popcll(x & ((1ull << t) - 1))] = (uint16_t)t;
        }
        n = __popcll(x);
    } else {
        const RegMoveMasks q = reg_move_masks(mk);
        const int nm = __popcll(q.lm) + __popcll(q.rm);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            if (t < T) {
                const uint64_t below = (1ull << t) - 1;
                const int pm = __popcll(q.lm & below) + __popcll(q.rm & below);
                const int pr = nm + __popcll(q.lr & below) + __popcll(q.rr & below);
                const int lm = (q.lm >> t) & 1, lr = (q.lr >> t) & 1;
                if (lm)
                    s.mv[pm] = (uint16_t)(2 * t);
                if ((q.rm >> t) & 1)
                    s.mv[pm + lm] = (uint16_t)(2 * t + 1);
                if (lr)
                    s.mv[pr] = (uint16_t)(2 * T + 2 * t);
                if ((q.rr >> t) & 1)
                    s.mv[pr + lr] = (uint16_t)(2 * T + 2 * t + 1);
            }
        }
        n = nm + __popcll(q.lr) + __popcll(q.rr);
    }
    __syncwarp();
    return n;
}

// Shared-memory rows (T > 63): the same masks word by word (lane w owns
// periods 32w..32w+31, T <= 32 x 32 here is not assumed: lanes loop over
// words), warp prefix sums of the per-word counts, and each lane writes its
// word's slots in period order.
struct WordMoveMasks {
    uint32_t lm, rm, lr, rr, sw;   // N3 left/right of the M and R rows, N4
};
__device__ inline WordMoveMasks word_move_masks(const MaskSmem &mk, int w, int NW)
{
    const int T = mk.T;
    const uint32_t m = mk.bm[w], r = mk.br[w];
    const uint32_t mp = w > 0 ? mk.bm[w - 1] : 0u, rp = w > 0 ? mk.br[w - 1] : 0u;
    const uint32_t mn = w + 1 < NW ? mk.bm[w + 1] : 0u, rn = w + 1 < NW ? mk.br[w + 1] : 0u;
    const int base = 32 * w;
    const uint32_t in_t = T - base >= 32 ? 0xffffffffu : (1u << (T - base)) - 1;      // t < T
    const uint32_t in_t1 = T - 1 - base >= 32 ? 0xffffffffu
                           : T - 1 - base <= 0 ? 0u : (1u << (T - 1 - base)) - 1;   // t + 1 < T
    const uint32_t not0 = w == 0 ? ~1u : 0xffffffffu;                                // t > 0
    WordMoveMasks q;
    q.lm = m & ~((m << 1) | (mp >> 31)) & in_t & not0;
    q.rm = m & ~((m >> 1) | (mn << 31)) & in_t1;
    q.lr = r & ~((r << 1) | (rp >> 31)) & in_t & not0;
    q.rr = r & ~((r >> 1) | (rn << 31)) & in_t1;
    q.sw = (m ^ r) & in_t;
    return q;
}

template <typename C>
__device__ inline int warp_excl_scan(int x, int lane, int &total)
{
    int incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(FULL, incl, off);
        if (lane >= off)
            incl += o;
    }
    total = __shfl_sync(FULL, incl, 31);
    return incl - x;
}

template <typename V, typename C, int SB>
__device__ inline int enumerate_moves(const Slot<V, C, SB> &s, const MaskSmem &mk, int nbh, int T,
                                      int lane)
{
    if (nbh <= 2)
        return T;
    // few words: ballot rounds (the two are within noise up to T ~ 130;
    // the word path wins at C4: 214 -> 196 ms)
    if (T <= RL_WORD_ENUM_MIN_T)
        return enumerate_moves_ballot(s, mk, nbh, T, lane);
    const int NW = (T + 31) >> 5;
    int n = 0;   // slots written by earlier word groups
    for (int w0 = 0; w0 < NW; w0 += 32) {
        const int w = w0 + lane;
        WordMoveMasks q{0u, 0u, 0u, 0u, 0u};
        if (w < NW)
            q = word_move_masks(mk, w, NW);
        if (nbh == 4) {
            int tot;
            int pos = n + warp_excl_scan<C>(__popc(q.sw), lane, tot);
            for (uint32_t x = q.sw; x; x &= x - 1)
                s.mv[pos++] = (uint16_t)(32 * w + __ffs(x) - 1);
            n += tot;
        } else {
            // row M slots of every word come before row R slots of any word,
            // so the M counts are scanned over all word groups first
            int totm;
            int pm = warp_excl_scan<C>(__popc(q.lm) + __popc(q.rm), lane, totm);
            (void)pm;
            n += totm;
        }
    }
    if (nbh == 4) {
        __syncwarp();
        return n;
    }
    // N3: second sweep writes the slots (row M at [0, nM), row R after)
    const int nM = n;
    int om = 0, orr = nM;
    for (int w0 = 0; w0 < NW; w0 += 32) {
        const int w = w0 + lane;
        WordMoveMasks q{0u, 0u, 0u, 0u, 0u};
        if (w < NW)
            q = word_move_masks(mk, w, NW);
        int tm, tr;
        int pm = om + warp_excl_scan<C>(__popc(q.lm) + __popc(q.rm), lane, tm);
        int pr = orr + warp_excl_scan<C>(__popc(q.lr) + __popc(q.rr), lane, tr);
        for (uint32_t x = q.lm | q.rm; x; x &= x - 1) {
            const int i = __ffs(x) - 1, t = 32 * w + i;
            if ((q.lm >> i) & 1)
                s.mv[pm++] = (uint16_t)(2 * t);
            if ((q.rm >> i) & 1)
                s.mv[pm++] = (uint16_t)(2 * t + 1);
        }
        for (uint32_t x = q.lr | q.rr; x; x &= x - 1) {
            const int i = __ffs(x) - 1, t = 32 * w + i;
            if ((q.lr >> i) & 1)
                s.mv[pr++] = (uint16_t)(2 * T + 2 * t);
            if ((q.rr >> i) & 1)
                s.mv[pr++] = (uint16_t)(2 * T + 2 * t + 1);
        }
        om += tm;
        orr += tr;
    }
    __syncwarp();
    return orr;
}

template <typename V, typename C, typename Mask, int SB>
__device__ inline int enumerate_moves_ballot(const Slot<V, C, SB> &s, const Mask &mk, int nbh, int T,
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

// lexicographic (cost, slot) minimum over the warp by redux.sync: the
// minimum cost (int64: high words signed, then low words of the lanes
// holding the minimal high word), then the smallest key among its lanes
template <typename C>
__device__ inline void warp_argmin(C &best, int &key)
{
    bool at;
    if constexpr (sizeof(C) == 4) {
        const C m = (C)__reduce_min_sync(FULL, (int)best);
        at = best == m;
        best = m;
    } else {
        const int hi = (int)((uint64_t)best >> 32);
        const unsigned lo = (unsigned)(uint64_t)best;
        const int mh = __reduce_min_sync(FULL, hi);
        const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
        at = hi == mh && lo == ml;
        best = (C)(((uint64_t)(uint32_t)mh << 32) | ml);
    }
    key = (int)__reduce_min_sync(FULL, at ? (unsigned)key : 0xffffffffu);
}

// Score the moves i = wi, wi + nw, wi + 2 nw, ... (< n) of the current list
// on this warp (nw warps share a product in the CTA variant); per-lane
// results in best/key (initialise best = S, key = INT_MAX).
//
// Lane state: 0 idle, 1 a move just taken, 2 walking.  A walking lane is at
// setup u of its candidate plan with entering X, the candidate's segment
// costs so far in acc, and cd[u], cr[u+1] carried from the previous step
// (each step loads one {cd, cr} pair and one {cpre, xin} pair).
// Previous-setup table for the dense passes (N1/N2) of shared-memory rows:
// pv[t] = last setup < t (0xffff if none), t <= T, written into the move-list
// area (unused by dense passes).  A dense move's set-up then reads pv[a]
// beside nx[a] instead of scanning the setup words backwards (one shared-
// memory round trip instead of a data-dependent loop).  Lane chunks with a
// warp max-scan of each chunk's last setup, like build_tables.
__device__ inline void build_prev_table(const MaskSmem &mk, uint16_t *pv, int T, int lane)
{
    const int L = (T + 32) >> 5;   // periods 0..T
    const int lo = lane * L, hi = min(lo + L, T + 1);
    int last = -1;   // last setup in [lo, hi) (periods < T)
    if (lo < hi) {
        const int top = min(hi, T) - 1;
        if (top >= lo) {
            int w = top >> 5;
            uint32_t bits = mk.bs[w] & (0xffffffffu >> (31 - (top & 31)));
            const int wl = lo >> 5;
            while (!bits && w > wl) {
                --w;
                bits = mk.bs[w];
            }
            const int f = bits ? (w << 5) + 31 - __clz(bits) : -1;
            last = f >= lo ? f : -1;
        }
    }
    int sm = last;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(FULL, sm, off);
        if (lane >= off)
            sm = max(sm, o);
    }
    int run = __shfl_up_sync(FULL, sm, 1);   // last setup before this chunk
    if (lane == 0)
        run = -1;
    for (int t = lo; t < hi; ++t) {
        pv[t] = (uint16_t)run;   // -1 -> 0xffff
        if (t < T && mk.setup(t))
            run = t;
    }
    __syncwarp();
}

template <typename V, typename C, typename Mask, bool Skip = false, int SB = 4>
__device__ inline void walk_moves(const Slot<V, C, SB> &s, const Mask &mk, int T,
                                  const ProductCosts<C> &pc, C S, int nbh, int n, int lane,
                                  int wi, int nw, C &best, int &key, bool pv_table = false)
{
    const bool dense = nbh <= 2;
    const unsigned lt = (1u << lane) - 1;
    constexpr bool kSkip = Skip && std::is_same<Mask, MaskReg>::value;
    constexpr bool kRegMask = std::is_same<Mask, MaskReg>::value;
    // the base rows (a valid candidate for the discarded steps of idle lanes)
    typename PatchOf<Mask>::type pw =
        PatchOf<Mask>::make(mk, 0, 0, mk.m(0), mk.r(0), mk.m(0), mk.r(0));
    int u = 0, b = 0, slot = 0, tu = 0;   // tu: kind (m | r << 1) of setup u
    V X = 0, cdu = 0, cru = 0;
    C acc = 0;
    int gi = lane * nw + wi;
    int state = gi < n ? 1 : 0;
    int next = 32;   // move indices handed out so far (in units of this warp's share)
#ifdef RL_WALK_STATS
    int ws_cur = 0, ws_max = 0, ws_lane = 0, ws_it = 0, ws_pend = 0;
#endif
    for (;;) {
#ifdef RL_WALK_STATS
        ++ws_it;
        ws_pend += __any_sync(FULL, state == 1);
        if (state == 1 && ws_cur) {
            atomicAdd(&g_walk_stats[8 + min(ws_cur, 63)], 1ull);
            ws_max = max(ws_max, ws_cur);
            ws_cur = 0;
        }
#endif
#ifndef RL_SETUP_REPS
#define RL_SETUP_REPS 1   // measurement only: > 1 repeats the (idempotent) move set-up
#endif
        const bool setup_now = state == 1;
        for (int rep = 0; rep < RL_SETUP_REPS; ++rep) {
            if (!setup_now)
                break;
            state = 1;
            RL_ASSERT(gi < n && gi < 4 * T);
            slot = dense ? gi : s.mv[gi];
            const MoveDesc d = slot_move(mk, nbh, slot, T);
            int a;
            pw = patch_of<V, C, Mask>(mk, d, a, b);
            int p;
            if constexpr (!kRegMask && RL_DENSE_PREV_TABLE) {
                p = dense && pv_table ? (int)(int16_t)s.mv[a] : mk.prev(a);   // build_prev_table
            } else {
                p = mk.prev(a);
            }
            if (p >= 0) {   // the prefix before p is the base plan's
                const XC<V, C> e = s.xc[p];
                u = p;
                if (!kRegMask)
                    tu = mk.setup_type(p);
                acc = e.c;
                X = e.x;
            } else {
                u = kRegMask ? pw.next(0) : pw.next_t(0, tu);
                acc = 0;
                X = 0;
            }
            const DR<V> e = s.dr[u];
            cdu = e.d;
            cru = e.r;
            // no setup before the move: demand ahead of the first setup is
            // infeasible; no setup at all and no demand: cost 0
            state = (p >= 0 || cdu == 0) ? 2 : 0;
            if (state == 2 && u >= T) {
                state = 0;
                if (acc < best) {
                    best = acc;
                    key = slot;
                }
            }
        }
#ifndef RL_STEP_BRANCH
#define RL_STEP_BRANCH 0
#endif
        // one segment of the walk, branch-free (every busy lane issues the
        // same instructions): cost, resync test, finish, argmin update.
        // Issued unconditionally (no divergent branch and reconvergence per
        // iteration): idle lanes step from period T - 1 (a valid query whose
        // next setup is the end, T) and their results are discarded.
#pragma unroll
        for (int rep = 0; rep < (kRegMask ? RL_WALK_STEPS_REG : RL_WALK_STEPS_SMEM); ++rep) {
            const bool walking = state == 2;
            if (RL_STEP_BRANCH == 0 || walking) {
#ifdef RL_WALK_STATS
                ws_cur += walking;
                ws_lane += walking;
#endif
                if (!walking)
                    u = T - 1;   // a valid start for the discarded step
                // register masks test the candidate's bits directly (measured
                // faster); shared-memory masks carry the kind from the nx table
                int tv = 0, v;
                bool mu, ru;
                if constexpr (kRegMask) {
                    v = pw.next(u + 1);
                    mu = pw.m(u);
                    ru = pw.r(u);
                } else {
                    v = pw.next_t(u + 1, tv);
                    mu = tu & 1;
                    ru = tu >> 1;
                }
                const DR<V> ev = s.dr[v];
                C c;
                V xr;
                const bool ok = seg_cost<V, C>(cdu, cru, ev.d, u, mu, ru, X, pc, c, xr);
                const XC<V, C> bv = s.xc[v];   // v <= T; xc[T].c = S
                acc += c;
                X += xr;
                // past the move the rows equal the base plan's; only X may differ
                bool fin;
                C total;
                if constexpr (kSkip) {
                    const bool past = v < T && v > b;
                    // Slack skip: with X = base + delta at v, a later segment costs
                    // what it costs in the base plan unless it starts at an sR setup
                    // whose slack < max(delta, 0) (for delta < 0: slack < 0), where
                    // min(seg, avail) changes.  Jump to the next setup of the
                    // slack-level mask bounding that set (false positives are just
                    // walked exactly), adding the base cost of the segments skipped;
                    // no such setup left = the rest of the base plan (resync).
                    const V delta = X - bv.x;
                    const int li = delta < 0 ? kSlackLevels + 1 : min(ceil_log2(delta), kSlackLevels);
                    const int q = MaskReg::next_of(s.lm[li] | MaskReg::sentinel_of(T), v, T);
                    fin = v >= T || (past && (delta == 0 || q >= T));
                    total = acc + (S - bv.c);
                    const int qq = past && q < T ? q : v;
                    const XC<V, C> bq = s.xc[qq];
                    const DR<V> eq = s.dr[qq];
                    acc += bq.c - bv.c;   // 0 unless past (qq == v otherwise)
                    X = past ? bq.x + delta : X;
                    u = qq;
                    cdu = eq.d;
                    cru = eq.r;
                } else {
                    // done at the end (v = T > b) or once X re-synchronises past
                    // the move
                    fin = v > b && (v >= T || X == bv.x);
                    if constexpr (sizeof(C) == 4)
                        total = acc * pc.one + (bv.c * pc.mone + S);   // two IMADs, not an IADD3
                    else
                        total = acc + (S - bv.c);
                    u = v;
                    tu = tv;
                    cdu = ev.d;
                    cru = ev.r;
                }
                // total = acc + S - cpre[v]: the base suffix when resynced, and
                // just acc at v = T (xc[T].c = S); only read when fin
                const bool take = walking && ok && fin && total < best;
                best = take ? total : best;
                key = take ? slot : key;
                state = walking && ok && !fin ? 2 : 0;
            }
        }
        const unsigned m = __ballot_sync(FULL, state == 0);
        const bool more = m != FULL || next * nw + wi < n;
        // refill idle lanes in batches (the set-up branch costs the whole
        // warp's issue slots however few lanes take a move)
        if (m == FULL || __popc(m) >= (kRegMask ? RL_REFILL_MIN : RL_REFILL_MIN_SMEM)) {
            if (state == 0) {
                gi = (next + __popc(m & lt)) * nw + wi;
                state = gi < n ? 1 : 0;
            }
            next += __popc(m);
        }
        if (!more)
            break;
    }
#ifdef RL_WALK_STATS
    if (ws_cur) {
        atomicAdd(&g_walk_stats[8 + min(ws_cur, 63)], 1ull);
        ws_max = max(ws_max, ws_cur);
    }
    int tot = ws_lane, mx = ws_max, busy = ws_lane;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        tot += __shfl_xor_sync(FULL, tot, off);
        mx = max(mx, __shfl_xor_sync(FULL, mx, off));
        busy = max(busy, __shfl_xor_sync(FULL, busy, off));
    }
    if (lane == 0) {
        atomicAdd(&g_walk_stats[0], 1ull);
        atomicAdd(&g_walk_stats[1], (unsigned long long)ws_it);
        atomicAdd(&g_walk_stats[2], (unsigned long long)n);
        atomicAdd(&g_walk_stats[3], (unsigned long long)tot);
        atomicAdd(&g_walk_stats[4], (unsigned long long)mx);
        atomicAdd(&g_walk_stats[5], (unsigned long long)busy);
        atomicAdd(&g_walk_stats[72 + min(ws_it, 63)], 1ull);
        atomicAdd(&g_walk_stats[6], (unsigned long long)ws_pend);
    }
#endif
}

template <typename V, typename C, typename Mask, bool Skip = false, int SB = 4>
__device__ inline PassResult scan_pass(const Slot<V, C, SB> &s, const Mask &mk, int T,
                                       const ProductCosts<C> &pc, C S, int nbh, int lane,
                                       C &best_out)
{
    int n = enumerate_moves(s, mk, nbh, T, lane);
#ifdef RL_ENUM_TWICE   // measurement only: the enumeration's share of the descent
    n = enumerate_moves(s, mk, nbh, T, lane);
#endif
    C best = S;
    int key = 0x7fffffff;
    const bool pv = std::is_same<Mask, MaskSmem>::value && RL_DENSE_PREV_TABLE && nbh <= 2;
    if constexpr (std::is_same<Mask, MaskSmem>::value)
        if (pv)
            build_prev_table(mk, s.mv, T, lane);
    walk_moves<V, C, Mask, Skip>(s, mk, T, pc, S, nbh, n, lane, 0, 1, best, key, pv);
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
__device__ inline int move_count(const MaskReg &mk, int nbh, int T, int)
{
    if (nbh <= 2)
        return T;
    if (nbh == 4)
        return __popcll((mk.M ^ mk.R) & ((1ull << T) - 1));
    const RegMoveMasks q = reg_move_masks(mk);
    return __popcll(q.lm) + __popcll(q.rm) + __popcll(q.lr) + __popcll(q.rr);
}

__device__ inline int move_count(const MaskSmem &mk, int nbh, int T, int lane)
{
    if (nbh <= 2)
        return T;
    const int NW = (T + 31) >> 5;
    int c = 0;
    for (int w = lane; w < NW; w += 32) {
        const WordMoveMasks q = word_move_masks(mk, w, NW);
        c += nbh == 4 ? __popc(q.sw) : __popc(q.lm) + __popc(q.rm) + __popc(q.lr) + __popc(q.rr);
    }
    return __reduce_add_sync(FULL, (unsigned)c);
}

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
