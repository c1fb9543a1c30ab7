// remlot_b200.cu -- sm_100a kernels and the C ABI (include/remlot_b200.h).
//
// Kernels (DESIGN.md section 4 has the roofline of each):
//   k_bounds          per-product range check that picks exact narrow types
//   k_narrow          int64 -> V conversion of demand/returns (instance layout)
//   k_product_costs   plan.evaluate / _kernels.product_costs
//   k_scan            one lockstep pass: _kernels.scan_products
//   k_vnd             persistent resident VND to local optimum (vnd.vnd)
//   k_vnd_finalize    totals, reference-equivalent eval count
//   k_apply_scan      _kernels.apply_scan
//   k_initial         plan.initial_solution
//   k_list_moves      _kernels.list_moves for one product row
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <type_traits>

#include "../../include/remlot_b200.h"
#include "rng_device.cuh"
#include "vnd_device.cuh"

using namespace rl;

constexpr int kWarpsPerCta = 4;

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            return fail(RL_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                           \
    } while (0)

// Calls on one handle are serialised by its recursive mutex (the reference's
// kernels are nogil and reentrant, _kernels.py:3-4; bench.py:196-198 runs
// solve_scheme from several threads on one Instance).  Recursive: entry
// points call each other (rl_vnd -> rl_vnd_device -> ...).
#define RL_GUARD(h) \
    std::unique_lock<std::recursive_mutex> rl_guard_ = (h) ? std::unique_lock<std::recursive_mutex>((h)->mu) \
                                                           : std::unique_lock<std::recursive_mutex>()

#define CKL()                                                                        \
    do {                                                                             \
        ++h->launches;                                                               \
        cudaError_t e_ = cudaGetLastError();                                         \
        if (e_ != cudaSuccess)                                                       \
            return fail(RL_ECUDA, "kernel launch failed: %s (%s:%d)",                \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                 \
    } while (0)

// ------------------------------------------------------------------ views

template <typename V>
struct InstView {
    int64_t K;
    int T;
    const V *dem, *ret;
    const int64_t *cost6;   // 6 x K int64
    int one;                // 1, a kernel parameter the compiler cannot see through
};

template <typename C>
__device__ inline ProductCosts<C> load_costs(const int64_t *c6, int64_t K, int64_t k, int T,
                                             int one)
{
    ProductCosts<C> p;
    p.km = C(c6[k]);
    p.kr = C(c6[K + k]);
    p.hm = C(c6[2 * K + k]);
    p.hr = C(c6[3 * K + k]);
    p.pm = C(c6[4 * K + k]);
    p.pr = C(c6[5 * K + k]);
    p.a0 = p.pm + C(T) * p.hm;            // wrapping is exact
    p.b0 = p.pr - p.pm - C(T) * p.hr;
    p.one = C(one);                        // 1, opaque to the compiler (kernel parameter)
    p.mone = -p.one;
    return p;
}

template <typename V>
__device__ inline bool tma_ok(const InstView<V> &in, int64_t k)
{
    const size_t bytes = (size_t)in.T * sizeof(V);
    return !(bytes & 15) && !(((uintptr_t)(in.dem + k * in.T)) & 15) &&
           !(((uintptr_t)(in.ret + k * in.T)) & 15);
}

template <typename V, typename C, int SB>
__device__ inline void stage_begin(const Slot<V, C, SB> &s, const InstView<V> &in, int64_t k, int lane)
{
    if (lane == 0 && tma_ok(in, k)) {
        // order our earlier generic reads of the stage before the async-proxy write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_issue<V>(s.stage, in.dem, in.ret, k, in.T, s.bar);
    }
}

template <typename V, typename C, int SB>
__device__ inline void stage_end(const Slot<V, C, SB> &s, const InstView<V> &in, int64_t k, int lane,
                                 uint32_t &phase)
{
    if (tma_ok(in, k)) {
        mbar_wait(s.bar, phase);
        phase ^= 1;
    } else {
        stage_plain(s, in.dem, in.ret, k, in.T, lane);
    }
    __syncwarp();
}

// --------------------------------------------------------------- kernels

// Largest per-period cost coefficient of product k (seg_cost's a0 - u h_M,
// b0 + u h_R, k_M, k_R in magnitude): below 2^30 the int32-value /
// int64-cost kernels multiply in 32 x 32 -> 64 bits (seg_cost<int32, int64>).
__device__ inline double coef_bound(const double *c, int T)
{
    return fmax(fmax(c[4] + (double)T * c[2], c[5] + c[4] + (double)T * c[3]), fmax(c[0], c[1]));
}

__global__ void k_bounds(int64_t K, int T, const int64_t *dem, const int64_t *ret,
                         const int64_t *c6, unsigned long long *out /* [sumDR, B] as double bits */,
                         unsigned long long *qmax /* coef_bound, double bits */, int *negative,
                         unsigned long long *sdsr /* max sum D, max sum R, double bits */)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double sdr = 0.0, B = 0.0, Q = 0.0, SD = 0.0, SR = 0.0;
    if (k < K) {
        double sd = 0.0, sr = 0.0;
        bool neg = false;
        for (int t = 0; t < T; ++t) {
            const int64_t d = dem[k * T + t], r = ret[k * T + t];
            neg |= d < 0 || r < 0;
            sd += (double)d;
            sr += (double)r;
        }
        double c[6];
        for (int i = 0; i < 6; ++i) {
            c[i] = (double)c6[i * K + k];
            neg |= c6[i * K + k] < 0;
        }
        if (neg)
            atomicExch(negative, 1);
        sdr = sd + sr;
        SD = sd;
        SR = sr;
        // upper bound of any plan's cost and of every intermediate term
        B = (double)T * (c[0] + c[1]) + (c[4] + c[5]) * sd + (double)T * c[2] * sd +
            (double)T * c[3] * sr;
        Q = coef_bound(c, T);
    }
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(sdr));
    atomicMax(&out[1], (unsigned long long)__double_as_longlong(B));
    atomicMax(qmax, (unsigned long long)__double_as_longlong(Q));
    atomicMax(&sdsr[0], (unsigned long long)__double_as_longlong(SD));
    atomicMax(&sdsr[1], (unsigned long long)__double_as_longlong(SR));
}

template <typename V>
__global__ void k_narrow(int64_t n, const int64_t *src, V *dst)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = V(src[i]);
}

// Generic "warp per product" prologue: stage rows, costs, prefix, plan.
template <typename V, typename C, typename Mask, int SB>
__device__ inline C load_product(const Slot<V, C, SB> &s, const InstView<V> &in, const uint8_t *sm,
                                 const uint8_t *sr, int64_t k, int lane, uint32_t &phase,
                                 ProductCosts<C> &pc, Mask &mk)
{
    stage_begin(s, in, k, lane);
    pc = load_costs<C>(in.cost6, in.K, k, in.T, in.one);
    mk = load_rows(s, Mask{}, sm, sr, k, in.T, lane);
    stage_end(s, in, k, lane, phase);
    return build_prefix(s, in.T, pc, lane);
}

template <typename V, typename C, typename Mask>
__global__ void __launch_bounds__(128) k_product_costs(InstView<V> in, const uint8_t *sm,
                                                        const uint8_t *sr, int64_t lo, int64_t hi,
                                                        int64_t *out)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Slot<V, C> s = carve<V, C>(smem + warp * slot_bytes<V, C>(in.T), in.T);
    if (lane == 0)
        mbar_init(s.bar);
    __syncwarp();
    uint32_t phase = 0;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = lo + blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; k < hi; k += nwarps) {
        ProductCosts<C> pc;
        Mask mk;
        const C K0 = load_product(s, in, sm, sr, k, lane, phase, pc, mk);
        C S;
        const bool feas = base_pass(s, mk, in.T, pc, lane, S);
        if (lane == 0)
            out[k] = feas ? (int64_t)(K0 + S) : RL_INFEASIBLE;
        __syncwarp();
    }
}

template <typename V, typename C, typename Mask>
__global__ void __launch_bounds__(128) k_scan(InstView<V> in, const uint8_t *sm, const uint8_t *sr,
                                               int64_t lo, int64_t hi, int nbh, int64_t *dec,
                                               int64_t *p0, uint8_t *m0, uint8_t *r0, int64_t *p1,
                                               uint8_t *m1, uint8_t *r1,
                                               unsigned long long *evals)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Slot<V, C> s = carve<V, C>(smem + warp * slot_bytes<V, C>(in.T), in.T);
    if (lane == 0)
        mbar_init(s.bar);
    __syncwarp();
    uint32_t phase = 0;
    const int T = in.T;
    unsigned long long my_evals = 0;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = lo + blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; k < hi; k += nwarps) {
        ProductCosts<C> pc;
        Mask mk;
        load_product(s, in, sm, sr, k, lane, phase, pc, mk);
        C S;
        const bool feas = base_pass(s, mk, T, pc, lane, S);
        int64_t o_dec = 0;
        MoveDesc d{-1, -1, false, false, false, false};
        if (feas) {
            C best;
            const PassResult r = scan_pass(s, mk, T, pc, S, nbh, lane, best);
            my_evals += r.n_moves;
            if (r.improved) {
                d = slot_move(mk, nbh, r.slot, T);
                o_dec = (int64_t)(S - best);
            }
        }
        if (lane == 0) {
            dec[k] = o_dec;
            p0[k] = d.p0;
            p1[k] = d.p1;
            m0[k] = d.m0;
            r0[k] = d.r0;
            m1[k] = d.m1;
            r1[k] = d.r1;
        }
        __syncwarp();
    }
    if (lane == 0 && my_evals)
        atomicAdd(evals, my_evals);
}

struct VndStats {
    int64_t evals;
    int sweeps, moves, ntot;
};

// One product's VND to its fixpoint (vnd.py:277-288 restricted to one
// product): sweeps of N1..Nk_max, each pass scans and applies the best
// strictly improving move.  S0/S = segment-cost sums before/after; pass
// decreases go to trace_dec[sweep*k_max + nbh-1] when trace_dec != nullptr.
// Returns the base plan's feasibility (an infeasible product is skipped,
// _kernels.py:289-290, and counts one sweep).
template <typename V, typename C, typename Mask, bool Skip, int SB>
__device__ inline bool vnd_product(const Slot<V, C, SB> &s, Mask &mk, int T, const ProductCosts<C> &pc,
                                   int k_max, int lane, C &S0, C &S, VndStats &st,
                                   unsigned long long *trace_dec, int64_t cap_sweeps,
                                   int *overflow)
{
    st.evals = 0;
    st.sweeps = 0;
    st.moves = 0;
    st.ntot = 0;
    const bool feas = base_pass<V, C, Mask, Skip>(s, mk, T, pc, lane, S);
    S0 = S;
    if (!feas) {
        st.sweeps = 1;
        return false;
    }
    bool dirty = false;
    int ma = 0, mb = 0;   // the applied move's periods (a <= b)
    for (;;) {
        bool improved = false;
        for (int nbh = 1; nbh <= k_max; ++nbh) {
            if (dirty) {
#ifndef RL_NO_REBASE
                if constexpr (std::is_same<Mask, MaskSmem>::value)
                    rebase_smem<V, C, SB>(s, mk, T, pc, lane, S, ma, mb);
                else if constexpr (!Skip)
                    rebase_reg<V, C, SB>(s, mk, T, pc, lane, S, ma, mb);
                else
#endif
                    base_pass<V, C, Mask, Skip>(s, mk, T, pc, lane, S);
#ifdef RL_BASE_TWICE   // measurement only: the base pass's share of the descent
                base_pass<V, C, Mask, Skip>(s, mk, T, pc, lane, S);
#endif
                dirty = false;
            }
            C best;
            const PassResult r = scan_pass<V, C, Mask, Skip>(s, mk, T, pc, S, nbh, lane, best);
            st.evals += r.n_moves;
#ifdef RL_WALK_STATS
            if (lane == 0) {
                atomicAdd(&g_walk_stats[136 + nbh], 1ull);
                atomicAdd(&g_walk_stats[144 + nbh], (unsigned long long)r.improved);
                atomicAdd(&g_walk_stats[152 + nbh], (unsigned long long)r.n_moves);
            }
#endif
            if (r.improved) {
                const MoveDesc md = slot_move(mk, nbh, r.slot, T);
                ma = md.p1 >= 0 && md.p1 < md.p0 ? md.p1 : md.p0;
                mb = md.p1 > md.p0 ? md.p1 : md.p0;
                apply_slot(mk, nbh, r.slot, T, lane);
                dirty = true;
                improved = true;
                ++st.moves;
                if (trace_dec && lane == 0) {
                    if (st.sweeps < cap_sweeps)
                        atomicAdd(&trace_dec[(int64_t)st.sweeps * k_max + nbh - 1],
                                  (unsigned long long)(int64_t)(S - best));
                    else
                        atomicExch(overflow, 1);
                }
                S = best;
            }
        }
        ++st.sweeps;
        if (!improved)
            break;
    }
    for (int nbh = 1; nbh <= k_max; ++nbh)
        st.ntot += move_count(mk, nbh, T, lane);
    return true;
}

struct VndOut {
    int64_t *start_cost, *final_cost, *evals, *ntot;
    int32_t *sweeps, *moves;
    unsigned long long *trace_dec;   // [cap_sweeps * k_max]
    int64_t cap_sweeps;
    int *overflow;
    int *queue;              // products k_lo + atomicAdd(queue) < k_hi
    int64_t k_lo, k_hi;
};

// Persistent resident VND.  Every warp pulls products from a global queue
// and runs that product's VND to its own fixpoint (global VND decomposes
// exactly per product), logging each pass's decrease
// into trace_dec[sweep * k_max + nbh - 1] with exact int64 atomics so the
// reference's lockstep trace is reproduced.  A product's rows are staged by
// TMA into the warp's (then free) xc area.
// CTAs per SM the register allocation must allow (measured):
// int32 register-mask variant 7 x 4 warps per SM; shared-memory-mask
// variants 6 (int32 costs) and 4 (int64 costs: 13.9 KB shared per warp at
// T = 520 allows no more).
template <typename V, typename C, typename Mask> struct VndMinBlocks { static constexpr int value = 1; };
#ifndef RL_REG_MINB
#define RL_REG_MINB 7
#endif
template <> struct VndMinBlocks<int32_t, int32_t, MaskReg> { static constexpr int value = RL_REG_MINB; };
#ifndef RL_SMEM_MINB
#define RL_SMEM_MINB 4
#endif
#ifndef RL_SMEM32_MINB
#define RL_SMEM32_MINB 6
#endif
template <> struct VndMinBlocks<int32_t, int64_t, MaskSmem> { static constexpr int value = RL_SMEM_MINB; };
template <> struct VndMinBlocks<int32_t, int32_t, MaskSmem> { static constexpr int value = RL_SMEM32_MINB; };
#ifndef RL_SMEM16_MINB
#define RL_SMEM16_MINB 5   // 16-bit rows: 9.8 KB shared per warp at T = 520
#endif
#ifndef RL_REG_SKIP_MINB
#define RL_REG_SKIP_MINB 6   // latency-bound launches (slack skip): more registers, measured C2 -4%
#endif
#ifdef RL_VND_MINB
#define RL_VND_MINB_OF(V, C, M, SB, SKIP) RL_VND_MINB
#else
#define RL_VND_MINB_OF(V, C, M, SB, SKIP)                                                      \
    (SB == 2 ? RL_SMEM16_MINB                                                                \
     : (SKIP && VndMinBlocks<V, C, M>::value == RL_REG_MINB) ? RL_REG_SKIP_MINB            \
                                                              : VndMinBlocks<V, C, M>::value)
#endif
template <typename V, typename C, typename Mask, bool Skip, int SB = (int)sizeof(V)>
__global__ void __launch_bounds__(128, RL_VND_MINB_OF(V, C, Mask, SB, Skip)) k_vnd(InstView<V> in, const uint8_t *sm_in,
                                             const uint8_t *sr_in, uint8_t *sm_out,
                                             uint8_t *sr_out, int k_max, VndOut o)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = in.T;
    Slot<V, C, SB> s = carve<V, C, SB>(smem + warp * slot_bytes<V, C, SB>(T), T);
    if (lane == 0)
        mbar_init(s.bar);
    __syncwarp();
    uint32_t phase = 0;

    int64_t k = 0;
    if (lane == 0)
        k = o.k_lo + atomicAdd(o.queue, 1);
    k = __shfl_sync(FULL, k, 0);
    while (k < o.k_hi) {
        // the stage aliases xc (free between products): no prefetch; the
        // copy's latency is hidden by the other resident warps
        stage_begin(s, in, k, lane);
        const ProductCosts<C> pc = load_costs<C>(in.cost6, in.K, k, in.T, in.one);
        Mask mk = load_rows(s, Mask{}, sm_in, sr_in, k, T, lane);
        stage_end(s, in, k, lane, phase);
        const C K0 = build_prefix(s, T, pc, lane);
        int64_t next = 0;
        if (lane == 0)
            next = o.k_lo + atomicAdd(o.queue, 1);
        next = __shfl_sync(FULL, next, 0);

        C S, S0;
        VndStats st;
        const bool feas = vnd_product<V, C, Mask, Skip>(s, mk, T, pc, k_max, lane, S0, S, st, o.trace_dec,
                                      o.cap_sweeps, o.overflow);
        store_rows(mk, sm_out, sr_out, k, T, lane);
        if (lane == 0) {
            o.start_cost[k] = feas ? (int64_t)(K0 + S0) : RL_INFEASIBLE;
            o.final_cost[k] = feas ? (int64_t)(K0 + S) : RL_INFEASIBLE;
            o.evals[k] = st.evals;
            o.ntot[k] = st.ntot;
            o.sweeps[k] = st.sweeps;
            o.moves[k] = st.moves;
        }
        __syncwarp();
        k = next;
    }
}

// Long horizons (T > 63): one CTA of kWarpsPerCta warps per product.  A pass
// has ~2T moves, so the walks are split over all warps (move i goes to warp
// i mod 4; each lane still sees its moves in slot order) and the per-warp
// minima are combined in shared memory.  Warp 0 does the inherently
// per-product steps (staging, base pass, enumeration, apply) -- the same
// device functions as k_vnd, so results are identical.
template <typename V, typename C>
__global__ void __launch_bounds__(128) k_vnd_cta(InstView<V> in, const uint8_t *sm_in,
                                                 const uint8_t *sr_in, uint8_t *sm_out,
                                                 uint8_t *sr_out, int k_max, VndOut o)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ C part_best[kWarpsPerCta];
    __shared__ int part_key[kWarpsPerCta];
    __shared__ int64_t sh_k, sh_next;
    __shared__ C sh_S, sh_best;
    __shared__ int sh_n, sh_key, sh_feas;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = in.T;
    const Slot<V, C> s = carve<V, C>(smem, T);
    const MaskSmem mk{s.bm, s.br, s.bs, s.nx, T};
    if (threadIdx.x == 0) {
        mbar_init(s.bar);
        sh_k = o.k_lo + atomicAdd(o.queue, 1);
    }
    __syncthreads();
    uint32_t phase = 0;
    while (sh_k < o.k_hi) {
        const int64_t k = sh_k;
        const ProductCosts<C> pc = load_costs<C>(in.cost6, in.K, k, in.T, in.one);
        C K0 = 0;
        if (warp == 0) {
            stage_begin(s, in, k, lane);   // stage aliases xc: no prefetch
            load_rows(s, MaskSmem{}, sm_in, sr_in, k, T, lane);
            stage_end(s, in, k, lane, phase);
            K0 = build_prefix(s, T, pc, lane);
            int64_t nx = 0;
            if (lane == 0)
                nx = o.k_lo + atomicAdd(o.queue, 1);
            nx = __shfl_sync(FULL, nx, 0);
            C S;
            const bool f = base_pass<V, C, MaskSmem, false>(s, mk, T, pc, lane, S);
            if (lane == 0) {
                sh_next = nx;
                sh_S = S;
                sh_feas = f;
            }
        }
        __syncthreads();
        const bool feas = sh_feas;
        const C S0 = sh_S;
        C S = S0;
        int64_t evals = 0;
        int sweeps = 0, moves = 0, ntot = 0;
        if (feas) {
            bool dirty = false;
            int ma = 0, mb = 0;   // the applied move's periods (warp 0)
            for (;;) {
                bool improved = false;
                for (int nbh = 1; nbh <= k_max; ++nbh) {
                    if (warp == 0) {
                        if (dirty) {
#ifndef RL_NO_REBASE
                            rebase_smem<V, C, (int)sizeof(V)>(s, mk, T, pc, lane, S, ma, mb);
#else
                            base_pass<V, C, MaskSmem, false>(s, mk, T, pc, lane, S);
#endif
                        }
                        const int n = enumerate_moves(s, mk, nbh, T, lane);
                        if (lane == 0) {
                            sh_n = n;
                            sh_S = S;
                        }
                    }
                    __syncthreads();
                    const int n = sh_n;
                    S = sh_S;
                    C best = S;
                    int key = 0x7fffffff;
                    walk_moves<V, C, MaskSmem, false>(s, mk, T, pc, S, nbh, n, lane, warp,
                                                      kWarpsPerCta, best, key);
                    warp_argmin(best, key);
                    if (lane == 0) {
                        part_best[warp] = best;
                        part_key[warp] = key;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        C b = lane < kWarpsPerCta ? part_best[lane] : S;
                        int kk = lane < kWarpsPerCta ? part_key[lane] : 0x7fffffff;
                        warp_argmin(b, kk);
                        if (kk != 0x7fffffff) {
                            MaskSmem mw = mk;
                            const MoveDesc md = slot_move(mw, nbh, kk, T);
                            ma = md.p1 >= 0 && md.p1 < md.p0 ? md.p1 : md.p0;
                            mb = md.p1 > md.p0 ? md.p1 : md.p0;
                            apply_slot(mw, nbh, kk, T, lane);
                            if (lane == 0) {
                                if (sweeps < o.cap_sweeps)
                                    atomicAdd(&o.trace_dec[(int64_t)sweeps * k_max + nbh - 1],
                                              (unsigned long long)(int64_t)(S - b));
                                else
                                    atomicExch(o.overflow, 1);
                            }
                        }
                        if (lane == 0) {
                            sh_key = kk;
                            sh_best = b;
                        }
                    }
                    __syncthreads();
                    evals += n;
                    if (sh_key != 0x7fffffff) {
                        S = sh_best;
                        dirty = true;
                        improved = true;
                        ++moves;
                    }
                }
                ++sweeps;
                if (!improved)
                    break;
            }
            if (warp == 0)
                for (int nbh = 1; nbh <= k_max; ++nbh)
                    ntot += move_count(mk, nbh, T, lane);
        } else {
            sweeps = 1;
        }
        if (warp == 0) {
            store_rows(mk, sm_out, sr_out, k, T, lane);
            if (lane == 0) {
                o.start_cost[k] = feas ? (int64_t)(K0 + S0) : RL_INFEASIBLE;
                o.final_cost[k] = feas ? (int64_t)(K0 + S) : RL_INFEASIBLE;
                o.evals[k] = evals;
                o.ntot[k] = ntot;
                o.sweeps[k] = sweeps;
                o.moves[k] = moves;
                sh_k = sh_next;
            }
        }
        __syncthreads();
    }
}

#include "lane_vnd.cuh"

// Totals (one block).  summary: 0 final, 1 start, 2 sweeps, 3 evals done,
// 4 reference-equivalent evals, 5 moves, 6 K, 8 overflow, 9 sum of decreases.
__global__ void k_vnd_finalize(int64_t K, VndOut o, int64_t *summary)
{
    __shared__ long long s_sum[8][32];
    long long start = 0, dec = 0, ev = 0, sw_nt = 0, nt = 0, mv = 0, inf = 0, smax = 0;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const int64_t sc = o.start_cost[k];
        if (sc == RL_INFEASIBLE) {
            inf = 1;
        } else {
            start += sc;
            dec += sc - o.final_cost[k];
        }
        ev += o.evals[k];
        sw_nt += (long long)o.sweeps[k] * o.ntot[k];
        nt += o.ntot[k];
        mv += o.moves[k];
        smax = max(smax, (long long)o.sweeps[k]);
    }
    long long v[8] = {start, dec, ev, sw_nt, nt, mv, inf, smax};
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = 0; i < 8; ++i) {
        long long x = v[i];
        for (int off = 16; off; off >>= 1) {
            long long y = __shfl_xor_sync(FULL, x, off);
            x = (i >= 6) ? max(x, y) : x + y;
        }
        if (lane == 0)
            s_sum[i][w] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < (int)(blockDim.x >> 5); ++j)
                r[i] = (i >= 6) ? max(r[i], s_sum[i][j]) : r[i] + s_sum[i][j];
        const long long S = K > 0 ? r[7] : 0;
        const long long start_total = r[6] ? RL_INFEASIBLE : r[0];
        summary[0] = start_total - r[1];
        summary[1] = start_total;
        summary[2] = S;
        summary[3] = r[2];
        summary[4] = r[2] + S * r[4] - r[3];
        summary[5] = r[5];
        summary[6] = K;
        summary[8] = *o.overflow;
        summary[9] = r[1];
        summary[10] = r[4];
    }
}

__global__ void k_apply_scan(int64_t T, int64_t lo, int64_t hi, const int64_t *dec,
                             const int64_t *p0, const uint8_t *m0, const uint8_t *r0,
                             const int64_t *p1, const uint8_t *m1, const uint8_t *r1, uint8_t *sm,
                             uint8_t *sr, unsigned long long *diff)
{
    const int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= hi || dec[k] <= 0)
        return;
    sm[k * T + p0[k]] = m0[k];
    sr[k * T + p0[k]] = r0[k];
    if (p1[k] >= 0) {
        sm[k * T + p1[k]] = m1[k];
        sr[k * T + p1[k]] = r1[k];
    }
    atomicAdd(diff, (unsigned long long)dec[k]);
}

// plan.initial_solution (plan.py:140-167): recoverable stock a_t follows
// a_t = max(a_{t-1} + R[t] - D[t], 0) on demand periods.
template <typename V>
__global__ void k_initial(InstView<V> in, uint8_t *sm, uint8_t *sr)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= in.K)
        return;
    const int T = in.T;
    const V *d = in.dem + k * T, *r = in.ret + k * T;
    uint8_t *a = sm + k * T, *b = sr + k * T;
    V avail = 0;
    for (int t = 0; t < T; ++t) {
        avail += r[t];
        const V dt = d[t];
        uint8_t fm = 0, fr = 0;
        if (dt > 0) {
            const V take = avail < dt ? avail : dt;
            if (take > 0) {
                fr = 1;
                avail -= take;
            }
            fm = dt - take > 0;
        }
        a[t] = fm;
        b[t] = fr;
    }
}

// plan.decode / _kernels.row_decode (_kernels.py:100-168): quantities and
// stocks per period, rows zeroed when infeasible.  One thread per product
// (not on the VND hot loop).
template <typename V>
__global__ void k_decode(InstView<V> in, const uint8_t *sm, const uint8_t *sr, int64_t *xm_o,
                         int64_t *xr_o, int64_t *ym_o, int64_t *yr_o, int64_t *cost_o)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= in.K)
        return;
    const int T = in.T;
    const V *d = in.dem + k * T, *r = in.ret + k * T;
    const uint8_t *a = sm + k * T, *b = sr + k * T;
    int64_t *XM = xm_o + k * T, *XR = xr_o + k * T, *YM = ym_o + k * T, *YR = yr_o + k * T;
    const int64_t *c6 = in.cost6;
    const int64_t K = in.K;
    const int64_t km = c6[k], kr = c6[K + k], hm = c6[2 * K + k], hr = c6[3 * K + k],
                  pm = c6[4 * K + k], pr = c6[5 * K + k];
    int64_t cost = 0, rec = 0, stock = 0;
    bool ok = true;
    int t = 0;
    for (; t < T && !(a[t] | b[t]); ++t) {
        XM[t] = XR[t] = YM[t] = 0;
        if (d[t] > 0)
            ok = false;
        rec += r[t];
        YR[t] = rec;
        cost += hr * rec;
    }
    while (ok && t < T) {
        int u = t, v = t + 1;
        while (v < T && !(a[v] | b[v]))
            ++v;
        int64_t need = 0;
        for (int i = u; i < v; ++i)
            need += d[i];
        const int64_t have = rec + r[u];
        const int64_t take = b[u] ? (need < have ? need : have) : 0;
        const int64_t make = need - take;
        if (make > 0 && !a[u]) {
            ok = false;
            break;
        }
        cost += (take > 0 ? kr : 0) + (make > 0 ? km : 0) + pr * take + pm * make;
        for (int i = u; i < v; ++i) {
            XM[i] = i == u ? make : 0;
            XR[i] = i == u ? take : 0;
            if (i == u) {
                stock += make + take;
                rec += r[i] - take;
            } else {
                rec += r[i];
            }
            stock -= d[i];
            YM[i] = stock;
            YR[i] = rec;
            cost += hm * stock + hr * rec;
        }
        t = v;
    }
    if (!ok) {
        for (int i = 0; i < T; ++i)
            XM[i] = XR[i] = YM[i] = YR[i] = 0;
        cost = RL_INFEASIBLE;
    }
    cost_o[k] = cost;
}

__global__ void k_list_moves(int nbh, int T, const uint8_t *sm, const uint8_t *sr, int64_t *mp0,
                             uint8_t *mm0, uint8_t *mr0, int64_t *mp1, uint8_t *mm1, uint8_t *mr1,
                             int64_t *count)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    Slot<int32_t, int32_t> s = carve<int32_t, int32_t>(smem, T);
    const MaskSmem mk = load_rows(s, MaskSmem{}, sm, sr, 0, T, lane);
    const int nslots = nbh == 3 ? 4 * T : T;
    int n = 0;
    for (int base = 0; base < nslots; base += 32) {
        const int slot = base + lane;
        const bool ok = slot < nslots && slot_valid(mk, nbh, slot, T);
        const uint32_t bal = __ballot_sync(FULL, ok);
        if (ok) {
            const int i = n + __popc(bal & ((1u << lane) - 1));
            const MoveDesc d = slot_move(mk, nbh, slot, T);
            mp0[i] = d.p0;
            mm0[i] = d.m0;
            mr0[i] = d.r0;
            mp1[i] = d.p1;
            mm1[i] = d.m1;
            mr1[i] = d.r1;
        }
        n += __popc(bal);
    }
    if (lane == 0)
        *count = n;
}

// ------------------------------------------------------------------ handle

#ifndef RL_E2E_CHUNKS
#define RL_E2E_CHUNKS 3   // measured at C3 (geometric, ratio 2): 2 / 3 / 4 / 6 / 8 chunks
#endif                    // 17.93 / 17.62 / 17.90 / 18.14 / 18.57 ms per e2e step
constexpr int kMaxChunks = RL_E2E_CHUNKS;   // rl_vnd_host pipeline depth (<= 12: h->ints)

struct rl_instance {
    int64_t K = 0;
    int T = 0, vbytes = 8, cbytes = 8, device = 0, sms = 0;
    int smem_optin = 48 * 1024;            // max dynamic shared memory per CTA (opt-in)
    cudaStream_t stream = nullptr, stream2 = nullptr, stream3 = nullptr;
    cudaEvent_t evc[kMaxChunks + 2] = {};   // rl_vnd_host: chunk copies landed, joins
    int64_t *dem64 = nullptr, *ret64 = nullptr, *cost6 = nullptr;
    void *dem = nullptr, *ret = nullptr;   // V typed (alias dem64/ret64 when V = int64)
    uint8_t *plan = nullptr;               // 4 x K x T: sm_in, sr_in, sm_out, sr_out
    int64_t *p64 = nullptr;                // 4 x K: start, final, evals, ntot
    int32_t *p32 = nullptr;                // 2 x K: sweeps, moves
    unsigned long long *trace_dec = nullptr;
    int64_t cap_sweeps = 0;
    int *ints = nullptr;                   // queue, overflow, negative
    int64_t *summary = nullptr;            // 16
    unsigned long long *bounds = nullptr;  // 2 (double bits) + scan evals at [2]
    int64_t *scan_i64 = nullptr;           // 3 x K: dec, p0, p1
    uint8_t *scan_u8 = nullptr;            // 4 x K
    int64_t launches = 0;
    int last_kmax = 4;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timing = false;
    cudaEvent_t done = nullptr;            // recorded after k_vnd_finalize (rl_vnd_collect waits on it)
    mutable std::recursive_mutex mu;       // RL_GUARD
    struct GvnsState *gv = nullptr;        // device GVNS state (gvns_impl.cuh)
    double cost_bound = 0.0;               // upper bound of any plan's cost (upload)
    bool cta_long = true;                  // T > 63, few products: CTA per product (k_vnd_cta)
    int skip_mode = 0;                     // slack skip: 0 auto, 1 always, 2 never (A/B)
    bool force64 = false;                  // variant bit 4: int64 values and costs (A/B)
    int lane_mode = 0;                     // lane-per-product kernel: 2 = use it (variant bit 6)
    int lane_refill = RL_LANE_REFILL_MIN;  // idle lanes that trigger its control step
    double sdr_max = 0.0;                  // max over products of sum D + sum R
    bool p16 = false;                      // every product's sum D, sum R < 2^16
    bool no16 = false;                     // variant bit 7: never the 16-bit rows (A/B)
    bool cta_always = false;               // variant bit 8: CTA per product for T > 63 (A/B)
};

struct GvnsState;
static void gvns_free(GvnsState *gs);

static int ensure_trace(rl_instance *h, int64_t cap_sweeps, int k_max)
{
    if (h->trace_dec && h->cap_sweeps >= cap_sweeps)
        return 0;
    if (h->trace_dec)
        CK(cudaFree(h->trace_dec));
    h->trace_dec = nullptr;
    CK(cudaMalloc(&h->trace_dec, (size_t)cap_sweeps * 4 * sizeof(unsigned long long)));
    h->cap_sweeps = cap_sweeps;
    (void)k_max;
    return 0;
}

// Range check + exact-width selection + narrowing of the int64 rows already
// in dem64/ret64/cost6 (the device half of an upload).
static int prepare(rl_instance *h)
{
    const size_t kt = (size_t)h->K * h->T;
    CK(cudaMemsetAsync(h->bounds, 0, 6 * sizeof(unsigned long long), h->stream));
    CK(cudaMemsetAsync(h->ints, 0, 4 * sizeof(int), h->stream));
    const int blk = 256;
    k_bounds<<<(unsigned)((h->K + blk - 1) / blk), blk, 0, h->stream>>>(
        h->K, h->T, h->dem64, h->ret64, h->cost6, h->bounds, h->bounds + 3, h->ints + 2,
        h->bounds + 4);
    CKL();
    unsigned long long hb[6];
    int neg = 0;
    CK(cudaMemcpyAsync(hb, h->bounds, sizeof hb, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(&neg, h->ints + 2, sizeof neg, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    double sdr, B, Q;
    memcpy(&sdr, &hb[0], 8);
    memcpy(&B, &hb[1], 8);
    memcpy(&Q, &hb[3], 8);
    if (neg)
        return fail(RL_ERANGE, "instance has negative entries (validate_instance rejects them)");
    if (!(sdr < std::ldexp(1.0, 60)) || !(B < std::ldexp(1.0, 61)))
        return fail(RL_ERANGE,
                    "instance too large for exact int64 costs (max sum D+R %.3g, cost bound %.3g)",
                    sdr, B);
    h->cost_bound = B;
    h->sdr_max = sdr;
    {
        double sdm, srm;
        memcpy(&sdm, &hb[4], 8);
        memcpy(&srm, &hb[5], 8);
        h->p16 = sdm < 65536.0 && srm < 65536.0;
    }
    // new instance data: the device GVNS state (F, Fcost, the captured batch
    // graph and shake scratch sized for the old widths) is stale
    gvns_free(h->gv);
    h->gv = nullptr;
    // int32 values only with int32 coefficients (seg_cost<int32, int64>
    // multiplies 32 x 32 -> 64); int32 costs when every plan's cost fits
    const int vbytes =
        !h->force64 && sdr < std::ldexp(1.0, 28) && Q < std::ldexp(1.0, 30) ? 4 : 8;
    const int cbytes = (vbytes == 4 && B < std::ldexp(1.0, 30)) ? 4 : 8;
    if (h->dem && h->vbytes == 4 && vbytes != 4) {
        CK(cudaFree(h->dem));
        h->dem = h->ret = nullptr;
    }
    h->vbytes = vbytes;
    h->cbytes = cbytes;
    if (vbytes == 4) {
        if (!h->dem || h->dem == h->dem64) {
            void *p;
            CK(cudaMalloc(&p, kt * 2 * 4));
            h->dem = p;
            h->ret = (int32_t *)p + kt;
        }
        k_narrow<int32_t><<<h->sms * 4, 256, 0, h->stream>>>(kt, h->dem64, (int32_t *)h->dem);
        CKL();
        k_narrow<int32_t><<<h->sms * 4, 256, 0, h->stream>>>(kt, h->ret64, (int32_t *)h->ret);
        CKL();
    } else {
        h->dem = h->dem64;
        h->ret = h->ret64;
    }
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

static int upload(rl_instance *h, const int64_t *demand, const int64_t *returns,
                  const int64_t *const cost[6])
{
    const size_t kt = (size_t)h->K * h->T;
    CK(cudaMemcpyAsync(h->dem64, demand, kt * 8, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->ret64, returns, kt * 8, cudaMemcpyHostToDevice, h->stream));
    for (int i = 0; i < 6; ++i)
        CK(cudaMemcpyAsync(h->cost6 + i * h->K, cost[i], h->K * 8, cudaMemcpyHostToDevice,
                           h->stream));
    return prepare(h);
}

// Streams, events and every K x T / K buffer of a handle (h->K, h->T set).
static int alloc_instance(rl_instance *h)
{
    const int64_t K = h->K;
    const size_t kt = (size_t)K * h->T;
    cudaError_t e = cudaGetDevice(&h->device);
    if (e != cudaSuccess)
        return fail(RL_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
    e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device);
    if (e == cudaSuccess)
        e = cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                   h->device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream3, cudaStreamNonBlocking);
    for (auto &ev : h->evc)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&h->dem64, kt * 8 * 2);
    if (e == cudaSuccess) {
        h->ret64 = h->dem64 + kt;
        e = cudaMalloc(&h->cost6, K * 8 * 6);
    }
    if (e == cudaSuccess) e = cudaMalloc(&h->plan, kt * 4);
    if (e == cudaSuccess) e = cudaMalloc(&h->p64, K * 8 * 4);
    if (e == cudaSuccess) e = cudaMalloc(&h->p32, K * 4 * 2);
    if (e == cudaSuccess) e = cudaMalloc(&h->ints, 16 * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&h->summary, 16 * 8);
    if (e == cudaSuccess) e = cudaMalloc(&h->bounds, 8 * 8);
    if (e == cudaSuccess) e = cudaMalloc(&h->scan_i64, K * 8 * 3);
    if (e == cudaSuccess) e = cudaMalloc(&h->scan_u8, K * 4);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming);
    if (e != cudaSuccess)
        return fail(RL_ECUDA, "rl_instance_create: %s", cudaGetErrorString(e));
    return ensure_trace(h, 1024, 4);
}

static int finish_create(rl_instance *h, int rc, rl_instance **out)
{
    if (rc) {
        std::string keep = g_err;
        rl_instance_destroy(h);
        g_err = keep;
        return rc;
    }
    *out = h;
    return 0;
}

extern "C" int rl_instance_create(int64_t K, int64_t T, const int64_t *demand,
                                  const int64_t *returns, const int64_t *setup_m,
                                  const int64_t *setup_r, const int64_t *hold_m,
                                  const int64_t *hold_r, const int64_t *unit_m,
                                  const int64_t *unit_r, rl_instance **out)
{
    if (!out || K < 1 || T < 1 || T > 16000 || !demand || !returns || !setup_m || !setup_r ||
        !hold_m || !hold_r || !unit_m || !unit_r)
        return fail(RL_EINVAL, "rl_instance_create: bad arguments (K=%lld, T=%lld)",
                    (long long)K, (long long)T);
    *out = nullptr;
    rl_instance *h = new rl_instance();
    h->K = K;
    h->T = (int)T;
    if (const char *e = getenv("RL_LANE_REFILL"))   // A/B of the lane kernel's refill batch
        h->lane_refill = atoi(e) > 0 ? atoi(e) : h->lane_refill;
    int rc = alloc_instance(h);
    if (!rc) {
        const int64_t *cost[6] = {setup_m, setup_r, hold_m, hold_r, unit_m, unit_r};
        rc = upload(h, demand, returns, cost);
    }
    return finish_create(h, rc, out);
}

extern "C" int rl_instance_update(rl_instance *h, const int64_t *demand, const int64_t *returns,
                                  const int64_t *setup_m, const int64_t *setup_r,
                                  const int64_t *hold_m, const int64_t *hold_r,
                                  const int64_t *unit_m, const int64_t *unit_r)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !demand || !returns || !setup_m || !setup_r || !hold_m || !hold_r || !unit_m ||
        !unit_r)
        return fail(RL_EINVAL, "rl_instance_update: bad arguments");
    CK(cudaSetDevice(h->device));
    const int64_t *cost[6] = {setup_m, setup_r, hold_m, hold_r, unit_m, unit_r};
    return upload(h, demand, returns, cost);
}

extern "C" void rl_instance_destroy(rl_instance *h)
{
    if (!h)
        return;
    cudaSetDevice(h->device);
    if (h->stream)
        cudaStreamSynchronize(h->stream);
    if (h->dem && h->dem != h->dem64)
        cudaFree(h->dem);
    void *ptrs[] = {h->dem64, h->cost6, h->plan, h->p64, h->p32, h->trace_dec,
                    h->ints, h->summary, h->bounds, h->scan_i64, h->scan_u8};
    for (void *p : ptrs)
        if (p)
            cudaFree(p);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->done) cudaEventDestroy(h->done);
    if (h->stream)
        cudaStreamDestroy(h->stream);
    if (h->stream2)
        cudaStreamDestroy(h->stream2);
    if (h->stream3)
        cudaStreamDestroy(h->stream3);
    for (auto ev : h->evc)
        if (ev)
            cudaEventDestroy(ev);
    gvns_free(h->gv);
    delete h;
}


// Warp-per-product kernels: kWarpsPerCta warps (one shared-memory slot each)
// per CTA, fewer when a long horizon's slots do not fit one CTA's opt-in
// shared memory.  Returns the block size in `block`.
template <typename V, typename C, int SB = (int)sizeof(V)>
static int launch_cfg(rl_instance *h, const void *fn, int64_t nprod, int &grid, size_t &smem,
                      int &block)
{
    const size_t slot = slot_bytes<V, C, SB>(h->T);
    int nw = kWarpsPerCta;
    while (nw > 1 && (size_t)nw * slot > (size_t)h->smem_optin)
        --nw;
    smem = nw * slot;
    if (smem > (size_t)h->smem_optin)
        return fail(RL_EINVAL, "T=%d needs %zu B shared memory per product (max %d)", h->T,
                    slot, h->smem_optin);
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nw * 32, smem));
    if (occ < 1)
        return fail(RL_EINVAL, "T=%d needs %zu B shared memory per CTA", h->T, smem);
    const int64_t want = (nprod + nw - 1) / nw;
    const int64_t cap = (int64_t)h->sms * occ;
    grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
    block = nw * 32;
    return 0;
}

template <typename V, typename C>
static int launch_cfg_cta(rl_instance *h, const void *fn, int64_t nprod, int &grid, size_t &smem)
{
    smem = slot_bytes<V, C>(h->T);
    if (smem > (size_t)h->smem_optin)
        return fail(RL_EINVAL, "T=%d needs %zu B shared memory per product (max %d)", h->T,
                    smem, h->smem_optin);
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kWarpsPerCta * 32, smem));
    if (occ < 1)
        return fail(RL_EINVAL, "T=%d needs %zu B shared memory per CTA", h->T, smem);
    const int64_t cap = (int64_t)h->sms * occ;
    grid = (int)(nprod < cap ? (nprod > 0 ? nprod : 1) : cap);
    return 0;
}

extern "C" int rl_instance_set_variant(rl_instance *h, int variant)
{
    RL_GUARD(h);
    // bit 0 (two products per warp) was removed: measured slower
    if (!h || variant < 0 || variant > 511 || (variant & 12) == 12 || (variant & 1) ||
        (variant & 96) == 96)
        return fail(RL_EINVAL, "rl_instance_set_variant: bad arguments");
    h->lane_mode = (variant & 32) ? 1 : (variant & 64) ? 2 : 0;
    h->no16 = (variant & 128) != 0;
    h->cta_always = (variant & 256) != 0;
    h->cta_long = (variant & 2) == 0;
    h->skip_mode = (variant & 4) ? 1 : (variant & 8) ? 2 : 0;
    const bool f64 = (variant & 16) != 0;
    if (f64 != h->force64) {   // re-pick the widths from the resident int64 rows
        CK(cudaSetDevice(h->device));
        h->force64 = f64;
        return prepare(h);
    }
    return 0;
}

extern "C" int rl_instance_info(const rl_instance *h, int64_t *info)
{
    RL_GUARD(h);
    if (!h || !info)
        return fail(RL_EINVAL, "rl_instance_info: bad arguments");
    info[0] = h->K;
    info[1] = h->T;
    info[2] = h->vbytes;
    info[3] = h->cbytes;
    info[4] = h->sms;
    info[5] = kWarpsPerCta;
    return 0;
}

template <typename V>
static InstView<V> view(rl_instance *h)
{
    InstView<V> v;
    v.K = h->K;
    v.T = h->T;
    v.dem = (const V *)h->dem;
    v.ret = (const V *)h->ret;
    v.cost6 = h->cost6;
    v.one = 1;
    return v;
}

// dispatch on the exact narrow types chosen at upload
#define RL_DISPATCH(h, FN, ...)                                         \
    ((h)->vbytes == 4 && (h)->cbytes == 4 ? FN<int32_t, int32_t>(__VA_ARGS__) \
     : (h)->vbytes == 4                   ? FN<int32_t, int64_t>(__VA_ARGS__) \
                                          : FN<int64_t, int64_t>(__VA_ARGS__))

// ... and on where the setup rows live (registers for T <= 63)
#define RL_DISPATCH_M(h, FN, ...)                                                        \
    ((h)->T <= 63                                                                        \
         ? ((h)->vbytes == 4 && (h)->cbytes == 4 ? FN<int32_t, int32_t, MaskReg>(__VA_ARGS__)  \
            : (h)->vbytes == 4                   ? FN<int32_t, int64_t, MaskReg>(__VA_ARGS__)  \
                                                 : FN<int64_t, int64_t, MaskReg>(__VA_ARGS__)) \
         : ((h)->vbytes == 4 && (h)->cbytes == 4 ? FN<int32_t, int32_t, MaskSmem>(__VA_ARGS__) \
            : (h)->vbytes == 4                   ? FN<int32_t, int64_t, MaskSmem>(__VA_ARGS__) \
                                                 : FN<int64_t, int64_t, MaskSmem>(__VA_ARGS__)))

static int check_range(rl_instance *h, int64_t lo, int64_t hi)
{
    if (!h)
        return fail(RL_EINVAL, "null handle");
    if (lo < 0 || hi > h->K || lo > hi)
        return fail(RL_EINVAL, "product range [%lld, %lld) outside 0..%lld", (long long)lo,
                    (long long)hi, (long long)h->K);
    return 0;
}

template <typename V, typename C, typename Mask>
static int do_costs(rl_instance *h, int64_t lo, int64_t hi, int64_t *d_out)
{
    int grid;
    size_t smem;
    int block;
    int rc = launch_cfg<V, C>(h, (const void *)k_product_costs<V, C, Mask>, hi - lo, grid, smem,
                              block);
    if (rc)
        return rc;
    const size_t kt = (size_t)h->K * h->T;
    k_product_costs<V, C, Mask><<<grid, block, smem, h->stream>>>(
        view<V>(h), h->plan, h->plan + kt, lo, hi, d_out);
    CKL();
    return 0;
}

extern "C" int rl_product_costs(rl_instance *h, int64_t lo, int64_t hi, const uint8_t *sm,
                                const uint8_t *sr, int64_t *out)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    int rc = check_range(h, lo, hi);
    if (rc)
        return rc;
    if (!sm || !sr || !out)
        return fail(RL_EINVAL, "rl_product_costs: null buffer");
    if (hi == lo)
        return 0;
    CK(cudaSetDevice(h->device));
    const size_t kt = (size_t)h->K * h->T;
    CK(cudaMemcpyAsync(h->plan, sm, kt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->plan + kt, sr, kt, cudaMemcpyHostToDevice, h->stream));
    if ((rc = RL_DISPATCH_M(h, do_costs, h, lo, hi, h->p64)))
        return rc;
    CK(cudaMemcpyAsync(out + lo, h->p64 + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

template <typename V, typename C, typename Mask>
static int do_scan(rl_instance *h, int64_t lo, int64_t hi, int nbh)
{
    int grid;
    size_t smem;
    int block;
    int rc = launch_cfg<V, C>(h, (const void *)k_scan<V, C, Mask>, hi - lo, grid, smem, block);
    if (rc)
        return rc;
    const size_t kt = (size_t)h->K * h->T;
    const int64_t K = h->K;
    k_scan<V, C, Mask><<<grid, block, smem, h->stream>>>(
        view<V>(h), h->plan, h->plan + kt, lo, hi, nbh, h->scan_i64, h->scan_i64 + K,
        h->scan_u8, h->scan_u8 + K, h->scan_i64 + 2 * K, h->scan_u8 + 2 * K, h->scan_u8 + 3 * K,
        h->bounds + 2);
    CKL();
    return 0;
}

extern "C" int rl_scan_products(rl_instance *h, int64_t lo, int64_t hi, const uint8_t *sm,
                                const uint8_t *sr, int nbh, int64_t *dec, int64_t *p0,
                                uint8_t *m0, uint8_t *r0, int64_t *p1, uint8_t *m1, uint8_t *r1,
                                int64_t *evals)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    int rc = check_range(h, lo, hi);
    if (rc)
        return rc;
    if (nbh < 1 || nbh > 4)
        return fail(RL_EINVAL, "neighborhood id must be in 1..4, got %d", nbh);
    if (!sm || !sr || !dec || !p0 || !m0 || !r0 || !p1 || !m1 || !r1)
        return fail(RL_EINVAL, "rl_scan_products: null buffer");
    if (hi == lo) {
        if (evals)
            *evals = 0;
        return 0;
    }
    CK(cudaSetDevice(h->device));
    const size_t kt = (size_t)h->K * h->T;
    const int64_t K = h->K, n = hi - lo;
    CK(cudaMemcpyAsync(h->plan, sm, kt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->plan + kt, sr, kt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(h->bounds + 2, 0, 8, h->stream));
    if ((rc = RL_DISPATCH_M(h, do_scan, h, lo, hi, nbh)))
        return rc;
    int64_t *i64[3] = {dec, p0, p1};
    uint8_t *u8[4] = {m0, r0, m1, r1};
    for (int i = 0; i < 3; ++i)
        CK(cudaMemcpyAsync(i64[i] + lo, h->scan_i64 + i * K + lo, n * 8, cudaMemcpyDeviceToHost,
                           h->stream));
    for (int i = 0; i < 4; ++i)
        CK(cudaMemcpyAsync(u8[i] + lo, h->scan_u8 + i * K + lo, n, cudaMemcpyDeviceToHost,
                           h->stream));
    unsigned long long ev = 0;
    CK(cudaMemcpyAsync(&ev, h->bounds + 2, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (evals)
        *evals = (int64_t)ev;
    return 0;
}

extern "C" int rl_apply_scan(rl_instance *h, int64_t lo, int64_t hi, const int64_t *dec,
                             const int64_t *p0, const uint8_t *m0, const uint8_t *r0,
                             const int64_t *p1, const uint8_t *m1, const uint8_t *r1, uint8_t *sm,
                             uint8_t *sr, int64_t *diff)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    int rc = check_range(h, lo, hi);
    if (rc)
        return rc;
    if (!dec || !p0 || !m0 || !r0 || !p1 || !m1 || !r1 || !sm || !sr || !diff)
        return fail(RL_EINVAL, "rl_apply_scan: null buffer");
    CK(cudaSetDevice(h->device));
    const size_t kt = (size_t)h->K * h->T;
    const int64_t K = h->K;
    for (int64_t k = lo; k < hi; ++k)   // validate periods like the reference's indexing would
        if (dec[k] > 0 && (p0[k] < 0 || p0[k] >= h->T || p1[k] >= h->T))
            return fail(RL_EINVAL, "apply_scan: period out of range at product %lld",
                        (long long)k);
    const int64_t *i64[3] = {dec, p0, p1};
    const uint8_t *u8[4] = {m0, r0, m1, r1};
    for (int i = 0; i < 3; ++i)
        CK(cudaMemcpyAsync(h->scan_i64 + i * K, i64[i], K * 8, cudaMemcpyHostToDevice, h->stream));
    for (int i = 0; i < 4; ++i)
        CK(cudaMemcpyAsync(h->scan_u8 + i * K, u8[i], K, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->plan, sm, kt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->plan + kt, sr, kt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(h->bounds + 2, 0, 8, h->stream));
    if (hi > lo) {
        k_apply_scan<<<(unsigned)((hi - lo + 255) / 256), 256, 0, h->stream>>>(
            h->T, lo, hi, h->scan_i64, h->scan_i64 + K, h->scan_u8, h->scan_u8 + K,
            h->scan_i64 + 2 * K, h->scan_u8 + 2 * K, h->scan_u8 + 3 * K, h->plan, h->plan + kt,
            h->bounds + 2);
        CKL();
    }
    CK(cudaMemcpyAsync(sm, h->plan, kt, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(sr, h->plan + kt, kt, cudaMemcpyDeviceToHost, h->stream));
    unsigned long long d = 0;
    CK(cudaMemcpyAsync(&d, h->bounds + 2, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *diff = (int64_t)d;
    return 0;
}

static VndOut vnd_out(rl_instance *h, int64_t lo, int64_t hi, int *queue)
{
    const int64_t K = h->K;
    VndOut o;
    o.start_cost = h->p64;
    o.final_cost = h->p64 + K;
    o.evals = h->p64 + 2 * K;
    o.ntot = h->p64 + 3 * K;
    o.sweeps = h->p32;
    o.moves = h->p32 + K;
    o.trace_dec = h->trace_dec;
    o.cap_sweeps = h->cap_sweeps;
    o.overflow = h->ints + 1;
    o.queue = queue;
    o.k_lo = lo;
    o.k_hi = hi;
    return o;
}

// Launch the VND kernel variant for products [lo, hi) (queue reset by caller).
template <typename V, typename C, typename Mask>
static int launch_vnd_range(rl_instance *h, int k_max, const uint8_t *sm_in, const uint8_t *sr_in,
                            uint8_t *sm_out, uint8_t *sr_out, int64_t lo, int64_t hi, int *queue,
                            cudaStream_t st)
{
    int grid, block = kWarpsPerCta * 32;
    size_t smem;
    const int64_t nprod = hi - lo;
    // CTA per product only when the launch is latency-bound (few products):
    // at C4 scale one warp per product keeps 2.4x more products in flight
    // and measured 296 ms vs 434 ms
    const bool cta = std::is_same<Mask, MaskSmem>::value && h->cta_long &&
                     (nprod <= (int64_t)h->sms * 2 || h->cta_always);
    // skip pays when the launch is latency-bound: fewer products than ~2
    // waves of resident warps (C2, GVNS) -- measured, DESIGN.md section 5
    const bool skip = std::is_same<Mask, MaskReg>::value &&
                      (h->skip_mode == 1 || (h->skip_mode == 0 && nprod < (int64_t)h->sms * 64));
    // the slack skip exists for register rows only: Skip=true is never
    // instantiated for shared-memory rows
    constexpr bool kReg = std::is_same<Mask, MaskReg>::value;
    // 16-bit {cd, cr} / xin rows for long horizons when every product's sum D
    // and sum R < 2^16 (upload proof): 9.8 instead of 12.9 KB per warp at
    // T = 520, 5 instead of 4 CTAs per SM
    constexpr bool k16ok = !kReg && std::is_same<V, int32_t>::value &&
                           std::is_same<C, int64_t>::value;
    const bool p16 = k16ok && !cta && h->p16 && !h->no16;
    const void *fn = cta    ? (const void *)k_vnd_cta<V, C>
                     : p16  ? (const void *)k_vnd<V, C, Mask, false, k16ok ? 2 : (int)sizeof(V)>
                     : skip ? (const void *)k_vnd<V, C, Mask, kReg>
                            : (const void *)k_vnd<V, C, Mask, false>;
    int rc = cta ? launch_cfg_cta<V, C>(h, fn, nprod, grid, smem)
             : p16 ? launch_cfg<V, C, k16ok ? 2 : (int)sizeof(V)>(h, fn, nprod, grid, smem, block)
                   : launch_cfg<V, C>(h, fn, nprod, grid, smem, block);
    if (rc)
        return rc;
    const VndOut o = vnd_out(h, lo, hi, queue);
    // lane per product (T <= 63, variant bit 6 only): exact, but measured
    // slower than a warp per product at C3 (29 vs 18.8 ms: latency-bound at
    // the 13 warps/SM its shared memory allows, plus the tail of ~1.6
    // products per lane)
    if (std::is_same<Mask, MaskReg>::value && h->lane_mode == 2) {
        // 16-bit packed rows when every product's sum D + sum R < 2^15
        const bool packed = sizeof(V) == 4 && h->sdr_max < 32768.0;
        const void *fl = packed ? (const void *)k_vnd_lane<V, C, true>
                                : (const void *)k_vnd_lane<V, C, false>;
        const size_t lsm = packed ? lane_slot_bytes<V, C, true>(h->T)
                                  : lane_slot_bytes<V, C, false>(h->T);
        if (lsm > 48 * 1024)
            CK(cudaFuncSetAttribute(fl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fl, 32, lsm));
        if (occ > 0) {
            const int64_t want = (nprod + 31) / 32;
            int64_t cap = h->sms * (int64_t)occ;
            if (const char *e = getenv("RL_LANE_WARPS_PER_SM"))   // A/B: fewer lanes
                cap = atoi(e) > 0 && atoi(e) < occ ? (int64_t)h->sms * atoi(e) : cap;
            const int g = (int)(want < cap ? want : cap);
            if (packed)
                k_vnd_lane<V, C, true><<<g, 32, lsm, st>>>(view<V>(h), sm_in, sr_in, sm_out,
                                                          sr_out, k_max, o, h->lane_refill);
            else
                k_vnd_lane<V, C, false><<<g, 32, lsm, st>>>(view<V>(h), sm_in, sr_in, sm_out,
                                                           sr_out, k_max, o, h->lane_refill);
            CKL();
            return 0;
        }
    }
    if (cta)
        k_vnd_cta<V, C><<<grid, kWarpsPerCta * 32, smem, st>>>(view<V>(h), sm_in, sr_in, sm_out,
                                                                sr_out, k_max, o);
    else if (p16)
        k_vnd<V, C, Mask, false, k16ok ? 2 : (int)sizeof(V)><<<grid, block, smem, st>>>(
            view<V>(h), sm_in, sr_in, sm_out, sr_out, k_max, o);
    else if (skip)
        k_vnd<V, C, Mask, kReg><<<grid, block, smem, st>>>(view<V>(h), sm_in, sr_in,
                                                            sm_out, sr_out, k_max, o);
    else
        k_vnd<V, C, Mask, false><<<grid, block, smem, st>>>(view<V>(h), sm_in, sr_in,
                                                                         sm_out, sr_out, k_max, o);
    CKL();
    return 0;
}

template <typename V, typename C, typename Mask>
static int do_vnd(rl_instance *h, int k_max, const uint8_t *sm_in, const uint8_t *sr_in,
                  uint8_t *sm_out, uint8_t *sr_out, cudaStream_t st)
{
    CK(cudaMemsetAsync(h->ints, 0, 2 * sizeof(int), st));
    CK(cudaMemsetAsync(h->trace_dec, 0, (size_t)h->cap_sweeps * k_max * 8, st));
    CK(cudaEventRecord(h->ev0, st));
    int rc = launch_vnd_range<V, C, Mask>(h, k_max, sm_in, sr_in, sm_out, sr_out, 0, h->K,
                                          h->ints, st);
    if (rc)
        return rc;
    CK(cudaEventRecord(h->ev1, st));
    k_vnd_finalize<<<1, 1024, 0, st>>>(h->K, vnd_out(h, 0, h->K, h->ints), h->summary);
    CKL();
    CK(cudaEventRecord(h->done, st));
    return 0;
}

extern "C" int rl_vnd_device(rl_instance *h, int k_max, const uint8_t *d_sm_in,
                             const uint8_t *d_sr_in, uint8_t *d_sm_out, uint8_t *d_sr_out,
                             void *stream)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h)
        return fail(RL_EINVAL, "null handle");
    if (k_max < 1 || k_max > 4)
        return fail(RL_EINVAL, "k_max must be in 1..4, got %d", k_max);
    if (!d_sm_in || !d_sr_in || !d_sm_out || !d_sr_out)
        return fail(RL_EINVAL, "rl_vnd_device: null buffer");
    CK(cudaSetDevice(h->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
    h->last_kmax = k_max;
    return RL_DISPATCH_M(h, do_vnd, h, k_max, d_sm_in, d_sr_in, d_sm_out, d_sr_out, st);
}

extern "C" int rl_vnd_collect(rl_instance *h, int64_t *trace, int64_t trace_cap, int64_t *n_trace,
                              int64_t *stats)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !stats)
        return fail(RL_EINVAL, "rl_vnd_collect: bad arguments");
    CK(cudaSetDevice(h->device));
    // the descent may have been enqueued on a caller's stream: wait for its
    // finalize only (no device-wide sync: other handles keep running)
    CK(cudaEventSynchronize(h->done));
    int64_t sum[16];
    CK(cudaMemcpyAsync(sum, h->summary, sizeof sum, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    const int64_t S = sum[2];
    const int k_max = h->last_kmax;
    if (sum[8])
        return fail(RL_ERANGE, "trace overflow: more than %lld sweeps", (long long)h->cap_sweeps);
    const int64_t n = 1 + S * k_max;
    if (n_trace)
        *n_trace = n;
    if (trace && trace_cap > 0) {
        const int64_t m = (n - 1 < trace_cap - 1 ? n - 1 : trace_cap - 1);
        int64_t *dec = new int64_t[m > 0 ? m : 1];
        if (m > 0) {
            const cudaError_t e = cudaMemcpyAsync(dec, h->trace_dec, m * 8, cudaMemcpyDeviceToHost,
                                                  h->stream);
            const cudaError_t e2 = e == cudaSuccess ? cudaStreamSynchronize(h->stream) : e;
            if (e2 != cudaSuccess) {
                delete[] dec;
                return fail(RL_ECUDA, "rl_vnd_collect: %s", cudaGetErrorString(e2));
            }
        }
        trace[0] = sum[1];
        for (int64_t i = 0; i < m; ++i)
            trace[i + 1] = trace[i] - dec[i];
        delete[] dec;
    }
    stats[0] = sum[0];
    stats[1] = sum[1];
    stats[2] = S;
    stats[3] = sum[3];
    stats[4] = sum[4];
    stats[5] = sum[5];
    stats[6] = sum[6];
    stats[7] = (int64_t)((double)ms * 1e6);
    stats[8] = sum[10];
    return 0;
}

extern "C" int rl_vnd(rl_instance *h, int k_max, const uint8_t *sm_in, const uint8_t *sr_in,
                      uint8_t *sm_out, uint8_t *sr_out, int64_t *trace, int64_t trace_cap,
                      int64_t *n_trace, int64_t *stats)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h)
        return fail(RL_EINVAL, "null handle");
    if (!sm_in || !sr_in || !sm_out || !sr_out || !stats)
        return fail(RL_EINVAL, "rl_vnd: null buffer");
    CK(cudaSetDevice(h->device));
    const size_t kt = (size_t)h->K * h->T;
    CK(cudaMemcpyAsync(h->plan, sm_in, kt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->plan + kt, sr_in, kt, cudaMemcpyHostToDevice, h->stream));
    for (;;) {
        int rc = rl_vnd_device(h, k_max, h->plan, h->plan + kt, h->plan + 2 * kt,
                               h->plan + 3 * kt, h->stream);
        if (rc)
            return rc;
        rc = rl_vnd_collect(h, trace, trace_cap, n_trace, stats);
        if (rc == RL_ERANGE && h->cap_sweeps < (int64_t)1 << 26) {
            // more sweeps than the trace buffer holds: grow and rerun
            if ((rc = ensure_trace(h, h->cap_sweeps * 8, k_max)))
                return rc;
            continue;
        }
        if (rc)
            return rc;
        break;
    }
    CK(cudaMemcpyAsync(sm_out, h->plan + 2 * kt, kt, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(sr_out, h->plan + 3 * kt, kt, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

#ifdef RL_WALK_STATS
extern "C" int rl_lane_stats(int64_t *out, int reset)
{
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(out, g_lane_stats, sizeof(g_lane_stats)));
    if (reset) {
        static const unsigned long long z[16] = {};
        CK(cudaMemcpyToSymbol(g_lane_stats, z, sizeof z));
    }
    return 0;
}

extern "C" int rl_walk_stats(int64_t *out, int reset)
{
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(out, g_walk_stats, sizeof(g_walk_stats)));
    if (reset) {
        static const unsigned long long z[160] = {};
        CK(cudaMemcpyToSymbol(g_walk_stats, z, sizeof z));
    }
    return 0;
}
#endif

// Per-product results of the last rl_vnd / rl_vnd_device on this handle
// (diagnostics: work distribution over products).
extern "C" int rl_vnd_product_stats(rl_instance *h, int32_t *sweeps, int32_t *moves,
                                    int64_t *evals)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !sweeps || !moves || !evals)
        return fail(RL_EINVAL, "rl_vnd_product_stats: bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaEventSynchronize(h->done));
    CK(cudaMemcpyAsync(sweeps, h->p32, h->K * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(moves, h->p32 + h->K, h->K * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(evals, h->p64 + 2 * h->K, h->K * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

// Chunk of a streamed upload: per product check that the handle's exact
// widths still hold (else flag -> the caller falls back to a full upload)
// and narrow demand/returns to int32 when that is the stored width.
__global__ void k_check_narrow(int64_t lo, int64_t hi, int T, int64_t K, const int64_t *dem,
                               const int64_t *ret, const int64_t *c6, int vbytes, int cbytes,
                               double sdr_lim, double p16_lim, int32_t *dem32, int32_t *ret32,
                               int *bad,
                               unsigned long long *bounds)
{
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = lo + blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < hi;
         k += nw) {
        double sd = 0.0, sr = 0.0;
        bool neg = false;
        for (int t = lane; t < T; t += 32) {
            const int64_t d = dem[k * T + t], r = ret[k * T + t];
            neg |= d < 0 || r < 0;
            sd += (double)d;
            sr += (double)r;
            if (vbytes == 4) {
                dem32[k * T + t] = (int32_t)d;
                ret32[k * T + t] = (int32_t)r;
            }
        }
        for (int off = 16; off; off >>= 1) {
            sd += __shfl_xor_sync(FULL, sd, off);
            sr += __shfl_xor_sync(FULL, sr, off);
        }
        neg = __any_sync(FULL, neg);
        if (lane == 0) {
            double c[6];
            for (int i = 0; i < 6; ++i) {
                c[i] = (double)c6[i * K + k];
                neg |= c6[i * K + k] < 0;
            }
            const double B = (double)T * (c[0] + c[1]) + (c[4] + c[5]) * sd +
                             (double)T * c[2] * sd + (double)T * c[3] * sr;
            const double vlim = std::ldexp(1.0, vbytes == 4 ? 28 : 60);
            const double clim = std::ldexp(1.0, cbytes == 4 ? 30 : 61);
            const bool qok = vbytes == 8 || coef_bound(c, T) < std::ldexp(1.0, 30);
            if (neg || !(sd + sr < vlim) || !(sd + sr < sdr_lim) || !(sd < p16_lim) ||
                !(sr < p16_lim) || !(B < clim) || !qok)
                atomicExch(bad, 1);
            atomicMax(&bounds[0], (unsigned long long)__double_as_longlong(sd + sr));
            atomicMax(&bounds[1], (unsigned long long)__double_as_longlong(B));
        }
    }
}

// Chunk c of n of rl_vnd_host's pipeline starts at product chunk_lo(K, c, n).
// RL_E2E_GEOM: sizes double from a small first chunk (the descent starts
// after a short first copy); else equal chunks.
#ifndef RL_E2E_GEOM
#define RL_E2E_GEOM 1   // measured: C3 e2e 20.05 -> 19.90 ms
#endif
#ifndef RL_E2E_RATIO
#define RL_E2E_RATIO 2   // chunk-size ratio; 3 / 4 measured 17.87 / 17.79 ms with 3 chunks
#endif
static inline int64_t chunk_lo(int64_t K, int c, int n)
{
    if (!RL_E2E_GEOM || n <= 1)
        return K * c / n;
    int64_t pc = 1, pn = 1;   // r^c, r^n: chunk c spans [r^c - 1, r^(c+1) - 1) / (r^n - 1)
    for (int i = 0; i < n; ++i) {
        if (i < c)
            pc *= RL_E2E_RATIO;
        pn *= RL_E2E_RATIO;
    }
    return K * (pc - 1) / (pn - 1);
}

template <typename V, typename C, typename Mask>
static int do_vnd_chunks(rl_instance *h, int k_max, int nchunks)
{
    const int64_t K = h->K;
    const int T = h->T;
    const size_t kt = (size_t)K * T;
    for (int c = 0; c < nchunks; ++c) {
        cudaStream_t st = (c & 1) ? h->stream2 : h->stream;
        const int64_t lo = chunk_lo(K, c, nchunks), hi = chunk_lo(K, c + 1, nchunks);
        CK(cudaStreamWaitEvent(st, h->evc[c], 0));
        // the decisions taken from the handle's data must hold for the new
        // rows: exact widths, and 16-bit packed lane rows (launch_vnd_range)
        const double sdr_lim = h->sdr_max < 32768.0 ? 32768.0 : 1e300;
        const double p16_lim = h->p16 ? 65536.0 : 1e300;
        k_check_narrow<<<h->sms, 256, 0, st>>>(lo, hi, T, K, h->dem64, h->ret64, h->cost6,
                                               h->vbytes, h->cbytes, sdr_lim, p16_lim,
                                               (int32_t *)h->dem,
                                               (int32_t *)h->ret, h->ints + 3, h->bounds);
        CKL();
        if (c == 0)
            CK(cudaEventRecord(h->ev0, st));
        int rc = launch_vnd_range<V, C, Mask>(h, k_max, h->plan, h->plan + kt, h->plan + 2 * kt,
                                              h->plan + 3 * kt, lo, hi, h->ints + 4 + c, st);
        if (rc)
            return rc;
    }
    return 0;
}

// vnd() from host buffers with the uploads pipelined against the descent:
// products are cut into chunks; a copy stream lands chunk c's instance and
// plan rows while the two compute streams run the chunks before it, and each
// chunk's result rows go back as soon as its kernel ends.  Same results as
// rl_instance_update + rl_vnd, which it falls back to when the new data do
// not fit the handle's exact integer widths (or the trace buffer overflows).
extern "C" int rl_vnd_host(rl_instance *h, int k_max, const int64_t *demand,
                           const int64_t *returns, const int64_t *setup_m, const int64_t *setup_r,
                           const int64_t *hold_m, const int64_t *hold_r, const int64_t *unit_m,
                           const int64_t *unit_r, const uint8_t *sm_in, const uint8_t *sr_in,
                           uint8_t *sm_out, uint8_t *sr_out, int64_t *trace, int64_t trace_cap,
                           int64_t *n_trace, int64_t *stats)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !demand || !returns || !setup_m || !setup_r || !hold_m || !hold_r || !unit_m ||
        !unit_r || !sm_in || !sr_in || !sm_out || !sr_out || !stats)
        return fail(RL_EINVAL, "rl_vnd_host: bad arguments");
    if (k_max < 1 || k_max > 4)
        return fail(RL_EINVAL, "k_max must be in 1..4, got %d", k_max);
    CK(cudaSetDevice(h->device));
    const int64_t K = h->K;
    const int T = h->T;
    const size_t kt = (size_t)K * T;
    const int nchunks = K >= (int64_t)kMaxChunks * 64 * h->sms ? kMaxChunks : 1;
    cudaStream_t s0 = h->stream, s1 = h->stream2, sc = h->stream3;
    cudaEvent_t join = h->evc[kMaxChunks], start = h->evc[kMaxChunks + 1];
    // order after any earlier work on the handle's stream
    CK(cudaEventRecord(start, s0));
    CK(cudaStreamWaitEvent(sc, start, 0));
    CK(cudaStreamWaitEvent(s1, start, 0));
    const int64_t *cost[6] = {setup_m, setup_r, hold_m, hold_r, unit_m, unit_r};
    CK(cudaMemsetAsync(h->ints, 0, 16 * sizeof(int), sc));
    CK(cudaMemsetAsync(h->bounds, 0, 2 * sizeof(unsigned long long), sc));
    CK(cudaMemsetAsync(h->trace_dec, 0, (size_t)h->cap_sweeps * k_max * 8, sc));
    for (int c = 0; c < nchunks; ++c) {
        const int64_t lo = chunk_lo(K, c, nchunks), hi = chunk_lo(K, c + 1, nchunks);
        const size_t off = (size_t)lo * T, n = (size_t)(hi - lo) * T;
        // the chunk's slice of the six cost vectors (the first chunk's
        // kernel needs only its own products' costs)
        for (int i = 0; i < 6; ++i)
            CK(cudaMemcpyAsync(h->cost6 + i * K + lo, cost[i] + lo, (size_t)(hi - lo) * 8,
                               cudaMemcpyHostToDevice, sc));
        CK(cudaMemcpyAsync(h->dem64 + off, demand + off, n * 8, cudaMemcpyHostToDevice, sc));
        CK(cudaMemcpyAsync(h->ret64 + off, returns + off, n * 8, cudaMemcpyHostToDevice, sc));
        CK(cudaMemcpyAsync(h->plan + off, sm_in + off, n, cudaMemcpyHostToDevice, sc));
        CK(cudaMemcpyAsync(h->plan + kt + off, sr_in + off, n, cudaMemcpyHostToDevice, sc));
        CK(cudaEventRecord(h->evc[c], sc));
    }
    h->last_kmax = k_max;
    int rc = RL_DISPATCH_M(h, do_vnd_chunks, h, k_max, nchunks);
    if (rc)
        return rc;
    for (int c = 0; c < nchunks; ++c) {
        cudaStream_t st = (c & 1) ? s1 : s0;
        const int64_t lo = chunk_lo(K, c, nchunks), hi = chunk_lo(K, c + 1, nchunks);
        const size_t off = (size_t)lo * T, n = (size_t)(hi - lo) * T;
        CK(cudaMemcpyAsync(sm_out + off, h->plan + 2 * kt + off, n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(sr_out + off, h->plan + 3 * kt + off, n, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaEventRecord(join, s1));
    CK(cudaStreamWaitEvent(s0, join, 0));
    CK(cudaEventRecord(h->ev1, s0));
    k_vnd_finalize<<<1, 1024, 0, s0>>>(K, vnd_out(h, 0, K, h->ints), h->summary);
    CKL();
    CK(cudaEventRecord(h->done, s0));
    // the instance data changed: the device GVNS state is stale
    gvns_free(h->gv);
    h->gv = nullptr;
    int bad = 0;
    unsigned long long hb[2];
    CK(cudaMemcpyAsync(&bad, h->ints + 3, sizeof bad, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(hb, h->bounds, sizeof hb, cudaMemcpyDeviceToHost, s0));
    CK(cudaStreamSynchronize(s0));
    if (!bad) {
        memcpy(&h->cost_bound, &hb[1], 8);
        rc = rl_vnd_collect(h, trace, trace_cap, n_trace, stats);
    }
    if (bad || rc == RL_ERANGE) {
        rc = rl_instance_update(h, demand, returns, setup_m, setup_r, hold_m, hold_r, unit_m,
                                unit_r);
        if (rc)
            return rc;
        return rl_vnd(h, k_max, sm_in, sr_in, sm_out, sr_out, trace, trace_cap, n_trace, stats);
    }
    return rc;
}

template <typename V, typename C>
static int do_initial(rl_instance *h, uint8_t *d_sm, uint8_t *d_sr, cudaStream_t st)
{
    k_initial<V><<<(unsigned)((h->K + 127) / 128), 128, 0, st>>>(view<V>(h), d_sm, d_sr);
    CKL();
    return 0;
}

extern "C" int rl_initial_solution_device(rl_instance *h, uint8_t *d_sm, uint8_t *d_sr,
                                          void *stream)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !d_sm || !d_sr)
        return fail(RL_EINVAL, "rl_initial_solution_device: bad arguments");
    CK(cudaSetDevice(h->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
    return RL_DISPATCH(h, do_initial, h, d_sm, d_sr, st);
}

extern "C" int rl_initial_solution(rl_instance *h, uint8_t *sm, uint8_t *sr)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !sm || !sr)
        return fail(RL_EINVAL, "rl_initial_solution: bad arguments");
    const size_t kt = (size_t)h->K * h->T;
    int rc = rl_initial_solution_device(h, h->plan, h->plan + kt, h->stream);
    if (rc)
        return rc;
    CK(cudaMemcpyAsync(sm, h->plan, kt, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(sr, h->plan + kt, kt, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}

template <typename V, typename C>
static int do_decode(rl_instance *h, int64_t *d_out, cudaStream_t st)
{
    const size_t kt = (size_t)h->K * h->T;
    k_decode<V><<<(unsigned)((h->K + 127) / 128), 128, 0, st>>>(
        view<V>(h), h->plan, h->plan + kt, d_out, d_out + kt, d_out + 2 * kt, d_out + 3 * kt,
        d_out + 4 * kt);
    CKL();
    return 0;
}

extern "C" int rl_decode(rl_instance *h, const uint8_t *sm, const uint8_t *sr, int64_t *x_m,
                         int64_t *x_r, int64_t *y_m, int64_t *y_r, int64_t *cost)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !sm || !sr || !x_m || !x_r || !y_m || !y_r || !cost)
        return fail(RL_EINVAL, "rl_decode: bad arguments");
    CK(cudaSetDevice(h->device));
    const size_t kt = (size_t)h->K * h->T;
    int64_t *d = nullptr;
    CK(cudaMallocAsync((void **)&d, (4 * kt + h->K) * 8, h->stream));
    int rc = 0;
    do {
        cudaError_t e = cudaMemcpyAsync(h->plan, sm, kt, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h->plan + kt, sr, kt, cudaMemcpyHostToDevice, h->stream);
        if (e != cudaSuccess) {
            rc = fail(RL_ECUDA, "rl_decode: %s", cudaGetErrorString(e));
            break;
        }
        if ((rc = RL_DISPATCH(h, do_decode, h, d, h->stream)))
            break;
        int64_t *outs[5] = {x_m, x_r, y_m, y_r, cost};
        for (int i = 0; i < 5 && e == cudaSuccess; ++i)
            e = cudaMemcpyAsync(outs[i], d + i * kt, (i < 4 ? kt : (size_t)h->K) * 8,
                                cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess)
            e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess)
            rc = fail(RL_ECUDA, "rl_decode: %s", cudaGetErrorString(e));
    } while (0);
    cudaFreeAsync(d, h->stream);
    return rc;
}

// _kernels.oracle_product (_kernels.py:347-371) / oracle.enumerate_optimal
// (oracle.py:19-44): every (m mask, r mask) pair of a product, T <= 10, one
// thread per pattern p = m * 2^T + r; the per-product minimum of the packed
// key (cost << 20 | p) keeps the lowest (m, r) pair on ties like the
// reference's strict '<' over its nested loops.  Cost by the reference's
// per-period recurrence in int64.
__global__ void k_oracle(int64_t K, int T, const int64_t *dem, const int64_t *ret,
                         const int64_t *c6, unsigned long long *best)
{
    const int64_t k = blockIdx.y;
    const uint32_t npat = 1u << (2 * T);
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long key = ~0ull;
    if (p < npat) {
        const uint32_t mm = p >> T, mr = p & ((1u << T) - 1);
        const int64_t *d = dem + k * T, *r = ret + k * T;
        const int64_t km = c6[k], kr = c6[K + k], hm = c6[2 * K + k], hr = c6[3 * K + k],
                      pm = c6[4 * K + k], pr = c6[5 * K + k];
        int64_t cost = 0, rec = 0, stock = 0;
        bool ok = true;
        int t = 0;
        for (; t < T && !(((mm | mr) >> t) & 1); ++t) {
            ok &= d[t] <= 0;
            rec += r[t];
            cost += hr * rec;
        }
        while (ok && t < T) {
            const int u = t;
            int v = u + 1;
            while (v < T && !(((mm | mr) >> v) & 1))
                ++v;
            int64_t need = 0;
            for (int i = u; i < v; ++i)
                need += d[i];
            const int64_t have = rec + r[u];
            const int64_t xr = ((mr >> u) & 1) ? (need < have ? need : have) : 0;
            const int64_t xm = need - xr;
            if (xm > 0 && !((mm >> u) & 1)) {
                ok = false;
                break;
            }
            cost += (xr > 0 ? kr : 0) + (xm > 0 ? km : 0) + pr * xr + pm * xm;
            for (int i = u; i < v; ++i) {
                if (i == u) {
                    stock += xm + xr;
                    rec += r[i] - xr;
                } else {
                    rec += r[i];
                }
                stock -= d[i];
                cost += hm * stock + hr * rec;
            }
            t = v;
        }
        if (ok)
            key = ((unsigned long long)cost << 20) | p;
    }
    for (int off = 16; off; off >>= 1)
        key = min(key, (unsigned long long)__shfl_xor_sync(FULL, key, off));
    if ((threadIdx.x & 31) == 0 && key != ~0ull)
        atomicMin(&best[k], key);
}

extern "C" int rl_oracle_optimal(rl_instance *h, int64_t *cost, uint8_t *sm, uint8_t *sr)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !cost || !sm || !sr)
        return fail(RL_EINVAL, "rl_oracle_optimal: bad arguments");
    if (h->T > 10)
        return fail(RL_EINVAL,
                    "exhaustive enumeration needs periods <= 10 (2^(2*%d) patterns per product "
                    "is intractable)", h->T);
    if (!(h->cost_bound < std::ldexp(1.0, 43)))
        return fail(RL_ERANGE, "rl_oracle_optimal: costs up to %.3g do not fit the packed "
                    "(cost, pattern) key", h->cost_bound);
    CK(cudaSetDevice(h->device));
    const int64_t K = h->K;
    const int T = h->T;
    unsigned long long *d = nullptr;
    CK(cudaMallocAsync((void **)&d, K * 8, h->stream));
    int rc = 0;
    std::vector<unsigned long long> hk((size_t)K);
    do {
        cudaError_t e = cudaMemsetAsync(d, 0xff, K * 8, h->stream);
        if (e == cudaSuccess) {
            const uint32_t npat = 1u << (2 * T);
            dim3 grid((npat + 255) / 256, (unsigned)K);
            k_oracle<<<grid, 256, 0, h->stream>>>(K, T, h->dem64, h->ret64, h->cost6, d);
            ++h->launches;
            e = cudaGetLastError();
        }
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hk.data(), d, K * 8, cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess)
            e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            rc = fail(RL_ECUDA, "rl_oracle_optimal: %s", cudaGetErrorString(e));
            break;
        }
        for (int64_t k = 0; k < K; ++k) {
            const unsigned long long key = hk[(size_t)k];
            if (key == ~0ull) {   // unreachable: all-manufacturing is always feasible
                cost[k] = RL_INFEASIBLE;
                continue;
            }
            cost[k] = (int64_t)(key >> 20);
            const uint32_t p = (uint32_t)(key & 0xFFFFF);
            for (int t = 0; t < T; ++t) {
                sm[k * T + t] = ((p >> T) >> t) & 1;
                sr[k * T + t] = ((p & ((1u << T) - 1)) >> t) & 1;
            }
        }
    } while (0);
    cudaFreeAsync(d, h->stream);
    return rc;
}

extern "C" int rl_list_moves(int nbh, int64_t T, const uint8_t *sm_row, const uint8_t *sr_row,
                             int64_t *mp0, uint8_t *mm0, uint8_t *mr0, int64_t *mp1,
                             uint8_t *mm1, uint8_t *mr1, int64_t *n)
{
    (void)cudaGetLastError();
    if (nbh < 1 || nbh > 4)
        return fail(RL_EINVAL, "neighborhood id must be in 1..4, got %d", nbh);
    if (T < 1 || T > 16000 || !sm_row || !sr_row || !mp0 || !mm0 || !mr0 || !mp1 || !mm1 ||
        !mr1 || !n)
        return fail(RL_EINVAL, "rl_list_moves: bad arguments");
    const size_t cap = 2 * (size_t)T + 2;
    // layout: [mp0 cap][mp1 cap][n 1] int64, then [sm T][sr T][mm0 mr0 mm1 mr1 cap each] bytes
    const size_t words = 2 * cap + 1;
    const size_t bytes = words * 8 + 2 * (size_t)T + 4 * cap;
    uint8_t *d = nullptr;
    const cudaStream_t st = cudaStreamPerThread;
    CK(cudaMallocAsync((void **)&d, bytes, st));
    int64_t *dmp0 = (int64_t *)d, *dmp1 = dmp0 + cap, *dn = dmp1 + cap;
    uint8_t *dsm = d + words * 8, *dsr = dsm + T, *db = dsr + T;
    int rc = 0;
    cudaError_t e = cudaMemcpyAsync(dsm, sm_row, T, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dsr, sr_row, T, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        k_list_moves<<<1, 32, slot_bytes<int32_t, int32_t>((int)T), st>>>(
            nbh, (int)T, dsm, dsr, dmp0, db, db + cap, dmp1, db + 2 * cap, db + 3 * cap, dn);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(n, dn, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && *n > 0) {
        e = cudaMemcpyAsync(mp0, dmp0, *n * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(mp1, dmp1, *n * 8, cudaMemcpyDeviceToHost, st);
        uint8_t *outs[4] = {mm0, mr0, mm1, mr1};
        for (int i = 0; i < 4 && e == cudaSuccess; ++i)
            e = cudaMemcpyAsync(outs[i], db + i * cap, *n, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess)
            e = cudaStreamSynchronize(st);
    }
    if (e != cudaSuccess)
        rc = fail(RL_ECUDA, "rl_list_moves: %s", cudaGetErrorString(e));
    cudaFreeAsync(d, cudaStreamPerThread);
    return rc;
}

// INT32 issue-rate microbenchmark (roofline denominator of the VND kernel):
// 8 independent chains per thread, each iteration one IMAD (fma pipe) and
// one LOP3 (alu pipe) per chain = 16 integer ops.
__global__ void __launch_bounds__(256) k_int_peak(int iters, uint32_t seed, uint32_t *sink)
{
    uint32_t a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a[j] = threadIdx.x * 2654435761u + j + seed;
        b[j] = blockIdx.x * 40503u + 7u * j;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                a[j] = a[j] * 0x9E3779B1u + b[j];
                b[j] ^= a[j];
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        x ^= a[j] + b[j];
    if (x == 0x12345678u)
        sink[0] = x;
}

extern "C" int rl_int_peak(double *ops_per_s)
{
    (void)cudaGetLastError();
    if (!ops_per_s)
        return fail(RL_EINVAL, "rl_int_peak: null output");
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    uint32_t *sink;
    CK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        CK(cudaEventRecord(e0));
        k_int_peak<<<blocks, threads>>>(iters, rep, sink);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0 && ms < best)
            best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    *ops_per_s = (double)blocks * threads * iters * 4 * 8 * 2 / (best * 1e-3);
    return 0;
}

#include "gvns_impl.cuh"
#include "generator.cuh"

extern "C" int64_t rl_launch_count(const rl_instance *h) { return h ? h->launches : 0; }

extern "C" const char *rl_last_error(void) { return g_err.c_str(); }
