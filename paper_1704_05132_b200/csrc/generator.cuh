// generate_instance on device (reference pkg/src/remlot/model.py:115-153).
//
// The reference draws everything from ONE Generator(Philox(SeedSequence(seed)))
// through Generator.integers with 32-bit ranges, i.e. numpy's
// random_bounded_uint64 -> buffered_bounded_lemire_uint32 -> next_uint32.
// next_uint32 hands out the low then the high half of successive next_uint64
// words, so the draws form one uint32 stream: draw q is half (q & 1) of
// Philox output word q >> 1, i.e. word (q >> 1) & 3 of the block with counter
// (q >> 3) + 1.  Any draw is a pure function of its stream position.
//
// A cell (one integers() element) consumes 0 draws when its range is 0,
// otherwise 1 + (Lemire rejections).  Positions are a prefix sum of the
// per-cell draw counts, so a fill runs in parallel speculatively: assume no
// rejections, scan, draw every cell at its position, and re-scan with the
// counts actually used until nothing changes.  Each pass fixes at least the
// first cell whose count was wrong (its position depends only on earlier
// cells), and rejections occur with probability < range / 2^32 per draw, so
// a fill normally converges in one or two passes; after 8 passes the tail
// from the first unsettled cell runs sequentially (exact either way).
//
// Draw order (model.py:123-153): demand K x T cells row-major; while any row
// is all zero (demand_max > 0), those rows in ascending order are redrawn
// as a block; returns cell by cell with range floor(ratio * demand + 1e-12)
// (IEEE double, no contraction); then the six K-vectors setup m, setup r,
// holding m, holding r, unit m, unit r.
#pragma once
#include <cub/device/device_scan.cuh>

namespace rl {

struct U32Stream {
    uint64_t key[2];

    __host__ __device__ uint32_t at(uint64_t q) const
    {
        Philox g;
        g.st.key[0] = key[0];
        g.st.key[1] = key[1];
        const uint64_t j = q >> 1;
        g.st.ctr[0] = (j >> 2) + 1;
        g.st.ctr[1] = g.st.ctr[2] = g.st.ctr[3] = 0;
        g.block();
        const uint64_t w = g.st.buf[j & 3];
        return (q & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
    }
};

// buffered_bounded_lemire_uint32 at stream position q, rng in 1..2^32-2:
// value and number of draws consumed
struct LemireDraw {
    uint64_t value;
    int64_t n;
};

__host__ __device__ inline LemireDraw lemire_at(const U32Stream &s, uint64_t q, uint32_t rng)
{
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)s.at(q) * excl;
    int64_t n = 1;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
        while (left < thr) {
            m = (uint64_t)s.at(q + n) * excl;
            ++n;
            left = (uint32_t)m;
        }
    }
    return {m >> 32, n};
}

// demand cells; rows == nullptr: cell i is flat index i, else the cells of
// the listed rows in list order (a redraw block)
struct DemandCells {
    int64_t T;
    uint32_t range;
    const int64_t *rows;
    int64_t *out;
    __device__ uint32_t rng(int64_t) const { return range; }
    __device__ int64_t off(int64_t) const { return 0; }
    __device__ int64_t dest(int64_t i) const { return rows ? rows[i / T] * T + i % T : i; }
};

struct ReturnCells {
    const int64_t *dem;
    double ratio;
    int64_t *out;
    __device__ uint32_t rng(int64_t i) const
    {
        // np.floor(ratio * demand + 1e-12).astype(int64) (model.py:134)
        return (uint32_t)(int64_t)floor(__dadd_rn(__dmul_rn(ratio, (double)dem[i]), 1e-12));
    }
    __device__ int64_t off(int64_t) const { return 0; }
    __device__ int64_t dest(int64_t i) const { return i; }
};

struct VectorCells {
    uint32_t range;
    int64_t lo;
    int64_t *out;
    __device__ uint32_t rng(int64_t) const { return range; }
    __device__ int64_t off(int64_t) const { return lo; }
    __device__ int64_t dest(int64_t i) const { return i; }
};

template <class Cells>
__global__ void k_gen_count(Cells c, int64_t n, int64_t *draws)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        draws[i] = c.rng(i) ? 1 : 0;
}

template <class Cells>
__global__ void k_gen_fill(Cells c, int64_t n, U32Stream s, uint64_t pos, const int64_t *incl,
                           const int64_t *draws, int64_t *draws_new,
                           unsigned long long *first_bad)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = c.rng(i);
        int64_t used = 0;
        if (r == 0) {
            c.out[c.dest(i)] = c.off(i);
        } else {
            const LemireDraw d = lemire_at(s, pos + incl[i] - draws[i], r);
            c.out[c.dest(i)] = c.off(i) + (int64_t)d.value;
            used = d.n;
        }
        draws_new[i] = used;
        if (used != draws[i])
            atomicMin(first_bad, (unsigned long long)i);
    }
}

// the tail [from, n) one cell after another (after 8 unsettled passes)
template <class Cells>
__global__ void k_gen_serial(Cells c, int64_t from, int64_t n, U32Stream s, uint64_t pos,
                             unsigned long long *end)
{
    for (int64_t i = from; i < n; ++i) {
        const uint32_t r = c.rng(i);
        if (r == 0) {
            c.out[c.dest(i)] = c.off(i);
            continue;
        }
        const LemireDraw d = lemire_at(s, pos, r);
        c.out[c.dest(i)] = c.off(i) + (int64_t)d.value;
        pos += d.n;
    }
    *end = pos;
}

// flag[i] = row (rows ? rows[i] : i) of dem is all zero; warp per row
__global__ void k_zero_rows(const int64_t *dem, int64_t T, const int64_t *rows, int64_t nrows,
                            int64_t *flag)
{
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nrows;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t k = rows ? rows[w] : w;
        bool any = false;
        for (int64_t t = lane; t < T; t += 32)
            any |= dem[k * T + t] != 0;
        any = __any_sync(0xffffffffu, any);
        if (lane == 0)
            flag[w] = any ? 0 : 1;
    }
}

// order-preserving compaction of the flagged rows (incl = inclusive scan)
__global__ void k_compact_rows(const int64_t *rows, const int64_t *flag, const int64_t *incl,
                               int64_t nrows, int64_t *out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
         i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i])
            out[incl[i] - 1] = rows ? rows[i] : i;
}

struct GenCtx {
    rl_instance *h = nullptr;   // for launch counting / stream / SM count
    cudaStream_t st = nullptr;
    U32Stream s{};
    uint64_t pos = 0;           // next uint32 draw of the stream
    int64_t cap = 0;
    int64_t *draws = nullptr, *draws2 = nullptr, *incl = nullptr, *rows = nullptr,
            *rows2 = nullptr, *flag = nullptr;
    unsigned long long *scal = nullptr;   // [first_bad, end]
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int passes = 0, serial = 0;           // diagnostics

    int grid() const { return h->sms * 8; }

    int scan(const int64_t *in, int64_t *out, int64_t n)
    {
        size_t need = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, need, in, out, n, st));
        if (need > tmp_bytes) {
            if (tmp)
                CK(cudaFree(tmp));
            tmp = nullptr;
            CK(cudaMalloc(&tmp, need));
            tmp_bytes = need;
        }
        CK(cub::DeviceScan::InclusiveSum(tmp, need, in, out, n, st));
        return 0;
    }

    int64_t read(const int64_t *p)
    {
        int64_t v = 0;
        if (cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return -1;
        return v;
    }

    template <class Cells>
    int fill(Cells c, int64_t n)
    {
        if (n == 0)
            return 0;
        k_gen_count<<<grid(), 256, 0, st>>>(c, n, draws);
        CKL();
        for (int it = 0;; ++it) {
            ++passes;
            if (int rc = scan(draws, incl, n))
                return rc;
            CK(cudaMemsetAsync(scal, 0xff, 8, st));
            k_gen_fill<<<grid(), 256, 0, st>>>(c, n, s, pos, incl, draws, draws2, scal);
            CKL();
            unsigned long long fb = 0;
            CK(cudaMemcpyAsync(&fb, scal, 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (fb == ~0ull) {
                pos += (uint64_t)read(incl + n - 1);
                return 0;
            }
            if (it >= 7) {
                const int64_t i = (int64_t)fb;
                const uint64_t start = pos + read(incl + i) - read(draws + i);
                ++serial;
                k_gen_serial<<<1, 1, 0, st>>>(c, i, n, s, start, scal + 1);
                CKL();
                unsigned long long end = 0;
                CK(cudaMemcpyAsync(&end, scal + 1, 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                pos = end;
                return 0;
            }
            std::swap(draws, draws2);
        }
    }

    void release()
    {
        void *p[] = {draws, draws2, incl, rows, rows2, flag, scal, tmp};
        for (void *q : p)
            if (q)
                cudaFree(q);
    }
};

// Generate the whole K x T instance into dem/ret (K*T each) and cost6 (6*K).
static int generate_full(GenCtx &g, int64_t K, int64_t T, uint64_t seed, int64_t demand_max,
                         double ratio, const int64_t ranges[6], int64_t *dem, int64_t *ret,
                         int64_t *cost6)
{
    rl_instance *h = g.h;
    const int64_t kt = K * T;
    g.cap = kt;
    CK(cudaMalloc(&g.draws, kt * 8));
    CK(cudaMalloc(&g.draws2, kt * 8));
    CK(cudaMalloc(&g.incl, kt * 8));
    CK(cudaMalloc(&g.rows, K * 8));
    CK(cudaMalloc(&g.rows2, K * 8));
    CK(cudaMalloc(&g.flag, K * 8));
    CK(cudaMalloc(&g.scal, 16));
    SeedSeq::key_n(&seed, 1, g.s.key);
    g.pos = 0;
    int rc;
    if ((rc = g.fill(DemandCells{T, (uint32_t)demand_max, nullptr, dem}, kt)))
        return rc;
    if (demand_max > 0) {
        // while rows are all zero: redraw those rows (ascending) as a block
        const int64_t *list = nullptr;   // nullptr = all rows
        int64_t nrows = K;
        for (;;) {
            k_zero_rows<<<g.grid(), 256, 0, g.st>>>(dem, T, list, nrows, g.flag);
            CKL();
            if ((rc = g.scan(g.flag, g.incl, nrows)))
                return rc;
            const int64_t ndead = g.read(g.incl + nrows - 1);
            if (ndead < 0)
                return fail(RL_ECUDA, "generate: read failed");
            if (ndead == 0)
                break;
            k_compact_rows<<<g.grid(), 256, 0, g.st>>>(list, g.flag, g.incl, nrows, g.rows);
            CKL();
            if ((rc = g.fill(DemandCells{T, (uint32_t)demand_max, g.rows, dem}, ndead * T)))
                return rc;
            std::swap(g.rows, g.rows2);
            list = g.rows2;
            nrows = ndead;
        }
    }
    if ((rc = g.fill(ReturnCells{dem, ratio, ret}, kt)))
        return rc;
    for (int v = 0; v < 6; ++v) {
        const int64_t lo = ranges[2 * (v / 2)], hi = ranges[2 * (v / 2) + 1];
        if ((rc = g.fill(VectorCells{(uint32_t)(hi - lo), lo, cost6 + v * K}, K)))
            return rc;
    }
    return 0;
}

}  // namespace rl

// generate_instance(GeneratorConfig(K, T, demand_max, return_ratio, ranges,
// seed)) on the device, keeping products [lo, hi) in the new handle.
extern "C" int rl_generate_instance(int64_t K, int64_t T, uint64_t seed, int64_t demand_max,
                                    double return_ratio, const int64_t *ranges, int64_t lo,
                                    int64_t hi, rl_instance **out)
{
    (void)cudaGetLastError();
    if (!out || !ranges)
        return fail(RL_EINVAL, "rl_generate_instance: null argument");
    *out = nullptr;
    // GeneratorConfig._validate (model.py:100-112)
    if (K < 1)
        return fail(RL_EINVAL, "products must be >= 1");
    if (T < 1 || T > 16000)
        return fail(RL_EINVAL, "periods must be in 1..16000, got %lld", (long long)T);
    if (demand_max < 0)
        return fail(RL_EINVAL, "demand_max must be >= 0");
    if (!(return_ratio >= 0.0 && return_ratio <= 1.0))
        return fail(RL_EINVAL, "return_ratio must be in [0, 1]");
    for (int i = 0; i < 3; ++i)
        if (ranges[2 * i] < 0 || ranges[2 * i + 1] < ranges[2 * i])
            return fail(RL_EINVAL, "cost range %d must satisfy 0 <= lo <= hi", i);
    // the device path covers numpy's 32-bit draw path (every range < 2^32-1)
    const int64_t lim = 0xFFFFFFFEll;
    if (demand_max > lim || ranges[1] - ranges[0] > lim || ranges[3] - ranges[2] > lim ||
        ranges[5] - ranges[4] > lim)
        return fail(RL_EINVAL, "ranges of 2^32-1 or more are outside the device generator");
    if (lo < 0 || hi > K || hi <= lo)
        return fail(RL_EINVAL, "product range [%lld, %lld) not inside [0, %lld)",
                    (long long)lo, (long long)hi, (long long)K);
    rl_instance *h = new rl_instance();
    h->K = hi - lo;
    h->T = (int)T;
    int rc = alloc_instance(h);
    if (!rc) {
        rl::GenCtx g;
        g.h = h;
        g.st = h->stream;
        const bool whole = lo == 0 && hi == K;
        int64_t *dem = h->dem64, *ret = h->ret64, *c6 = h->cost6, *buf = nullptr;
        if (!whole) {
            cudaError_t e = cudaMalloc(&buf, (size_t)K * (2 * T + 6) * 8);
            if (e != cudaSuccess)
                rc = fail(RL_ECUDA, "rl_generate_instance: %s", cudaGetErrorString(e));
            dem = buf;
            ret = buf + K * T;
            c6 = buf + 2 * K * T;
        }
        if (!rc)
            rc = rl::generate_full(g, K, T, seed, demand_max, return_ratio, ranges, dem, ret, c6);
        if (!rc && !whole) {
            const size_t n = (size_t)(hi - lo) * T;
            cudaStream_t st = h->stream;
            cudaError_t e = cudaMemcpyAsync(h->dem64, dem + lo * T, n * 8,
                                            cudaMemcpyDeviceToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(h->ret64, ret + lo * T, n * 8, cudaMemcpyDeviceToDevice, st);
            for (int v = 0; v < 6 && e == cudaSuccess; ++v)
                e = cudaMemcpyAsync(h->cost6 + v * h->K, c6 + v * K + lo, h->K * 8,
                                    cudaMemcpyDeviceToDevice, st);
            if (e == cudaSuccess)
                e = cudaStreamSynchronize(st);
            if (e != cudaSuccess)
                rc = fail(RL_ECUDA, "rl_generate_instance: %s", cudaGetErrorString(e));
        }
        cudaStreamSynchronize(h->stream);
        g.release();
        if (buf)
            cudaFree(buf);
        if (!rc)
            rc = prepare(h);
    }
    return finish_create(h, rc, out);
}

// Copy the handle's instance back to host arrays (K x T, K x T, 6 x K).
extern "C" int rl_instance_download(rl_instance *h, int64_t *demand, int64_t *returns,
                                    int64_t *setup_m, int64_t *setup_r, int64_t *hold_m,
                                    int64_t *hold_r, int64_t *unit_m, int64_t *unit_r)
{
    RL_GUARD(h);
    (void)cudaGetLastError();
    if (!h || !demand || !returns || !setup_m || !setup_r || !hold_m || !hold_r || !unit_m ||
        !unit_r)
        return fail(RL_EINVAL, "rl_instance_download: bad arguments");
    CK(cudaSetDevice(h->device));
    const size_t kt = (size_t)h->K * h->T;
    CK(cudaMemcpyAsync(demand, h->dem64, kt * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(returns, h->ret64, kt * 8, cudaMemcpyDeviceToHost, h->stream));
    int64_t *cost[6] = {setup_m, setup_r, hold_m, hold_r, unit_m, unit_r};
    for (int i = 0; i < 6; ++i)
        CK(cudaMemcpyAsync(cost[i], h->cost6 + i * h->K, h->K * 8, cudaMemcpyDeviceToHost,
                           h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
}
