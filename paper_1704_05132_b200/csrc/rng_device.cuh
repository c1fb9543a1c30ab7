// rng_device.cuh -- numpy-exact counter-based RNG on the device.
//
// The reference shakes with Generator(Philox(SeedSequence((seed, round,
// worker)))) (reference gvns.py:88-90) and draws rng.choice(n, k,
// replace=False) / rng.shuffle (gvns.py:115, :130).  Those live in numpy
// (third-party, pinned numpy>=1.24, restated from the installed 2.3.5):
//   bit_generator.pyx   SeedSequence mix_entropy / generate_state
//   philox.h            Philox4x64-10, counter bumped before each block,
//                       next_uint32 = low half then high half
//   distributions.c     random_bounded_uint64 (Lemire), random_interval
//   _generator.pyx      choice(replace=False): Floyd + linear-probe set +
//                       _shuffle_int, or tail shuffle; shuffle -> _shuffle_raw
// Pinned against numpy's own outputs (tests/golden/rng.npz) by
// tests/test_gpu_gvns.py and, on the CPU, oracle/numpy_rng.py.
#pragma once
#include <cstdint>

namespace rl {

struct SeedSeq {
    // SeedSequence((seed, round, worker)).generate_state(2, uint64)
    __host__ __device__ static void key(uint64_t seed, uint64_t round, uint64_t worker,
                                        uint64_t out[2])
    {
        const uint64_t vals[3] = {seed, round, worker};
        key_n(vals, 3, out);
    }

    // SeedSequence(vals[0]) (nv = 1) or SeedSequence(tuple(vals)): each value
    // contributes its little-endian uint32 words (one 0 word for 0)
    __host__ __device__ static void key_n(const uint64_t *vals, int nv, uint64_t out[2])
    {
        uint32_t ent[8];
        int n = 0;
        for (int i = 0; i < nv; ++i) {
            uint64_t v = vals[i];
            if (v == 0) {
                ent[n++] = 0;
            } else {
                while (v) {
                    ent[n++] = (uint32_t)v;
                    v >>= 32;
                }
            }
        }
        uint32_t hc = 0x43b0d7e5u;
        auto hashmix = [&](uint32_t v) {
            v ^= hc;
            hc *= 0x931e8875u;
            v *= hc;
            return v ^ (v >> 16);
        };
        auto mix = [](uint32_t x, uint32_t y) {
            uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
            return r ^ (r >> 16);
        };
        uint32_t pool[4];
        for (int i = 0; i < 4; ++i)
            pool[i] = hashmix(i < n ? ent[i] : 0u);
        for (int s = 0; s < 4; ++s)
            for (int d = 0; d < 4; ++d)
                if (s != d)
                    pool[d] = mix(pool[d], hashmix(pool[s]));
        for (int s = 4; s < n; ++s)
            for (int d = 0; d < 4; ++d)
                pool[d] = mix(pool[d], hashmix(ent[s]));
        uint32_t hb = 0x8b51f9ddu, w[4];
        for (int i = 0; i < 4; ++i) {
            uint32_t v = pool[i] ^ hb;
            hb *= 0x58f38dedu;
            v *= hb;
            w[i] = v ^ (v >> 16);
        }
        out[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        out[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    }
};

__host__ __device__ inline uint64_t mulhi64(uint64_t a, uint64_t b)
{
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

struct PhiloxState {
    uint64_t ctr[4], key[2], buf[4];
    int pos;
    int has32;
    uint32_t u32;
};

struct Philox {
    PhiloxState st;

    __host__ __device__ void seed(uint64_t s, uint64_t round, uint64_t worker)
    {
        SeedSeq::key(s, round, worker, st.key);
        for (int i = 0; i < 4; ++i)
            st.ctr[i] = st.buf[i] = 0;
        st.pos = 4;
        st.has32 = 0;
        st.u32 = 0;
    }

    __host__ __device__ void block()
    {
        uint64_t c0 = st.ctr[0], c1 = st.ctr[1], c2 = st.ctr[2], c3 = st.ctr[3];
        uint64_t k0 = st.key[0], k1 = st.key[1];
        for (int r = 0; r < 10; ++r) {
            const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = mulhi64(0xD2E7470EE14C6C93ull, c0);
            const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = mulhi64(0xCA5A826395121157ull, c2);
            const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
            c0 = n0;
            c1 = lo1;
            c2 = n2;
            c3 = lo0;
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        st.buf[0] = c0;
        st.buf[1] = c1;
        st.buf[2] = c2;
        st.buf[3] = c3;
    }

    __host__ __device__ uint64_t next64()
    {
        if (st.pos < 4)
            return st.buf[st.pos++];
        if (++st.ctr[0] == 0 && ++st.ctr[1] == 0 && ++st.ctr[2] == 0)
            ++st.ctr[3];
        block();
        st.pos = 1;
        return st.buf[0];
    }

    __host__ __device__ uint32_t next32()
    {
        if (st.has32) {
            st.has32 = 0;
            return st.u32;
        }
        const uint64_t v = next64();
        st.has32 = 1;
        st.u32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }

    // random_bounded_uint64(off=0, rng, mask=0, use_masked=false)
    __host__ __device__ uint64_t bounded(uint64_t rng)
    {
        if (rng == 0)
            return 0;
        if (rng <= 0xFFFFFFFFull) {
            if (rng == 0xFFFFFFFFull)
                return next32();
            const uint32_t excl = (uint32_t)rng + 1;
            uint64_t m = (uint64_t)next32() * excl;
            uint32_t left = (uint32_t)m;
            if (left < excl) {
                const uint32_t thr = (0xFFFFFFFFu - (uint32_t)rng) % excl;
                while (left < thr) {
                    m = (uint64_t)next32() * excl;
                    left = (uint32_t)m;
                }
            }
            return m >> 32;
        }
        if (rng == ~0ull)
            return next64();
        const uint64_t excl = rng + 1;
        uint64_t x = next64();
        uint64_t lo = x * excl, hi = mulhi64(x, excl);
        if (lo < excl) {
            const uint64_t thr = (~0ull - rng) % excl;
            while (lo < thr) {
                x = next64();
                lo = x * excl;
                hi = mulhi64(x, excl);
            }
        }
        return hi;
    }

    // random_interval(max): masked rejection
    __host__ __device__ uint64_t interval(uint64_t mx)
    {
        if (mx == 0)
            return 0;
        uint64_t mask = mx;
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        mask |= mask >> 32;
        uint64_t v;
        if (mx <= 0xFFFFFFFFull) {
            while ((v = (next32() & mask)) > mx) {
            }
        } else {
            while ((v = (next64() & mask)) > mx) {
            }
        }
        return v;
    }

    // _shuffle_int(n, first, data)
    __host__ __device__ void shuffle_int(int64_t *data, int64_t n, int64_t first)
    {
        for (int64_t i = n - 1; i >= first; --i) {
            const int64_t j = (int64_t)bounded((uint64_t)i);
            const int64_t t = data[j];
            data[j] = data[i];
            data[i] = t;
        }
    }

    // Generator.shuffle of a 1-D int64 array (_shuffle_raw, random_interval)
    __host__ __device__ void shuffle(int64_t *data, int64_t n)
    {
        for (int64_t i = n - 1; i >= 1; --i) {
            const int64_t j = (int64_t)interval((uint64_t)i);
            const int64_t t = data[j];
            data[j] = data[i];
            data[i] = t;
        }
    }
};

// Floyd branch of Generator.choice(pop, size, replace=False, shuffle=True):
// `table` holds (smallest all-ones mask >= 1.2*size) + 1 slots.
__host__ __device__ inline uint64_t choice_table_mask(int64_t size)
{
    uint64_t m = (uint64_t)(1.2 * (double)size);
    m |= m >> 1;
    m |= m >> 2;
    m |= m >> 4;
    m |= m >> 8;
    m |= m >> 16;
    m |= m >> 32;
    return m;
}

__host__ __device__ inline bool choice_uses_tail_shuffle(int64_t pop, int64_t size)
{
    return pop > 10000 && size > pop / 50;
}

__host__ __device__ inline void choice_floyd(Philox &g, int64_t pop, int64_t size, int64_t *out,
                                             uint64_t *table)
{
    const uint64_t mask = choice_table_mask(size);
    for (uint64_t i = 0; i <= mask; ++i)
        table[i] = ~0ull;
    int64_t n = 0;
    for (int64_t j = pop - size; j < pop; ++j) {
        const uint64_t val = g.bounded((uint64_t)j);
        uint64_t loc = val & mask;
        while (table[loc] != ~0ull && table[loc] != val)
            loc = (loc + 1) & mask;
        if (table[loc] == ~0ull) {
            table[loc] = val;
            out[n++] = (int64_t)val;
        } else {
            loc = (uint64_t)j & mask;
            while (table[loc] != ~0ull)
                loc = (loc + 1) & mask;
            table[loc] = (uint64_t)j;
            out[n++] = j;
        }
    }
    g.shuffle_int(out, size, 1);
}

// Tail-shuffle branch (pop > 10000 and size > pop // 50): `idx` has pop slots.
__host__ __device__ inline void choice_tail(Philox &g, int64_t pop, int64_t size, int64_t *out,
                                            int64_t *idx)
{
    for (int64_t i = 0; i < pop; ++i)
        idx[i] = i;
    g.shuffle_int(idx, pop, pop - size > 1 ? pop - size : 1);
    for (int64_t i = 0; i < size; ++i)
        out[i] = idx[pop - size + i];
}

}  // namespace rl
