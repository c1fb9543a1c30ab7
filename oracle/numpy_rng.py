"""Pure-Python restatement of the numpy RNG pieces the reference's shake uses.

TEST INFRASTRUCTURE ONLY (checker for the device Philox shake).

The reference draws shake positions from
``Generator(Philox(SeedSequence((seed, round, worker))))`` (reference
gvns.py:88-90) with ``choice(n, k, replace=False)`` (gvns.py:115) and, on the
fallback path, ``shuffle`` (gvns.py:130).  Those algorithms live in the
third-party dependency numpy (pinned ``numpy>=1.24`` by reference
pyproject.toml:11; restated here from numpy 2.3.5 as installed):

  * numpy/random/bit_generator.pyx  SeedSequence: _coerce_to_uint32_array,
    mix_entropy (hashmix/mix), generate_state
  * numpy/random/_philox.pyx + src/philox/philox.h  Philox4x64-10, counter
    incremented before each 4-word block, next_uint32 = low then high half
  * numpy/random/src/distributions/distributions.c  random_bounded_uint64
    (Lemire for 32- and 64-bit ranges), random_interval (masked rejection)
  * numpy/random/_generator.pyx  choice(replace=False): Floyd + hash set +
    _shuffle_int, or tail-shuffle when pop > 10000 and size > pop // 50;
    shuffle(1-D) -> _shuffle_raw with random_interval

Parity is pinned by tests/test_rng.py against tests/golden/rng.npz (made
by the live numpy) -- the reference's own tests only pin self-consistency.
"""

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF

INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
XSHIFT = 16
POOL_SIZE = 4

PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def int_to_words(n):
    if n < 0:
        raise ValueError("expected non-negative integer")
    if n == 0:
        return [0]
    out = []
    while n > 0:
        out.append(n & M32)
        n >>= 32
    return out


def seed_words(entropy):
    """_coerce_to_uint32_array of an int or a tuple of ints."""
    if isinstance(entropy, int):
        return int_to_words(entropy)
    words = []
    for e in entropy:
        words += int_to_words(e)
    return words


def seed_sequence_state(entropy, n_words64=2):
    """SeedSequence(entropy).generate_state(n_words64, uint64)."""
    hc = INIT_A

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * MULT_A) & M32
        v = (v * hc) & M32
        return v ^ (v >> XSHIFT)

    def mix(x, y):
        r = (MIX_MULT_L * x - MIX_MULT_R * y) & M32
        return r ^ (r >> XSHIFT)

    ent = seed_words(entropy)
    pool = []
    for i in range(POOL_SIZE):
        pool.append(hashmix(ent[i] if i < len(ent) else 0))
    for i_src in range(POOL_SIZE):
        for i_dst in range(POOL_SIZE):
            if i_src != i_dst:
                pool[i_dst] = mix(pool[i_dst], hashmix(pool[i_src]))
    for i_src in range(POOL_SIZE, len(ent)):
        for i_dst in range(POOL_SIZE):
            pool[i_dst] = mix(pool[i_dst], hashmix(ent[i_src]))
    hb = INIT_B
    words = []
    for i in range(2 * n_words64):
        v = pool[i % POOL_SIZE]
        v ^= hb
        hb = (hb * MULT_B) & M32
        v = (v * hb) & M32
        v ^= v >> XSHIFT
        words.append(v)
    return [words[2 * i] | (words[2 * i + 1] << 32) for i in range(n_words64)]


def philox4x64(ctr, key, rounds=10):
    c = list(ctr)
    k0, k1 = key
    for r in range(rounds):
        p0 = PHILOX_M0 * c[0]
        p1 = PHILOX_M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & M64
        hi1, lo1 = p1 >> 64, p1 & M64
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        if r < rounds - 1:
            k0 = (k0 + PHILOX_W0) & M64
            k1 = (k1 + PHILOX_W1) & M64
    return c


class Philox:
    """numpy.random.Philox bit generator state machine."""

    def __init__(self, key):
        self.key = tuple(key)
        self.ctr = [0, 0, 0, 0]
        self.buf = [0, 0, 0, 0]
        self.pos = 4
        self.has32 = False
        self.u32 = 0

    @classmethod
    def from_entropy(cls, entropy):
        return cls(seed_sequence_state(entropy, 2))

    def next64(self):
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        for i in range(4):
            self.ctr[i] = (self.ctr[i] + 1) & M64
            if self.ctr[i] != 0:
                break
        self.buf = philox4x64(self.ctr, self.key)
        self.pos = 1
        return self.buf[0]

    def next32(self):
        if self.has32:
            self.has32 = False
            return self.u32
        v = self.next64()
        self.has32 = True
        self.u32 = v >> 32
        return v & M32

    # distributions.c ------------------------------------------------------
    def bounded_uint64(self, rng):
        """random_bounded_uint64(off=0, rng, mask=0, use_masked=False)."""
        if rng == 0:
            return 0
        if rng <= M32:
            if rng == M32:
                return self.next32()
            excl = rng + 1
            m = self.next32() * excl
            left = m & M32
            if left < excl:
                thr = (M32 - rng) % excl
                while left < thr:
                    m = self.next32() * excl
                    left = m & M32
            return m >> 32
        if rng == M64:
            return self.next64()
        excl = rng + 1
        m = self.next64() * excl
        left = m & M64
        if left < excl:
            thr = (M64 - rng) % excl
            while left < thr:
                m = self.next64() * excl
                left = m & M64
        return m >> 64

    def interval(self, mx):
        """random_interval(max): masked rejection."""
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= M32:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    # Generator ------------------------------------------------------------
    def shuffle_int(self, data, n, first):
        for i in range(n - 1, first - 1, -1):
            j = self.bounded_uint64(i)
            data[i], data[j] = data[j], data[i]

    def choice_noreplace(self, pop, size):
        if size > pop:
            raise ValueError("Cannot take a larger sample than population when replace is False")
        if pop > 10000 and size > pop // 50:
            idx = list(range(pop))
            self.shuffle_int(idx, pop, max(pop - size, 1))
            return idx[pop - size:]
        set_size = int(1.2 * size)
        mask = set_size
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        table = [None] * (mask + 1)
        out = []
        for j in range(pop - size, pop):
            val = self.bounded_uint64(j)
            loc = val & mask
            while table[loc] is not None and table[loc] != val:
                loc = (loc + 1) & mask
            if table[loc] is None:
                table[loc] = val
                out.append(val)
            else:
                loc = j & mask
                while table[loc] is not None:
                    loc = (loc + 1) & mask
                table[loc] = j
                out.append(j)
        self.shuffle_int(out, size, 1)
        return out

    def shuffle(self, data):
        for i in range(len(data) - 1, 0, -1):
            j = self.interval(i)
            data[i], data[j] = data[j], data[i]
