"""The numpy RNG restatement (oracle/numpy_rng.py) against streams made by
the live numpy the reference depends on (tests/golden/rng.npz)."""

import numpy as np

import numpy_rng
from conftest import golden

CHOICES = ((2, 1), (4, 4), (104000, 5), (12, 3), (10000, 7), (5, 5), (2**33, 3),
           (10001, 5), (20000, 401))


def test_seed_sequence_keys_and_raw_streams():
    g = golden("rng.npz")
    for i, (s, r, w) in enumerate(g["triples"].tolist()):
        key = numpy_rng.seed_sequence_state((s, r, w))
        assert key == g[f"t{i}_key"].tolist()
        ph = numpy_rng.Philox(key)
        assert [ph.next64() for _ in range(9)] == g[f"t{i}_raw"].tolist()


def test_choice_shuffle_and_state_continuation():
    g = golden("rng.npz")
    for i, (s, r, w) in enumerate(g["triples"].tolist()):
        ph = numpy_rng.Philox.from_entropy((s, r, w))
        picks = []
        for n, k in CHOICES:
            picks += ph.choice_noreplace(n, k)
        assert picks == g[f"t{i}_choice"].tolist()
        for n in (0, 1, 2, 7, 300):
            arr = [3 * x + 1 for x in range(n)]
            ph.shuffle(arr)
            assert arr == g[f"t{i}_shuffle{n}"].tolist()
        assert [ph.next64() for _ in range(3)] == g[f"t{i}_tail"].tolist()


def test_matches_live_numpy_generator():
    """Also differential against the numpy in this environment."""
    for seed in (0, 5, 2**40 + 3):
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, 3, 7))))
        ph = numpy_rng.Philox.from_entropy((seed, 3, 7))
        for n, k in ((52000, 3), (9, 2), (1 << 40, 4)):
            assert rng.choice(n, size=k, replace=False).tolist() == ph.choice_noreplace(n, k)
        a = np.arange(50, dtype=np.int64)
        b = list(range(50))
        rng.shuffle(a)
        ph.shuffle(b)
        assert a.tolist() == b
