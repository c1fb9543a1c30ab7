"""Variable neighborhood descent on the GPU (mirror of reference vnd.py).

Neighborhoods act on one product's rows (reference vnd.py:1-15):
  1 flip a manufacturing bit, 2 flip a remanufacturing bit,
  3 shift a set bit one period within its row, 4 swap the two bits of a period.

``vnd`` runs the persistent resident kernel (``rl_vnd``): one warp per
product descends to that product's fixpoint, which is exactly the
reference's lockstep loop because products never interact; the per-pass
decreases are reduced on the device so ``trace`` matches the reference
entry for entry.  ``vnd_pass`` / ``best_neighbor`` are one lockstep pass
(``rl_scan_products``), ``enumerate_neighbors`` is ``rl_list_moves``.

``mode`` and ``parallelism`` are validated exactly as in the reference and
then have no effect: the device path is bit-identical for every setting
(the reference's own contract, vnd.py:213-217).
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .model import Instance
from .plan import SetupPlan, _check_dims

MODE_SERIAL = "serial"
MODE_PRODUCT_PARALLEL = "product-parallel"
VND_MODES = (MODE_SERIAL, MODE_PRODUCT_PARALLEL)

NEIGHBORHOOD_COUNT = 4
DEFAULT_PARALLELISM = 4

# kept for API compatibility (reference tests monkeypatch it); the device
# path has no host chunking
_MIN_CHUNK = 64


@dataclass(frozen=True)
class Move:
    """One edit of a single product's rows (reference vnd.py:53-79)."""

    product: int
    neighborhood: int
    periods: tuple
    new_m: tuple
    new_r: tuple
    old_m: tuple
    old_r: tuple

    def apply(self, plan: SetupPlan) -> SetupPlan:
        setup_m = plan.setup_m.copy()
        setup_r = plan.setup_r.copy()
        _write_move(setup_m, setup_r, self)
        return SetupPlan(setup_m, setup_r)

    def inverted(self) -> "Move":
        return Move(self.product, self.neighborhood, self.periods,
                    self.old_m, self.old_r, self.new_m, self.new_r)


@dataclass(frozen=True)
class ImprovementDelta:
    """Per-product best moves of one pass and their summed decrease."""

    moves: tuple
    decreases: tuple
    diff: int


def _write_move(setup_m, setup_r, move):
    k = move.product
    for i, t in enumerate(move.periods):
        if bool(setup_m[k, t]) != move.old_m[i] or bool(setup_r[k, t]) != move.old_r[i]:
            raise ValueError(f"stale move: plan bits at product {k} period {t} changed "
                             "since the move was computed")
    for i, t in enumerate(move.periods):
        setup_m[k, t] = move.new_m[i]
        setup_r[k, t] = move.new_r[i]


def _check_neighborhood(nbh):
    if not 1 <= nbh <= NEIGHBORHOOD_COUNT:
        raise ValueError(f"neighborhood id must be in 1..{NEIGHBORHOOD_COUNT}, got {nbh}")


def _check_mode(mode):
    if mode not in VND_MODES:
        raise ValueError(f"unknown vnd mode {mode!r}")


def _move(plan, nbh, k, p0, m0, r0, p1, m1, r1):
    periods, new_m, new_r = [int(p0)], [bool(m0)], [bool(r0)]
    if p1 >= 0:
        periods.append(int(p1))
        new_m.append(bool(m1))
        new_r.append(bool(r1))
    old_m = tuple(bool(plan.setup_m[k, t]) for t in periods)
    old_r = tuple(bool(plan.setup_r[k, t]) for t in periods)
    return Move(k, nbh, tuple(periods), tuple(new_m), tuple(new_r), old_m, old_r)


def enumerate_neighbors(plan: SetupPlan, nbh: int, k: int) -> list:
    """All moves of ``nbh`` for product ``k`` in canonical order (vnd.py:116-138)."""
    _check_neighborhood(nbh)
    K, _ = plan.shape
    if not 0 <= k < K:
        raise IndexError(f"product index {k} out of range 0..{K - 1}")
    mp0, mm0, mr0, mp1, mm1, mr1 = _native.list_moves(nbh, plan.setup_m[k], plan.setup_r[k])
    return [_move(plan, nbh, k, mp0[i], mm0[i], mr0[i], mp1[i], mm1[i], mr1[i])
            for i in range(len(mp0))]


def best_neighbor(inst: Instance, plan: SetupPlan, nbh: int, k: int):
    """(move, decrease) of the best strictly improving move, or None (vnd.py:171-188)."""
    _check_neighborhood(nbh)
    _check_dims(inst, plan)
    K, _ = plan.shape
    if not 0 <= k < K:
        raise IndexError(f"product index {k} out of range 0..{K - 1}")
    out, _ = _native.device_instance(inst).scan_products(plan.setup_m, plan.setup_r, nbh, k, k + 1)
    dec = int(out[0][k])
    if dec <= 0:
        return None
    return _move(plan, nbh, k, *(a[k] for a in out[1:])), dec


def vnd_pass(inst: Instance, plan: SetupPlan, nbh: int, mode: str = MODE_SERIAL,
             parallelism: int = DEFAULT_PARALLELISM) -> ImprovementDelta:
    """One best-move-per-product pass of one neighborhood (vnd.py:209-235)."""
    _check_neighborhood(nbh)
    _check_mode(mode)
    _check_dims(inst, plan)
    out, _ = _native.device_instance(inst).scan_products(plan.setup_m, plan.setup_r, nbh)
    dec = out[0]
    winners = np.flatnonzero(dec > 0)
    moves = tuple(_move(plan, nbh, int(k), *(a[k] for a in out[1:])) for k in winners)
    decreases = tuple(int(dec[k]) for k in winners)
    return ImprovementDelta(moves, decreases, sum(decreases))


def apply_delta(plan: SetupPlan, delta: ImprovementDelta) -> SetupPlan:
    """Apply every move of ``delta``; raises on stale bits (vnd.py:238-250)."""
    if not delta.moves:
        return plan
    setup_m = plan.setup_m.copy()
    setup_r = plan.setup_r.copy()
    for move in delta.moves:
        _write_move(setup_m, setup_r, move)
    return SetupPlan(setup_m, setup_r)


def vnd(inst: Instance, plan: SetupPlan, k_max: int = NEIGHBORHOOD_COUNT,
        mode: str = MODE_SERIAL, parallelism: int = DEFAULT_PARALLELISM,
        trace: list = None, stats: dict = None):
    """Descend through neighborhoods 1..k_max to a local optimum (vnd.py:253-289).

    Returns (plan, cost) with cost = evaluate(start) - sum of pass decreases
    exactly as the reference computes it; ``trace`` receives the start cost
    and the running cost after every lockstep pass.  ``stats`` (extension)
    receives sweeps, evaluation counts and kernel time.
    """
    if not 1 <= k_max <= NEIGHBORHOOD_COUNT:
        raise ValueError(f"k_max must be in 1..{NEIGHBORHOOD_COUNT}, got {k_max}")
    _check_mode(mode)
    _check_dims(inst, plan)
    sm, sr, tr, st = _native.device_instance(inst).vnd(plan.setup_m, plan.setup_r, k_max)
    if trace is not None:
        trace.extend(int(x) for x in tr)
    if stats is not None:
        stats.update(st)
    return SetupPlan(sm, sr), st["cost"]
