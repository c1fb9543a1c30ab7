"""ctypes front-end of the CPU oracle (oracle/remlot_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / reference arm -- never by the product package.

All functions take any object with the reference ``Instance`` attributes
(products, periods, demand, returns, setup_cost_m/r, holding_cost_m/r,
unit_cost_m/r) and boolean K x T setup matrices, exactly like the reference
kernels they restate (remlot/_kernels.py, vnd.py, plan.py).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
INFEASIBLE = 1 << 62

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        _lib.orc_row_cost.restype = I64
        _lib.orc_row_cost.argtypes = [I64, P, P, P, P] + [I64] * 6
        _lib.orc_product_costs.argtypes = [P, I64, I64, P, P, P]
        _lib.orc_list_moves.restype = I64
        _lib.orc_list_moves.argtypes = [ctypes.c_int, I64, P, P, P, P, P, P, P, P]
        _lib.orc_scan_products.restype = I64
        _lib.orc_scan_products.argtypes = [P, I64, I64, P, P, ctypes.c_int] + [P] * 7
        _lib.orc_apply_scan.restype = I64
        _lib.orc_apply_scan.argtypes = [I64, I64, I64] + [P] * 9
        _lib.orc_vnd.restype = ctypes.c_int
        _lib.orc_vnd.argtypes = [P, ctypes.c_int, P, P, ctypes.c_int, P, P, I64, P, P]
        _lib.orc_initial_solution.argtypes = [P, P, P]
        _lib.orc_row_decode.restype = I64
        _lib.orc_row_decode.argtypes = [I64, P, P, P, P] + [I64] * 6 + [P] * 4
    return _lib


class _OrcInst(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("T", ctypes.c_int64)] + [
        (n, ctypes.c_void_p) for n in ("dem", "ret", "km", "kr", "hm", "hr", "pm", "pr")]


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleInstance:
    """Holds contiguous int64 copies of an instance for the C oracle."""

    def __init__(self, inst):
        self.K = int(inst.products)
        self.T = int(inst.periods)
        c = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        self.arrays = [c(inst.demand), c(inst.returns), c(inst.setup_cost_m),
                       c(inst.setup_cost_r), c(inst.holding_cost_m),
                       c(inst.holding_cost_r), c(inst.unit_cost_m), c(inst.unit_cost_r)]
        self.s = _OrcInst(self.K, self.T, *[_ptr(a) for a in self.arrays])
        self.ref = ctypes.byref(self.s)


def _as(inst):
    return inst if isinstance(inst, OracleInstance) else OracleInstance(inst)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def product_costs(inst, sm, sr):
    o = _as(inst)
    out = np.empty(o.K, np.int64)
    sm, sr = _u8(sm), _u8(sr)
    lib().orc_product_costs(o.ref, 0, o.K, _ptr(sm), _ptr(sr), _ptr(out))
    return out


def evaluate(inst, sm, sr):
    c = product_costs(inst, sm, sr)
    return INFEASIBLE if (c == INFEASIBLE).any() else int(c.sum())


def row_cost(sm_row, sr_row, dem, ret, km, kr, hm, hr, pm=0, pr=0):
    sm_row, sr_row = _u8(sm_row), _u8(sr_row)
    dem = np.ascontiguousarray(dem, np.int64)
    ret = np.ascontiguousarray(ret, np.int64)
    return int(lib().orc_row_cost(len(dem), _ptr(sm_row), _ptr(sr_row), _ptr(dem),
                                  _ptr(ret), km, kr, hm, hr, pm, pr))


def list_moves(nbh, sm_row, sr_row):
    """Canonical move list of one product (mp0, mm0, mr0, mp1, mm1, mr1)."""
    sm_row, sr_row = _u8(sm_row), _u8(sr_row)
    T = len(sm_row)
    cap = 2 * T + 2
    mp0 = np.empty(cap, np.int64)
    mp1 = np.empty(cap, np.int64)
    b = [np.empty(cap, np.uint8) for _ in range(4)]
    n = lib().orc_list_moves(nbh, T, _ptr(sm_row), _ptr(sr_row), _ptr(mp0),
                             _ptr(b[0]), _ptr(b[1]), _ptr(mp1), _ptr(b[2]), _ptr(b[3]))
    return (mp0[:n], b[0][:n].astype(bool), b[1][:n].astype(bool), mp1[:n],
            b[2][:n].astype(bool), b[3][:n].astype(bool))


def scan_products(inst, sm, sr, nbh, lo=0, hi=None):
    """scan_products outputs (dec, p0, m0, r0, p1, m1, r1) and eval count.

    m0/r0 are False where dec == 0 and m1/r1 False where p1 < 0 (the
    reference leaves those slots unwritten)."""
    o = _as(inst)
    hi = o.K if hi is None else hi
    sm, sr = _u8(sm), _u8(sr)
    dec = np.zeros(o.K, np.int64)
    p0 = np.full(o.K, -1, np.int64)
    p1 = np.full(o.K, -1, np.int64)
    b = [np.zeros(o.K, np.uint8) for _ in range(4)]
    ev = lib().orc_scan_products(o.ref, lo, hi, _ptr(sm), _ptr(sr), nbh, _ptr(dec),
                                 _ptr(p0), _ptr(b[0]), _ptr(b[1]), _ptr(p1),
                                 _ptr(b[2]), _ptr(b[3]))
    m0, r0, m1, r1 = (x.astype(bool) for x in b)
    m0 &= dec > 0
    r0 &= dec > 0
    m1 &= (dec > 0) & (p1 >= 0)
    r1 &= (dec > 0) & (p1 >= 0)
    return (dec, p0, m0, r0, p1, m1, r1), int(ev)


def vnd(inst, sm, sr, k_max=4, threads=1, trace_cap=1 << 16):
    """Lockstep VND (vnd.py:253-289).  Returns (sm, sr, cost, trace, stats)
    with stats = dict(evals, moves, sweeps)."""
    o = _as(inst)
    sm = _u8(sm).copy()
    sr = _u8(sr).copy()
    trace = np.empty(trace_cap, np.int64)
    cost = np.zeros(1, np.int64)
    nt = np.zeros(1, np.int64)
    stats = np.zeros(3, np.int64)
    rc = lib().orc_vnd(o.ref, k_max, _ptr(sm), _ptr(sr), threads, _ptr(cost),
                       _ptr(trace), trace_cap, _ptr(nt), _ptr(stats))
    if rc == -1:
        return vnd(inst, sm, sr, k_max, threads, trace_cap * 4)
    if rc != 0:
        raise RuntimeError(f"oracle vnd failed: {rc}")
    return (sm.astype(bool), sr.astype(bool), int(cost[0]), trace[:nt[0]].copy(),
            dict(evals=int(stats[0]), moves=int(stats[1]), sweeps=int(stats[2])))


def initial_solution(inst):
    o = _as(inst)
    sm = np.zeros((o.K, o.T), np.uint8)
    sr = np.zeros((o.K, o.T), np.uint8)
    lib().orc_initial_solution(o.ref, _ptr(sm), _ptr(sr))
    return sm.astype(bool), sr.astype(bool)


def decode(inst, sm, sr):
    """Per product (x_m, x_r, y_m, y_r, cost) like plan.decode (plan.py:99-114)."""
    o = _as(inst)
    K, T = o.K, o.T
    sm, sr = _u8(sm), _u8(sr)
    out = [np.zeros((K, T), np.int64) for _ in range(4)]
    costs = np.zeros(K, np.int64)
    a = o.arrays
    for k in range(K):
        costs[k] = lib().orc_row_decode(
            T, _ptr(sm[k]), _ptr(sr[k]), _ptr(a[0][k]), _ptr(a[1][k]),
            int(a[2][k]), int(a[3][k]), int(a[4][k]), int(a[5][k]), int(a[6][k]),
            int(a[7][k]), _ptr(out[0][k]), _ptr(out[1][k]), _ptr(out[2][k]),
            _ptr(out[3][k]))
    return out[0], out[1], out[2], out[3], costs
