"""Product-sharded VND across ranks (one process per GPU).

Products are independent, so rank r of N descends products
[r*K//N, (r+1)*K//N) -- the contiguous blocks the reference's product-parallel
mode uses (vnd.py:195-206, np.linspace bounds) -- and the job only combines
totals: the start cost (INFEASIBLE if any shard is), the per-pass decrease
vectors (padded to the longest shard and summed, which rebuilds the
reference's lockstep trace exactly) and the evaluation/move counters.  No
data-path collective exists; the plan is gathered only on request.

The local descent is pluggable (``local_vnd``) so the combine logic is tested
on CPU with the gloo backend against the oracle; the product path uses the
device VND (``_native.DeviceInstance.vnd``).
"""

import numpy as np

INFEASIBLE = 1 << 62


def shard_bounds(K, rank, world):
    return K * rank // world, K * (rank + 1) // world


def _device_local_vnd(inst, sm, sr, k_max):
    from . import _native
    dev = _native.DeviceInstance(inst)
    out_m, out_r, trace, st = dev.vnd(sm, sr, k_max)
    return out_m, out_r, [int(x) for x in trace], st


def combine(trace, stats, group=None, device="cpu"):
    """Combine one shard's trace/stats into the job's (collective).

    Returns (global_trace, totals) where totals has start_cost, cost,
    sweeps, evals, evals_reference, moves (sums / max over ranks)."""
    import torch
    import torch.distributed as dist

    start = int(trace[0])
    feasible = 1 if start != INFEASIBLE else 0
    decs = [int(trace[i]) - int(trace[i + 1]) for i in range(len(trace) - 1)]
    hdr = torch.tensor([len(decs), -feasible], dtype=torch.int64, device=device)
    dist.all_reduce(hdr, op=dist.ReduceOp.MAX, group=group)
    n_pass, any_infeasible = int(hdr[0]), int(hdr[1]) == 0
    k_max = int(stats.get("k_max", 4))
    local_sweeps = len(decs) // k_max
    ntot = int(stats.get("ntot_sum", 0))
    vec = torch.zeros(n_pass + 5, dtype=torch.int64, device=device)
    if decs:
        vec[:len(decs)] = torch.tensor(decs, dtype=torch.int64)
    vec[n_pass] = start if feasible else 0
    vec[n_pass + 1] = int(stats.get("evals", 0))
    vec[n_pass + 2] = int(stats.get("moves", 0))
    # the lockstep count credits every product up to the GLOBAL sweep count:
    # ref = sum_shards (ref_local - S_local * ntot_local) + S_global * sum ntot
    vec[n_pass + 3] = int(stats.get("evals_reference", 0)) - local_sweeps * ntot
    vec[n_pass + 4] = ntot
    dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    tot = vec.cpu().tolist()
    start_total = INFEASIBLE if any_infeasible else tot[n_pass]
    g_trace = [start_total]
    for d in tot[:n_pass]:
        g_trace.append(g_trace[-1] - d)
    sweeps = n_pass // k_max
    totals = dict(start_cost=start_total, cost=g_trace[-1], sweeps=sweeps,
                  evals=tot[n_pass + 1], moves=tot[n_pass + 2],
                  evals_reference=tot[n_pass + 3] + sweeps * tot[n_pass + 4])
    return g_trace, totals


def sharded_vnd(inst, plan, k_max=4, group=None, local_vnd=None, device="cpu",
                gather_plan=True):
    """VND of ``inst`` from ``plan`` with products sharded over the ranks of
    ``group``.  Every rank returns (plan or None, cost, trace, totals); the
    plan (gathered, rank order = product order) only when gather_plan.
    ``local_vnd(shard, sm, sr, k_max) -> (sm, sr, trace, stats)`` with stats
    holding evals, moves, evals_reference (the shard's own lockstep count)
    and ntot_sum (sum over feasible products of their final move counts)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_bounds(inst.products, rank, world)
    if hi > lo:
        shard = inst.slice(lo, hi)
        fn = local_vnd or _device_local_vnd
        sm, sr, trace, st = fn(shard, plan.setup_m[lo:hi], plan.setup_r[lo:hi], k_max)
    else:   # more ranks than products
        sm = sr = np.zeros((0, inst.periods), bool)
        trace, st = [0], {}
    st = dict(st)
    st["k_max"] = k_max
    g_trace, totals = combine(trace, st, group=group, device=device)
    full = None
    if gather_plan:
        parts = [None] * world
        dist.all_gather_object(parts, (np.packbits(sm, axis=1), np.packbits(sr, axis=1)),
                               group=group)
        T = inst.periods
        m = np.concatenate([np.unpackbits(p[0], axis=1, count=T) for p in parts]).astype(bool)
        r = np.concatenate([np.unpackbits(p[1], axis=1, count=T) for p in parts]).astype(bool)
        from .plan import SetupPlan
        full = SetupPlan(m, r)
    return full, totals["cost"], g_trace, totals
