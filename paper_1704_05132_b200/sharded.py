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


def merge_shards(parts, k_max=4):
    """The job's (trace, totals) from every shard's (trace, stats) in one
    process -- what ``combine`` computes with collectives (used to pin the
    multi-rank result on one device and in tests)."""
    starts = [int(t[0]) for t, _ in parts]
    decs = [[int(t[i]) - int(t[i + 1]) for i in range(len(t) - 1)] for t, _ in parts]
    n_pass = max(len(d) for d in decs)
    vec = [0] * n_pass
    for d in decs:
        for i, x in enumerate(d):
            vec[i] += x
    start_total = INFEASIBLE if INFEASIBLE in starts else sum(starts)
    g_trace = [start_total]
    for d in vec:
        g_trace.append(g_trace[-1] - d)
    sweeps = n_pass // k_max
    ref = sum(int(st.get("evals_reference", 0)) - (len(d) // k_max) * int(st.get("ntot_sum", 0))
              for d, (_, st) in zip(decs, parts))
    ntot = sum(int(st.get("ntot_sum", 0)) for _, st in parts)
    totals = dict(start_cost=start_total, cost=g_trace[-1], sweeps=sweeps,
                  evals=sum(int(st.get("evals", 0)) for _, st in parts),
                  moves=sum(int(st.get("moves", 0)) for _, st in parts),
                  evals_reference=ref + sweeps * ntot)
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


# ---------------------------------------------------------------- replicas

class DeviceRounds:
    """Round backend of ``sharded_gvns`` on this rank's GPU (gvns_impl.cuh):
    speculative local batches (rl_gvns_run_local), the winning candidate's
    export and the job winner's import."""

    def __init__(self, inst):
        import torch
        from . import _native
        self.torch = torch
        self.dev = _native.DeviceInstance(inst)
        self.KT = inst.products * inst.periods
        self.buf = torch.empty(2 * self.KT, dtype=torch.uint8, device="cuda")
        self.device = "cuda"

    def begin(self, workers, worker_offset, config, sm, sr, batch=1):
        return self.dev.gvns_begin(workers, config.k_max, config.k_vnd_max, config.seed, sm, sr,
                                   worker_offset=worker_offset, batch=batch)

    def run_local(self, round0, strength, nb):
        self.dev.gvns_set_strength(strength)
        return self.dev.gvns_run_local(round0, nb)

    def export(self, jr):
        self.dev.gvns_export(jr, self.buf.data_ptr())
        return self.buf

    def plan_buffer(self):
        return self.buf

    def adopt(self, plan_tensor, cost):
        self.dev.gvns_import(plan_tensor.data_ptr(), cost)

    def incumbent(self):
        sm, sr, info = self.dev.gvns_state(0)
        return sm, sr


def _batch_rounds(local_workers):
    """Rounds per speculative batch of a rank: enough worker slots (about
    512) to fill its device, at most 4 (like gvns._batch)."""
    return max(1, min(4, 512 // max(local_workers, 1)))


def sharded_gvns(inst, config, group=None, backend=None, start_plan=None, batch=None):
    """GVNS whose W workers are split in contiguous blocks over the ranks
    (BASELINE config 5: 1,024 replicas over 8 GPUs), in speculative batches
    of rounds with one collective per batch.

    Each rank runs rounds r0 .. r0+nb-1 of its worker block at once, every
    round shaking the current incumbent with the strength it has if the
    rounds before it do not improve (round RNG streams depend only on (seed,
    round, worker), gvns.py:88-90).  One all-gather carries every rank's
    per-round best (cost, global worker) and rank 0's budget decision; all
    ranks then walk the rounds in order, take each round's minimum (lowest
    worker on ties, gvns.py:170-174) and stop at the first one that improves
    the incumbent (gvns.py:207-215): its winner broadcasts the candidate and
    every rank adopts it; the rounds after it are discarded and re-run from
    the new incumbent by the next batch.  The trajectory is therefore the
    sequential reference's, round for round.  The batch size adapts like
    the single-GPU loop: 1 after an accepted round, doubled (up to ``batch``)
    after a batch without one.  The wall-clock budget is checked between
    batches (overshoot at most one batch).
    Returns the reference's GvnsResult on every rank."""
    import time

    import torch
    import torch.distributed as dist

    from .gvns import GvnsResult, next_strength
    from .plan import SetupPlan

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    be = backend if backend is not None else DeviceRounds(inst)
    dev = getattr(be, "device", "cpu")
    W = config.workers
    w_lo, w_hi = shard_bounds(W, rank, world)
    local = w_hi - w_lo
    B = batch if batch is not None else _batch_rounds(-(-W // world))
    start = time.monotonic()
    if start_plan is None:
        if hasattr(be, "initial_solution"):
            sm0, sr0 = be.initial_solution()
        else:
            from .plan import initial_solution
            p = initial_solution(inst)
            sm0, sr0 = p.setup_m, p.setup_r
    else:
        sm0, sr0 = start_plan.setup_m, start_plan.setup_r
    inc_cost = be.begin(max(local, 1), w_lo, config, sm0, sr0, batch=B)
    strength, rounds, nb = 1, 0, 1
    BIG = (1 << 63) - 1
    cap = config.max_rounds

    def keep_going(done):   # rank 0's budget check before a batch (gvns.py:197-199)
        return not (time.monotonic() - start > config.t_max or (cap is not None and done >= cap))

    go = torch.tensor([1 if rank != 0 or keep_going(0) else 0], dtype=torch.int64, device=dev)
    dist.broadcast(go, src=0, group=group)
    going = int(go[0]) == 1
    while going:
        want = nb if cap is None else max(1, min(nb, cap - rounds))
        res = be.run_local(rounds, strength, want) if local else [(BIG, BIG)] * want
        # one all-gather per batch: [valid rounds, go, (cost, worker) x want]
        mine = torch.full((2 + 2 * want,), BIG, dtype=torch.int64)
        mine[0] = len(res)
        # rank 0's wall-clock decision for the next batch rides along
        # (gvns.py:197-199; the round cap is checked by every rank below)
        mine[1] = 1 if rank != 0 or time.monotonic() - start <= config.t_max else 0
        for j, (c, w) in enumerate(res):
            mine[2 + 2 * j] = c
            mine[3 + 2 * j] = w
        mine = mine.to(dev)
        allb = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allb, mine, group=group)
        rows = [t.tolist() for t in allb]
        n_use = min(int(r[0]) for r in rows)
        win = None
        for j in range(n_use):
            pairs = [(int(r[2 + 2 * j]), int(r[3 + 2 * j])) for r in rows]
            best = min(pairs)
            if best[0] < inc_cost:
                win = (j, best, min(q for q in range(world) if pairs[q] == best))
                break
            strength = next_strength(strength, False, config.k_max)
        if win is not None:
            j, (best_cost, _), src = win
            plan = be.export(j) if rank == src else be.plan_buffer()
            dist.broadcast(plan, src=src, group=group)
            be.adopt(plan, best_cost)
            inc_cost = best_cost
            strength = next_strength(strength, True, config.k_max)
            rounds += j + 1
            nb = 1
        else:
            rounds += n_use
            nb = 1 if n_use == 0 else min(2 * nb, B)
        going = int(rows[0][1]) == 1 and (cap is None or rounds < cap)
    sm, sr = be.incumbent()
    return GvnsResult(SetupPlan(sm, sr), inc_cost, rounds, time.monotonic() - start,
                      rounds * W)
