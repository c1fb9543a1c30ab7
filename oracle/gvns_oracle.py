"""CPU restatement of the reference's shake / worker rounds (gvns.py:88-174).

TEST INFRASTRUCTURE ONLY: a round backend for paper_1704_05132_b200.sharded
that the gloo tests use in place of the GPU.  Shaking follows
gvns.py:101-137 with the numpy RNG restatement (numpy_rng.py) and the VND is
the C oracle's lockstep loop (remlot_oracle.c)."""

import numpy as np

import numpy_rng
import oracle

_U64 = (1 << 64) - 1


def shake(oi, sm, sr, init, k, rng):
    """gvns.py:101-137 on (K x T bool) rows; oi = oracle.OracleInstance."""
    K, T = sm.shape
    KT = K * T
    k_eff = min(k, 2 * KT)

    def flip(m, r, pos):
        tgt = m if pos < KT else r
        kk, t = divmod(pos % KT, T)
        tgt[kk, t] = not tgt[kk, t]

    for _ in range(50):
        pos = rng.choice_noreplace(2 * KT, k_eff)
        m, r = sm.copy(), sr.copy()
        for p in pos:
            flip(m, r, int(p))
        if oracle.evaluate(oi, m, r) != oracle.INFEASIBLE:
            return m, r
    m, r = sm.copy(), sr.copy()
    diffs = list(np.flatnonzero(m != init[0])) + list(np.flatnonzero(r != init[1]) + KT)
    diffs = [int(x) for x in diffs]
    rng.shuffle(diffs)
    for i, p in enumerate(diffs, start=1):
        flip(m, r, p)
        if i >= k_eff and oracle.evaluate(oi, m, r) != oracle.INFEASIBLE:
            return m, r
    return init[0].copy(), init[1].copy()


class OracleRounds:
    """sharded_gvns round backend on the CPU (torch CPU tensors for gloo)."""

    device = "cpu"

    def __init__(self, inst):
        import torch
        self.torch = torch
        self.oi = oracle.OracleInstance(inst)
        self.K, self.T = inst.products, inst.periods
        self.init = oracle.initial_solution(self.oi)

    def initial_solution(self):
        return self.init[0].copy(), self.init[1].copy()

    def begin(self, workers, worker_offset, config, sm, sr, batch=1):
        self.W, self.w0, self.cfg = workers, worker_offset, config
        self.sm, self.sr = np.asarray(sm, bool).copy(), np.asarray(sr, bool).copy()
        self.last = []
        return oracle.evaluate(self.oi, self.sm, self.sr)

    def run_local(self, round0, strength, nb):
        """Rounds round0 .. round0+nb-1 from the current incumbent with the
        strengths of a non-improving run (sharded_gvns batches)."""
        self.last = []
        k = strength
        for j in range(nb):
            self.last.append(self.round(round0 + j, k))
            k = 1 if k >= self.cfg.k_max else k + 1
        return [(c, w) for c, w, _ in self.last]

    def export(self, jr):
        return self.last[jr][2]

    def plan_buffer(self):
        return self.torch.zeros(2 * self.K * self.T, dtype=self.torch.uint8)

    def round(self, round_index, strength):
        best = None
        for i in range(self.W):
            w = self.w0 + i
            rng = numpy_rng.Philox.from_entropy((self.cfg.seed & _U64, round_index, w))
            m, r = shake(self.oi, self.sm, self.sr, self.init, strength, rng)
            m, r, cost, _, _ = oracle.vnd(self.oi, m, r, self.cfg.k_vnd_max)
            if best is None or cost < best[0]:
                best = (cost, w, m, r)
        cost, w, m, r = best
        plan = self.torch.from_numpy(np.concatenate([m.ravel(), r.ravel()]).astype(np.uint8))
        return cost, w, plan

    def adopt(self, plan, cost):
        a = plan.numpy().astype(bool)
        KT = self.K * self.T
        self.sm = a[:KT].reshape(self.K, self.T).copy()
        self.sr = a[KT:].reshape(self.K, self.T).copy()

    def incumbent(self):
        return self.sm.copy(), self.sr.copy()
