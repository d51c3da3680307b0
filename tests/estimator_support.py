"""Test backend: the oracle restatement as the stepper under the product's
C++ estimator (pbn_estimate_with_backend) — test infrastructure."""
import numpy as np

import paper_1605_00854_b200 as pb


class OracleEnsemble:
    def __init__(self, orc, view, pred, seed, n_traj, stream=0, traj_begin=0, cap=1 << 22):
        self.orc, self.view, self.pred = orc, view, pred
        self.seed, self.n, self.stream, self.tb = seed, n_traj, stream, traj_begin
        self.cap = cap
        self.states = np.zeros((n_traj, view.n_kept // 64 + 1), np.uint64)
        self.tprev = np.zeros(n_traj, np.uint8)
        self.series = np.zeros((n_traj, (cap + 31) // 32), np.uint32)

    def run(self, s0, n, kappa, mode, bit0, init):
        st, cnt = self.orc.simulate_ex(self.view, self.seed, self.tb, self.n, n, states=self.states,
                                       step_begin=s0, pred=self.pred, stream=self.stream,
                                       kappa=kappa, thin_mode=mode, tprev=self.tprev,
                                       series=self.series if bit0 is not None else None,
                                       series_bit0=bit0 or 0, series_init=init)
        self.states = st
        return cnt.sum(axis=0)

    def stats(self, kappa, length):
        return pb.series_stats_host(self.series, length, kappa)

    def estimate(self, req):
        return pb.estimate_with_backend(req, self.n, self.run, self.stats, self.cap)
