"""The BASELINE configurations at their FULL stated shapes (trajectories x
steps of workloads/workloads.json), on the kernels the bench runs, checked
through properties that do not depend on the size:

* resume invariance — one launch of T steps equals two chained launches of
  T/2 (final states identical, step-class and hit counts add up);
* shard invariance — the ensemble in one launch equals its two halves
  launched separately (what the multi-GPU sharding relies on);
* class checksum — every step is exactly one of perturbed / leaf no-op /
  function phase, and with kappa = 1 every step is one predicate transition;
* spot trajectories — a few whole trajectories of the full-length run
  replayed by the oracle restatement on the CPU, bit-exact.

c5 runs the bench's slice of its 1e6 steps (1e5 per bench step, p = 0.1 and
1e-3: the PF and the general kernels)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# name: (config, p override, steps or None = the config's, oracle trajectories, shard check)
CASES = {
    "c2": ("c2", None, None, 3, True),
    "c1": ("c1", None, None, 8, True),
    "c4": ("c4", None, None, 1, False),
    "c5_p1e-1": ("c5", 0.1, 100000, 2, True),
    "c5_p1e-3": ("c5", 0.001, 100000, 1, False),
}


@pytest.mark.parametrize("name", list(CASES))
def test_full_size_properties(pb, orc, name):
    from paper_1605_00854_b200.configs import CONFIGS

    cfg, p, steps, n_orc, shard = CASES[name]
    w = CONFIGS[cfg]
    model, terms = w.model(p)
    plan = pb.prepare(pb.parse_model(model.serialize()), w.theta, w.k_max, w.mgp)
    pred = plan.compile_predicate(terms)
    n, T = w.n_traj, steps or w.n_steps
    eng = pb.GpuEnsemble(plan)
    full, cf = eng.simulate(seed=42, n_traj=n, n_steps=T, pred=pred)
    kernel = eng.last_kernel()
    assert kernel == eng.plan_launch(n, pb.STREAM_U53)  # the bench's launch for this ensemble

    # class checksum (PBN_C_* of include/pbn_b200.h)
    assert np.all(cf[:, 0] == T)
    assert np.all(cf[:, 6] + cf[:, 7] <= T)            # the rest are leaf no-ops
    if not plan.view.has_leaf:
        assert np.all(cf[:, 6] + cf[:, 7] == T)
    if len(pred[0]):
        assert np.all(cf[:, 2] + cf[:, 3] + cf[:, 4] + cf[:, 5] == T)  # kappa = 1: one transition per step
        assert np.all(cf[:, 3] + cf[:, 5] == cf[:, 1])                 # transitions into 1 = hits

    # resume invariance
    half, c1 = eng.simulate(seed=42, n_traj=n, n_steps=T // 2, pred=pred)
    rest, c2 = eng.simulate(seed=42, n_traj=n, n_steps=T - T // 2, step_begin=T // 2, states=half,
                            pred=pred)
    assert eng.last_kernel() == kernel
    assert np.array_equal(rest, full)
    for f in (0, 1, 6, 7):
        assert np.array_equal(c1[:, f] + c2[:, f], cf[:, f])

    # shard invariance
    if shard:
        a, ca = eng.simulate(seed=42, n_traj=n // 2, n_steps=T, pred=pred)
        b, cb = eng.simulate(seed=42, n_traj=n - n // 2, n_steps=T, traj_begin=n // 2, pred=pred)
        assert np.array_equal(np.vstack([a, b]), full)
        assert np.array_equal(np.vstack([ca, cb]), cf)

    # spot trajectories against the oracle, full length
    t0 = (n * 5) // 7
    ost, ocnt = orc.simulate(plan.view, 42, t0, n_orc, T, pred=pred)
    assert np.array_equal(full[t0:t0 + n_orc], ost)
    assert np.array_equal(cf[t0:t0 + n_orc], ocnt)
