"""Method_old / Method_reduction (the reference's node-by-node steppers,
engine.hpp:168-242) through the same flat-view machinery: the oracle on the
node-wise plan is bit-exact against the unmodified reference steppers on the
same stream (CPU), and the device against the oracle (GPU)."""
import numpy as np
import pytest

from helpers import config_text

CASES = [("c1", 0), ("c1", 1), ("c3", 0), ("c3", 1), ("c2", 1)]


def _setup(pb, ref, name, reduced):
    text, terms = config_text(name)
    plan = pb.prepare_nodewise(pb.parse_model(text), reduced)
    return text, plan, plan.compile_predicate(terms), ref.parse(text) if ref else None


@pytest.mark.parametrize("name,reduced", CASES)
@pytest.mark.parametrize("stream", [0, 1])
def test_oracle_nodewise_vs_reference(pb, orc, ref, name, reduced, stream):
    text, plan, pred, rm = _setup(pb, ref, name, reduced)
    n_traj, n_steps = (3, 300) if plan.n_kept > 500 else (8, 1500)
    a = rm.simulate_nodewise(reduced, plan.n_kept, 42, 5, n_traj, n_steps, pred=pred,
                             stream=stream, node_counts=True, step_begin=3)
    b = orc.simulate(plan.view, 42, 5, n_traj, n_steps, pred=pred, stream=stream,
                     node_counts=True, step_begin=3)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1][:, :2], b[1][:, :2])  # steps, hits
    assert np.array_equal(a[2], b[2])


def test_nodewise_plan_shape(pb):
    text, _ = config_text("c1")
    m = pb.parse_model(text)
    old = pb.prepare_nodewise(m, False)
    red = pb.prepare_nodewise(m, True)
    grp = pb.prepare(m, 1 << 25, 12, 8)
    assert old.n_kept == m.n and red.n_kept == grp.n_kept
    assert old.view.pert_mode == 1 and old.view.has_leaf == 0 and old.t == 1.0
    assert red.view.has_leaf == 1 and red.t == grp.t


@pytest.mark.gpu
@pytest.mark.parametrize("name,reduced", CASES + [("c5", 1)])
@pytest.mark.parametrize("stream", [0, 1])
def test_device_nodewise_vs_oracle(pb, orc, name, reduced, stream):
    text, plan, pred, _ = _setup(pb, None, name, reduced)
    eng = pb.GpuEnsemble(plan)
    n_traj, n_steps = (64, 300) if plan.n_kept > 500 else (200, 1000)
    st, cnt, nc = eng.simulate(seed=7, n_traj=n_traj, n_steps=n_steps, pred=pred, stream=stream,
                               node_counts=True)
    ost, ocnt, onc = orc.simulate(plan.view, 7, 0, n_traj, n_steps, pred=pred, stream=stream,
                                  node_counts=True)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt) and np.array_equal(nc, onc)
