"""The C-ABI device group (pbn_group_*, csrc/group.cpp): one ensemble over
several GPUs with ONE ncclAllReduce of the pooled counts and per-node
one-counts. The GPU box has one device, so the group runs with one member
(ncclCommInitAll over [0]; a one-rank ncclCommInitRank): the sharding,
pooling kernels and the collective run for real, and the results must equal
the single-device engine's and the oracle's (the multi-rank sharding logic
is covered on CPU by tests/test_sharding.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan(pb, k=16):
    model, terms = pb.generate_model(1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606)
    plan = pb.prepare(model, 1 << 25, k, 8)
    return plan, plan.compile_predicate(terms)


@pytest.mark.parametrize("node_counts", [False, True])
def test_group_of_one_equals_engine_and_oracle(pb, orc, node_counts):
    plan, pred = _plan(pb)
    grp = pb.GpuGroup(plan, devices=[0])
    assert (grp.n_members, grp.nranks, grp.first_rank) == (1, 1, 0)
    n_traj, n_steps = 96, 300
    st, cnt, tot, ntot = grp.simulate(42, n_traj, n_steps, traj_begin=5, pred=pred,
                                      node_counts=node_counts)
    eng = pb.GpuEnsemble(plan)
    est, ecnt = eng.simulate(42, n_traj, n_steps, traj_begin=5, pred=pred)
    assert np.array_equal(st, est) and np.array_equal(cnt, ecnt)
    assert np.array_equal(tot, ecnt.sum(axis=0, dtype=np.uint64))
    assert grp.member_kernel(0) == eng.last_kernel()
    if node_counts:
        _, ocnt, onc = orc.simulate(plan.view, 42, 5, n_traj, n_steps, pred=pred, node_counts=True)
        assert np.array_equal(cnt, ocnt)
        assert np.array_equal(ntot, onc.sum(axis=0, dtype=np.uint64))


def test_group_rank_mode_one_rank(pb, orc):
    plan, pred = _plan(pb, k=12)
    grp = pb.GpuGroup(plan, device=0, nranks=1, rank=0, nccl_id=pb.nccl_unique_id())
    st, cnt, tot, _ = grp.simulate(7, 40, 200, pred=pred, stream=pb.STREAM_U32)
    ost, ocnt = orc.simulate(plan.view, 7, 0, 40, 200, pred=pred, stream=pb.STREAM_U32)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)
    assert np.array_equal(tot, ocnt.sum(axis=0, dtype=np.uint64))


def test_group_resume_and_refusals(pb):
    plan, pred = _plan(pb, k=12)
    grp = pb.GpuGroup(plan, devices=[0])
    st, _, t1, _ = grp.simulate(3, 33, 100, pred=pred)
    st2, _, t2, _ = grp.simulate(3, 33, 150, step_begin=100, states=st, pred=pred)
    full, _, t, _ = grp.simulate(3, 33, 250, pred=pred)
    assert np.array_equal(st2, full)
    assert int(t1[1]) + int(t2[1]) == int(t[1])  # hits add up
    with pytest.raises(pb.UsageError):
        grp.simulate(3, 33, 10, states=np.zeros((5, grp.words), np.uint64))
