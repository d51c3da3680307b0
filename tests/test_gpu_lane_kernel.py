"""GPU parity of the lane-per-trajectory kernel (csrc/device/lane_ensemble.cu,
selected by lanes_per_traj=1 for networks with n' <= 255): one whole
trajectory per lane. Same bar as
test_gpu_parity.py — bit-exact states and statistics against the oracle on
the same injected Philox stream — over every feature the kernel carries."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    # name: (n, F, P, p, leaf, n_targets, fixed, seed, k, mgp)
    "c1": (100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605, 12, 8),
    "c3": (96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607, 12, 8),
    "c1_k16": (100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605, 16, 12),
    "tiny": (6, (1, 3), (1, 3), 0.25, 0.0, 2, False, 7, 3, 18),
    # >= 32 leading single-node alias groups: compact records, general
    # records of the single groups in the unstaged tail
    "singles": (120, (2, 3), (1, 4), 0.004, 0.0, 3, False, 21, 12, 8),
    # 5-parent functions and multi-member groups with wide tables
    "wide": (110, (1, 2), (3, 5), 0.003, 0.1, 2, False, 33, 10, 12),
    "n127": (127, (1, 4), (1, 4), 0.002, 0.0, 2, False, 5, 12, 8),
    "n64": (64, (1, 3), (1, 3), 0.01, 0.0, 2, False, 6, 12, 8),
    # eight state words (the widest network the lane kernel takes)
    "n250": (250, (1, 4), (1, 4), 0.002, 0.0, 3, False, 9, 12, 8),
}


def _setup(pb, case):
    n, f, p, pp, leaf, nt, fixed, seed, k, mgp = CASES[case]
    model, terms = pb.generate_model(n, f, p, pp, leaf, nt, fixed, seed)
    plan = pb.prepare(model, 1 << 25, k, mgp)
    return plan, plan.compile_predicate(terms)


@pytest.fixture(scope="module")
def cuda_ok(pb):
    assert pb.device_count() >= 1, "no CUDA device visible"


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("stream", [0, 1])
def test_lane_kernel_vs_oracle(pb, orc, cuda_ok, case, stream):
    plan, pred = _setup(pb, case)
    assert plan.n_kept <= 255
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    n_traj, n_steps = 300, 1500  # 300: the last warp is partial
    st, cnt = eng.simulate(seed=42, n_traj=n_traj, n_steps=n_steps, pred=pred, stream=stream)
    ost, ocnt = orc.simulate(plan.view, 42, 0, n_traj, n_steps, pred=pred, stream=stream)
    assert np.array_equal(cnt, ocnt)
    assert np.array_equal(st, ost)
    assert eng.info()["lanes_per_traj"] == 1


@pytest.mark.parametrize("placement", ["global", "core", "tables", "all", "core_pert"])
def test_lane_kernel_placements(pb, orc, cuda_ok, placement):
    plan, pred = _setup(pb, "singles")
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1, placement=placement)
    for stream in (0, 1):
        st, cnt = eng.simulate(seed=9, n_traj=64, n_steps=500, pred=pred, stream=stream)
        ost, ocnt = orc.simulate(plan.view, 9, 0, 64, 500, pred=pred, stream=stream)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


@pytest.mark.parametrize("case", ["c3", "singles"])
def test_lane_kernel_fp64_alias_path(pb, orc, cuda_ok, case):
    plan, pred = _setup(pb, case)
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    st, cnt = eng.simulate(seed=11, n_traj=96, n_steps=400, pred=pred, exact_alias=True)
    ost, ocnt = orc.simulate(plan.view, 11, 0, 96, 400, pred=pred)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_lane_kernel_edges_resume_and_initial_states(pb, orc, cuda_ok):
    plan, pred = _setup(pb, "c1")
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    for n_traj, n_steps in [(1, 1), (3, 0), (33, 257)]:
        st, cnt = eng.simulate(seed=3, n_traj=n_traj, n_steps=n_steps, pred=pred)
        ost, ocnt = orc.simulate(plan.view, 3, 0, n_traj, n_steps, pred=pred)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)
    full, _ = eng.simulate(seed=5, n_traj=70, n_steps=1000, pred=pred)
    half, _ = eng.simulate(seed=5, n_traj=70, n_steps=500, pred=pred)
    rest, _ = eng.simulate(seed=5, n_traj=70, n_steps=500, step_begin=500, states=half, pred=pred)
    assert np.array_equal(rest, full)
    a, _ = eng.simulate(seed=5, n_traj=40, n_steps=1000, pred=pred)
    b, _ = eng.simulate(seed=5, n_traj=30, n_steps=1000, traj_begin=40, pred=pred)
    assert np.array_equal(np.vstack([a, b]), full)
    rng = np.random.default_rng(0)
    n = plan.n_kept
    init = rng.integers(0, 2**63, size=(45, pb.state_words(n)), dtype=np.uint64)
    init[:, n // 64] &= np.uint64((1 << (n % 64)) - 1)
    init[:, n // 64 + 1:] = 0
    st, cnt = eng.simulate(seed=11, n_traj=45, n_steps=300, states=init, pred=pred)
    ost, ocnt = orc.simulate(plan.view, 11, 0, 45, 300, states=init, pred=pred)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


@pytest.mark.parametrize("kappa,mode", [(1, 0), (4, 1), (7, 2)])
def test_lane_kernel_transitions_and_series(pb, orc, cuda_ok, kappa, mode):
    plan, pred = _setup(pb, "c3")
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    n, steps = 70, 333
    tp_d = np.full(n, 2 | (1 << 2), np.uint8)
    tp_o = tp_d.copy()
    ser_d = np.zeros((n, 40), np.uint32)
    ser_o = ser_d.copy()
    st_d = st_o = None
    for call in range(3):
        st_d, c_d = eng.simulate(seed=4, n_traj=n, n_steps=steps, step_begin=call * steps,
                                 states=st_d, pred=pred, kappa=kappa,
                                 thin_mode=mode if call == 0 else 1, tprev=tp_d, series=ser_d,
                                 series_bit0=1 + call * steps, series_init=call == 0)
        st_o, c_o = orc.simulate_ex(plan.view, 4, 0, n, steps, states=st_o,
                                    step_begin=call * steps, pred=pred, kappa=kappa,
                                    thin_mode=mode if call == 0 else 1, tprev=tp_o,
                                    series=ser_o, series_bit0=1 + call * steps,
                                    series_init=call == 0)
        assert np.array_equal(c_d, c_o)
        assert np.array_equal(st_d, st_o)
        assert np.array_equal(tp_d, tp_o)
    assert np.array_equal(ser_d, ser_o)


@pytest.mark.parametrize("case", ["c1", "n127", "n250"])
def test_lane_kernel_node_counts(pb, orc, cuda_ok, case):
    plan, pred = _setup(pb, case)
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    st, cnt, nc = eng.simulate(seed=8, n_traj=100, n_steps=1000, pred=pred, node_counts=True)
    ost, ocnt, onc = orc.simulate(plan.view, 8, 0, 100, 1000, pred=pred, node_counts=True)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)
    assert np.array_equal(nc, onc)


@pytest.mark.parametrize("reduction", [False, True])
def test_lane_kernel_nodewise_plans(pb, orc, cuda_ok, reduction):
    """Method_old / Method_reduction plans (per-node Bernoulli perturbation)."""
    n, f, p, pp, leaf, nt, fixed, seed, _, _ = CASES["c1"]
    model, terms = pb.generate_model(n, f, p, pp, leaf, nt, fixed, seed)
    plan = pb.prepare_nodewise(model, reduction)
    if plan.n_kept > 255:
        pytest.skip("node-wise plan wider than the lane kernel")
    pred = plan.compile_predicate(terms)
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    for stream in (0, 1):
        st, cnt = eng.simulate(seed=2, n_traj=64, n_steps=600, pred=pred, stream=stream)
        ost, ocnt = orc.simulate(plan.view, 2, 0, 64, 600, pred=pred, stream=stream)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_auto_selection_large_ensemble(pb, orc, cuda_ok):
    """lanes_per_traj=0 picks the lane kernel for a small network once the
    ensemble reaches ~6 warps of trajectories per SM."""
    plan, pred = _setup(pb, "c3")
    eng = pb.GpuEnsemble(plan)
    n = 148 * 192 + 7
    st, cnt = eng.simulate(seed=6, n_traj=n, n_steps=40, pred=pred)
    assert eng.info()["lanes_per_traj"] == 1
    ost, ocnt = orc.simulate(plan.view, 6, 0, n, 40, pred=pred)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


@pytest.mark.parametrize("case", ["c1", "c1_k16", "n64"])
@pytest.mark.parametrize("stream", [0, 1])
def test_lane_kernel_queue_mode_statistics(pb, orc, cuda_ok, case, stream):
    """The rare-function-phase variant (per-lane queue of precomputed phase-A
    steps): thinned transitions, series, node counts and chained launches —
    queued steps never cross a launch, the statistics follow consume order."""
    plan, pred = _setup(pb, case)
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1)
    n, steps = 200, 517
    tp_d = np.full(n, 2 | (1 << 2), np.uint8)
    tp_o = tp_d.copy()
    ser_d = np.zeros((n, 3 * steps // 32 + 2), np.uint32)
    ser_o = ser_d.copy()
    st_d = st_o = None
    for call in range(3):
        st_d, c_d = eng.simulate(seed=11, n_traj=n, n_steps=steps, step_begin=call * steps,
                                 states=st_d, pred=pred, kappa=3,
                                 thin_mode=0 if call == 0 else 1, tprev=tp_d, series=ser_d,
                                 series_bit0=1 + call * steps, series_init=call == 0, stream=stream)
        assert eng.last_kernel().startswith("lane<queue") or eng.last_kernel().startswith("lane<scan"), \
            eng.last_kernel()
        st_o, c_o = orc.simulate_ex(plan.view, 11, 0, n, steps, states=st_o,
                                    step_begin=call * steps, pred=pred, kappa=3,
                                    thin_mode=0 if call == 0 else 1, tprev=tp_o,
                                    series=ser_o, series_bit0=1 + call * steps,
                                    series_init=call == 0, stream=stream)
        assert np.array_equal(c_d, c_o)
        assert np.array_equal(st_d, st_o)
        assert np.array_equal(tp_d, tp_o)
    assert np.array_equal(ser_d, ser_o)
    st, cnt, nc = eng.simulate(seed=8, n_traj=100, n_steps=700, pred=pred, node_counts=True, stream=stream)
    ost, ocnt, onc = orc.simulate(plan.view, 8, 0, 100, 700, pred=pred, node_counts=True, stream=stream)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt) and np.array_equal(nc, onc)
