"""GPU parity: the sm_100a ensemble kernel, called through the C-ABI, against
the oracle restatement (oracle/pbn_oracle.c, itself pinned to the unmodified
reference in test_oracle_pins.py) on the same injected Philox stream.

Bar: bit-exact final states (engine order, reference word layout) and exact
statistics (hits, predicate transitions, step classes) per trajectory.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    # name: (n, F, P, p, leaf, n_targets, fixed, seed, k, mgp)
    "c1": (100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605, 12, 8),
    "c2": (1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606, 12, 8),
    "c3": (96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607, 12, 8),
    "c5": (2000, (1, 3), (1, 4), 0.01, 0.0, 2, False, 1609, 12, 8),
    "c1_k16": (100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605, 16, 12),
    "tiny": (6, (1, 3), (1, 3), 0.25, 0.0, 2, False, 7, 3, 18),
    # n' <= 1023 with 5-parent functions: exercises the register/shuffle gather's 5th slot
    "p5": (900, (1, 4), (1, 5), 0.002, 0.0, 2, False, 11, 12, 8),
    # k=16 with two phase-A blocks per lane and frequent flips: the word-per-block phase A
    "c5_k16": (2000, (1, 3), (1, 4), 0.1, 0.0, 2, False, 1609, 16, 8),
    # 1023 < n' <= 2047 with 5-parent functions: two state words per lane (RG2)
    "p5w": (1500, (1, 3), (1, 5), 0.001, 0.0, 2, False, 12, 12, 8),
    "c4": (5000, (1, 4), (1, 5), 0.0001, 0.0, 2, False, 1608, 12, 12),
    # n' > 2047 with single-node groups of <= 4 functions: the compact
    # shared-memory-gather records (GM 4, dev_plan.h sgrp/sfn)
    "big_scl": (2600, (1, 4), (1, 5), 0.0002, 0.0, 2, False, 21, 16, 8),
}


def _setup(pb, case):
    n, f, p, pp, leaf, nt, fixed, seed, k, mgp = CASES[case]
    model, terms = pb.generate_model(n, f, p, pp, leaf, nt, fixed, seed)
    plan = pb.prepare(model, 1 << 25, k, mgp)
    return plan, plan.compile_predicate(terms)


@pytest.fixture(scope="module")
def cuda_ok(pb):
    assert pb.device_count() >= 1, "no CUDA device visible"


@pytest.mark.parametrize("case", ["c1", "c3", "c2", "c5", "c1_k16", "c5_k16", "p5", "p5w", "c4",
                                  "big_scl"])
@pytest.mark.parametrize("stream", [0, 1])
def test_bit_exact_vs_oracle(pb, orc, cuda_ok, case, stream):
    plan, pred = _setup(pb, case)
    n_traj, n_steps = (96, 400) if plan.n_kept > 500 else (256, 2000)
    if plan.n_kept > 3000:
        n_traj, n_steps = 40, 150
    eng = pb.GpuEnsemble(plan)
    st, cnt = eng.simulate(seed=42, n_traj=n_traj, n_steps=n_steps, pred=pred, stream=stream)
    ost, ocnt = orc.simulate(plan.view, 42, 0, n_traj, n_steps, pred=pred, stream=stream)
    assert np.array_equal(cnt, ocnt)
    assert np.array_equal(st, ost)
    assert eng.last_launches() == 1


@pytest.mark.parametrize("lpt", [1, 2, 4, 8, 16, 32])
def test_lanes_per_trajectory_invariance(pb, orc, cuda_ok, lpt):
    plan, pred = _setup(pb, "c1")
    eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
    st, cnt = eng.simulate(seed=7, n_traj=100, n_steps=1500, pred=pred)
    ost, ocnt = orc.simulate(plan.view, 7, 0, 100, 1500, pred=pred)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


@pytest.mark.parametrize("lpt", [8, 16])
def test_compact_plan_on_fallback_kernels(pb, orc, cuda_ok, lpt):
    """A plan with compact single-node records (its single groups' general
    records moved to the unstaged tail) run by the non-compact kernels."""
    plan, pred = _setup(pb, "c2")
    eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
    for stream in (0, 1):
        st, cnt = eng.simulate(seed=13, n_traj=48, n_steps=200, pred=pred, stream=stream)
        ost, ocnt = orc.simulate(plan.view, 13, 0, 48, 200, pred=pred, stream=stream)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


@pytest.mark.parametrize("placement", ["global", "core", "tables", "all", "core_pert"])
def test_placement_invariance(pb, orc, cuda_ok, placement):
    plan, pred = _setup(pb, "c2")
    eng = pb.GpuEnsemble(plan, placement=placement)
    for stream in (0, 1):
        st, cnt = eng.simulate(seed=9, n_traj=64, n_steps=300, pred=pred, stream=stream)
        ost, ocnt = orc.simulate(plan.view, 9, 0, 64, 300, pred=pred, stream=stream)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_resume_and_shard_invariance(pb, cuda_ok):
    """Counter-based stream: (seed, trajectory, step) fixes every draw, so
    chained launches and any trajectory split give identical results."""
    plan, pred = _setup(pb, "c3")
    eng = pb.GpuEnsemble(plan)
    full, cfull = eng.simulate(seed=5, n_traj=200, n_steps=1000, pred=pred)
    half, c1 = eng.simulate(seed=5, n_traj=200, n_steps=500, pred=pred)
    rest, c2 = eng.simulate(seed=5, n_traj=200, n_steps=500, step_begin=500, states=half, pred=pred)
    assert np.array_equal(rest, full)
    # hits/transitions add up across the split (transition across the seam is
    # counted by the second launch from its input state)
    assert np.array_equal(c1[:, 1] + c2[:, 1], cfull[:, 1])
    assert np.array_equal(c1[:, 6] + c2[:, 6], cfull[:, 6])
    a, _ = eng.simulate(seed=5, n_traj=120, n_steps=1000, pred=pred)
    b, _ = eng.simulate(seed=5, n_traj=80, n_steps=1000, traj_begin=120, pred=pred)
    assert np.array_equal(np.vstack([a, b]), full)


@pytest.mark.parametrize("case", ["c2", "c5", "c3"])
def test_integer_alias_path_vs_fp64_path(pb, orc, cuda_ok, case):
    """U53 combined-function choices: the integer fast path (dev_plan.h a53)
    and the forced FP64 path give the oracle's results."""
    plan, pred = _setup(pb, case)
    eng = pb.GpuEnsemble(plan)
    fast = eng.simulate(seed=11, n_traj=64, n_steps=300, pred=pred)
    exact = eng.simulate(seed=11, n_traj=64, n_steps=300, pred=pred, exact_alias=True)
    ost, ocnt = orc.simulate(plan.view, 11, 0, 64, 300, pred=pred)
    for st, cnt in (fast, exact):
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_groups_beyond_integer_alias_range(pb, orc, cuda_ok):
    """Groups with more than 2048 combined functions always take the FP64 path."""
    model, terms = pb.generate_model(8, (12, 16), (1, 1), 0.02, 0.0, 2, False, 0)
    plan = pb.prepare(model, 1 << 40, 12, 18)
    assert int(np.max(plan.flat().grp_alias_size)) > 2048
    pred = plan.compile_predicate(terms)
    eng = pb.GpuEnsemble(plan)
    for stream in (0, 1):
        st, cnt = eng.simulate(seed=4, n_traj=128, n_steps=2000, pred=pred, stream=stream)
        ost, ocnt = orc.simulate(plan.view, 4, 0, 128, 2000, pred=pred, stream=stream)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_tiny_network_and_edge_sizes(pb, orc, cuda_ok):
    plan, pred = _setup(pb, "tiny")
    eng = pb.GpuEnsemble(plan)
    for n_traj, n_steps in [(1, 1), (3, 0), (33, 257)]:
        st, cnt = eng.simulate(seed=3, n_traj=n_traj, n_steps=n_steps, pred=pred)
        ost, ocnt = orc.simulate(plan.view, 3, 0, n_traj, n_steps, pred=pred)
        assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_nonzero_initial_states(pb, orc, cuda_ok):
    plan, pred = _setup(pb, "c2")
    rng = np.random.default_rng(0)
    words = pb.state_words(plan.n_kept)
    init = rng.integers(0, 2**63, size=(50, words), dtype=np.uint64)
    # clear bits >= n_kept (the reference keeps them zero, bitstate.hpp:10)
    n = plan.n_kept
    init[:, n // 64] &= np.uint64((1 << (n % 64)) - 1)
    init[:, n // 64 + 1:] = 0
    eng = pb.GpuEnsemble(plan)
    st, cnt = eng.simulate(seed=11, n_traj=50, n_steps=200, states=init, pred=pred)
    ost, ocnt = orc.simulate(plan.view, 11, 0, 50, 200, states=init, pred=pred)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_philox_device_matches_oracle(pb, orc, cuda_ok):
    rng = np.random.default_rng(1)
    ctr = rng.integers(0, 2**32, size=(64, 4), dtype=np.uint64).astype(np.uint32)
    seed = 0x1234567890ABCDEF
    dev = pb.philox_kat_device(ctr, seed)
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], np.uint32)
    for i in range(len(ctr)):
        assert np.array_equal(dev[i], orc.philox(ctr[i], key))


@pytest.mark.parametrize("kappa,mode", [(1, 0), (3, 0), (4, 1), (7, 2), (16, 1)])
def test_sampled_transitions_and_series_vs_oracle(pb, orc, cuda_ok, kappa, mode):
    """Estimator statistics: kappa-thinned transitions with the sample and its
    phase carried in tprev across calls, and the recorded predicate series."""
    plan, pred = _setup(pb, "c3")
    eng = pb.GpuEnsemble(plan)
    n, steps = 70, 333
    tp_d = np.full(n, 2 | (1 << 2), np.uint8)
    tp_o = tp_d.copy()
    ser_d = np.zeros((n, 40), np.uint32)
    ser_o = ser_d.copy()
    st_d = st_o = None
    for call in range(3):
        st_d, c_d = eng.simulate(seed=4, n_traj=n, n_steps=steps, step_begin=call * steps,
                                 states=st_d, pred=pred, kappa=kappa, thin_mode=mode if call == 0 else 1,
                                 tprev=tp_d, series=ser_d, series_bit0=1 + call * steps,
                                 series_init=call == 0)
        st_o, c_o = orc.simulate_ex(plan.view, 4, 0, n, steps, states=st_o, step_begin=call * steps,
                                    pred=pred, kappa=kappa, thin_mode=mode if call == 0 else 1,
                                    tprev=tp_o, series=ser_o, series_bit0=1 + call * steps,
                                    series_init=call == 0)
        assert np.array_equal(c_d, c_o)
        assert np.array_equal(st_d, st_o)
        assert np.array_equal(tp_d, tp_o)
    assert np.array_equal(ser_d, ser_o)


@pytest.mark.parametrize("case,lpt", [("c1", 0), ("c1", 4), ("c2", 0), ("c3", 8), ("c5", 0)])
def test_node_one_counts_vs_oracle(pb, orc, cuda_ok, case, lpt):
    """simulate()'s per-node one-counts (engine.hpp:378-379), incl. >255-step
    flushes and the plan-placement fallback when the counter planes need room."""
    plan, pred = _setup(pb, case)
    eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
    n, steps = (40, 600) if plan.n_kept > 500 else (100, 1000)
    st, cnt, nc = eng.simulate(seed=8, n_traj=n, n_steps=steps, pred=pred, node_counts=True)
    ost, ocnt, onc = orc.simulate(plan.view, 8, 0, n, steps, pred=pred, node_counts=True)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)
    assert np.array_equal(nc, onc)


@pytest.mark.parametrize("lpt", [4, 8, 16, 32])
@pytest.mark.parametrize("stream", [0, 1])
def test_word_phase_a_any_lanes_per_trajectory(pb, orc, cuda_ok, lpt, stream):
    """k=16 plan with frequent flips: the U53 word-per-block phase A on every
    sub-warp width (U32 keeps the per-draw path)."""
    plan, pred = _setup(pb, "c1_k16")
    eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
    st, cnt = eng.simulate(seed=21, n_traj=90, n_steps=800, pred=pred, stream=stream)
    ost, ocnt = orc.simulate(plan.view, 21, 0, 90, 800, pred=pred, stream=stream)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


@pytest.mark.parametrize("case", ["big_scl", "c4"])
def test_compact_large_network_kernel(pb, orc, cuda_ok, case):
    """GM 4 (compact sgrp/sfn records, shared-memory gathers) is the U53
    kernel for these plans; bit-exact with the fast path, the forced FP64
    path (every function phase redone exactly) and on U32 (GM 0)."""
    plan, pred = _setup(pb, case)
    assert pb.plan_layout(plan)["single_compact"] == 0
    eng = pb.GpuEnsemble(plan)
    n_traj, n_steps = (64, 120)
    for stream, exact in ((0, False), (0, True), (1, False)):
        st, cnt = eng.simulate(seed=9, n_traj=n_traj, n_steps=n_steps, pred=pred, stream=stream,
                               exact_alias=exact, traj_begin=77, step_begin=1000)
        gm = "smem_compact" if stream == 0 else "smem"
        assert f"gather={gm}," in eng.last_kernel(), eng.last_kernel()
        ost, ocnt = orc.simulate(plan.view, 9, 77, n_traj, n_steps, pred=pred, stream=stream,
                                 step_begin=1000)
        assert np.array_equal(cnt, ocnt)
        assert np.array_equal(st, ost)
        assert cnt[:, 6].sum() > 0  # function phases ran


@pytest.mark.parametrize("stream", [0, 1])
@pytest.mark.parametrize("pp", [0.0022, 0.004, 0.05])
def test_perturbation_dominated_kernel(pb, orc, cuda_ok, stream, pp):
    """PF kernel (p_fn < 0.02, k = 16, one phase-A block per lane): the state
    lives in registers between function phases. Launches whose steps are
    ~1.2 %, ~0.03 % and never function phases; predicate hits, kappa-thinned
    transitions, the recorded series and chained launches from carried states."""
    model, terms = pb.generate_model(2000, (1, 3), (1, 4), pp, 0.0, 2, False, 1609)
    plan = pb.prepare(model, 1 << 25, 16, 8)
    pred = plan.compile_predicate(terms)
    eng = pb.GpuEnsemble(plan)
    n, steps = 70, 700
    tp_d = np.full(n, 2 | (1 << 2), np.uint8)
    tp_o = tp_d.copy()
    ser_d = np.zeros((n, 3 * steps // 32 + 2), np.uint32)
    ser_o = ser_d.copy()
    st_d = st_o = None
    fn_steps = 0
    for call in range(3):
        st_d, c_d = eng.simulate(seed=4, n_traj=n, n_steps=steps, step_begin=call * steps,
                                 states=st_d, pred=pred, kappa=3, thin_mode=0 if call == 0 else 1,
                                 tprev=tp_d, series=ser_d, series_bit0=1 + call * steps,
                                 series_init=call == 0, stream=stream)
        if stream == 0:
            assert "pa_prefetch" in eng.last_kernel(), eng.last_kernel()
        st_o, c_o = orc.simulate_ex(plan.view, 4, 0, n, steps, states=st_o, step_begin=call * steps,
                                    pred=pred, kappa=3, thin_mode=0 if call == 0 else 1,
                                    tprev=tp_o, series=ser_o, series_bit0=1 + call * steps,
                                    series_init=call == 0, stream=stream)
        assert np.array_equal(c_d, c_o)
        assert np.array_equal(st_d, st_o)
        assert np.array_equal(tp_d, tp_o)
        fn_steps += int(c_o[:, 6].sum())
    assert np.array_equal(ser_d, ser_o)
    if pp == 0.0022:
        assert fn_steps > 500  # the store / exact function phase / reload path ran
