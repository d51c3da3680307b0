"""Forced-draw replay on the device (pbn_gpu_run_scripted): the reference
tests' scripted_rng traces (tests/oracles.hpp:235-254, test_engine.cpp:89-153)
run through the sub-warp kernel built with scripted draw blocks, checked
against the oracle's and — where oracle/_ref travelled — the unmodified
reference's own scripted step, draw for draw (states and consumed counts)."""
import math
import os

import numpy as np
import pytest

from helpers import config_text

pytestmark = pytest.mark.gpu

IDENTITY4 = ("pbn 4\nperturbation 0.2\nnode x0\n  f 1 10 x0\nnode x1\n  f 1 10 x1\n"
             "node x2\n  f 1 10 x2\nnode x3\n  f 1 10 x3\n")


def _find_uniform(cut, alias, want):
    """A single uniform that makes the table emit `want` (test_engine.cpp:133-143)."""
    n = len(cut)
    for cell in range(n):
        if cut[cell] > 0 and cell == want:
            return (cell + cut[cell] * 0.5) / n
        if cut[cell] < 1 and alias[cell] == want:
            return (cell + cut[cell] + (1 - cut[cell]) * 0.5) / n
    raise AssertionError("pattern not reachable")


def _replay_cpu(step, s0, script, n_steps):
    """n_steps scripted steps with a wrapping script (scripted_rng semantics):
    `step(state, uniforms) -> (state, used)` is one forced step."""
    s, pos, n = np.array(s0, np.uint64), 0, len(script)
    for _ in range(n_steps):
        window = [script[(pos + i) % n] for i in range(n)]  # at most n draws per step here
        s, used = step(s, window)
        pos += used
    return s, pos


def test_hand_traced_grouped_perturbation_on_device(pb, orc):
    """test_engine.cpp:115-153: force c = 0b01 in group 1 -> bit 2 flips, two
    draws consumed, no leaf check."""
    plan = pb.prepare(pb.parse_model(IDENTITY4), 1 << 20, 2, 18)
    f = plan.flat()
    assert f.pert_groups == 2 and f.pert_k == 2
    z, o = _find_uniform(f.pert_cut, f.pert_alias, 0), _find_uniform(f.pert_cut, f.pert_alias, 1)
    eng = pb.GpuEnsemble(plan)
    st, cnt, used = eng.simulate_scripted([z, o], 1)
    assert int(used[0]) == 2
    assert int(st[0, 0]) == 0b0100
    assert int(cnt[0, 7]) == 1 and int(cnt[0, 6]) == 0  # one perturbed step, no function phase
    assert eng.last_kernel().startswith("subwarp_script<")
    # no flip, no leaf (t = 1): identity functions keep the state; g + 1 draws
    s0 = np.array([[0b0110]], np.uint64)
    st, cnt, used = eng.simulate_scripted([z, z, 0.5], 3, states=s0)
    assert int(used[0]) == 9 and int(st[0, 0]) == 0b0110 and int(cnt[0, 6]) == 3


@pytest.mark.parametrize("case,k,mgp,n_steps", [("c1", 12, 8, 60), ("c1", 16, 8, 40),
                                                 ("c3", 16, 8, 40), ("c2", 16, 8, 6)])
def test_random_scripts_match_the_scripted_reference_step(pb, orc, case, k, mgp, n_steps):
    import oracle

    text, terms = config_text(case)
    plan = pb.prepare(pb.parse_model(text), 1 << 25, k, mgp)
    pred = plan.compile_predicate(terms)
    refplan = None
    if os.path.exists(oracle.REF_SO):
        refplan = oracle.Reference().parse(text).prepare(1 << 25, k, mgp)
    rng = np.random.default_rng(1000 * k + len(case) + n_steps)
    n_traj, per_step = 6, plan.flat().pert_groups + 1 + int((plan.flat().grp_alias_size > 0).sum())
    n_draws = per_step * n_steps  # never wraps inside a step; wraps are exercised below
    draws = rng.random((n_traj, n_draws))
    # draws in [0.5, 1) pick zero-heavy cells rarely; force quiet steps so that
    # function phases are common: most perturbation draws land in cells whose
    # pattern is 0 anyway at these p; a few rows also get 0.999 runs
    draws[1, : per_step * 3] = 0.999
    words = plan.n_kept // 64 + 1
    s0 = rng.integers(0, 2**63, size=(n_traj, words), dtype=np.uint64)
    s0[:, -1] &= np.uint64((1 << (plan.n_kept % 64)) - 1)
    eng = pb.GpuEnsemble(plan)
    st, cnt, used = eng.simulate_scripted(draws, n_steps, states=s0, pred=pred)
    for t in range(n_traj):
        es, epos = _replay_cpu(lambda s, u: orc.step_scripted(plan.view, s, u), s0[t], draws[t], n_steps)
        assert int(used[t]) == epos
        assert np.array_equal(st[t], es)
        if refplan is not None:
            rs, rpos = _replay_cpu(refplan.step_scripted, s0[t], draws[t], n_steps)
            assert rpos == epos and np.array_equal(rs, es)
        assert int(cnt[t, 0]) == n_steps and int(cnt[t, 6] + cnt[t, 7]) <= n_steps


def test_script_wraps_like_scripted_rng(pb, orc):
    text, _ = config_text("c1")
    plan = pb.prepare(pb.parse_model(text), 1 << 25, 12, 8)
    rng = np.random.default_rng(9)
    script = rng.random(37)  # shorter than one step's draws: wraps inside steps
    eng = pb.GpuEnsemble(plan)
    st, _, used = eng.simulate_scripted(script, 25)
    s, pos = np.zeros(plan.n_kept // 64 + 1, np.uint64), 0
    per_step = 200
    for _ in range(25):
        window = [script[(pos + i) % len(script)] for i in range(per_step)]
        s, u = orc.step_scripted(plan.view, s, window)
        pos += u
    assert int(used[0]) == pos and np.array_equal(st[0], s)


def test_draws_off_the_2_pow_minus_53_grid(pb, orc):
    """A draw that is not a multiple of 2^-53 is replayed only when rounding it
    down to the grid provably keeps the decision; otherwise the call names it."""
    plan = pb.prepare(pb.parse_model(IDENTITY4), 1 << 20, 2, 18)
    eng = pb.GpuEnsemble(plan)
    st, _, used = eng.simulate_scripted([0.9, 0.9, 0.1], 2)  # 0.1 = off-grid leaf draw, t = 1
    es, epos = _replay_cpu(lambda s, u: orc.step_scripted(plan.view, s, u), np.zeros(1, np.uint64),
                           [0.9, 0.9, 0.1], 2)
    assert int(used[0]) == epos and np.array_equal(st[0], es)
    # a leaf threshold t in [0.25, 0.5): doubles there sit on the 2^-54 grid
    chain = ("pbn 3\nperturbation {p}\nnode x0\n  f 1 1\nnode x1\n  f 1 10 x0\n"
             "node x2\n  f 1 10 x1\ninterest x0\n")
    seen_reject = seen_accept = False
    for p in (0.3, 0.31, 0.32, 0.33, 0.34, 0.35, 0.36):
        plan = pb.prepare(pb.parse_model(chain.format(p=p)), 1 << 25, 16, 18)
        t = plan.t
        assert 0.25 <= t < 0.5
        eng = pb.GpuEnsemble(plan)
        quiet = _find_uniform(plan.flat().pert_cut, plan.flat().pert_alias, 0)
        for u in (math.nextafter(t, 1.0), math.nextafter(math.nextafter(t, 1.0), 1.0)):
            uq = math.floor(u * 2.0**53) / 2.0**53
            if (uq > t) != (u > t):
                with pytest.raises(pb.UsageError, match="not a multiple of 2\\^-53"):
                    eng.simulate_scripted([quiet, u], 1)
                seen_reject = True
            else:
                st, cnt, used = eng.simulate_scripted([quiet, u], 1)
                assert int(used[0]) == 2 and int(cnt[0, 6]) == 0 and int(cnt[0, 7]) == 0  # leaf fired
                seen_accept = True
    assert seen_reject and seen_accept
