"""Pooled two-state MC steady-state estimator (estimator.hpp:137-244).

The estimator is host C++ over a stepping backend. On CPU the oracle
restatement is the backend: a one-trajectory ensemble must reproduce the
unmodified reference estimator (oracle/_ref, pbn::estimate_steady_state on the
same Philox stream) bit-for-bit; pooled ensembles must land on the exact
stationary value (exact.hpp) at the requested precision."""
import numpy as np
import pytest

from estimator_support import OracleEnsemble
from helpers import config_text


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("stream", [0, 1])
def test_one_trajectory_reproduces_reference_estimator(pb, orc, ref, seed, stream):
    rm = ref.random_small_model(90 + seed, 5, 0.25, 2, 2)
    text = rm.serialize()
    rplan = ref.parse(text).prepare()
    plan = pb.prepare(pb.parse_model(text))
    terms = [(0, 1)]
    want = rplan.estimate(terms, 0.01, 0.95, 1000, seed, stream, 3)
    req = pb.make_request(precision=0.01, pilot=1000, seed=seed, traj_begin=3, n_traj=1,
                          stream=stream)
    got = OracleEnsemble(orc, plan.view, plan.compile_predicate(terms), seed, 1, stream,
                         traj_begin=3).estimate(req)
    assert got["estimate"] == want["estimate"]
    assert got["sample_size_used"] == want["sample_size"]
    assert got["burn_in_used"] == want["burn_in"]
    assert bool(got["degenerate"]) == want["degenerate"]


def test_one_trajectory_reproduces_reference_on_c3(pb, orc, ref):
    text, terms = config_text("c3")
    rplan = ref.parse(text).prepare(1 << 25, 12, 8)
    plan = pb.prepare(pb.parse_model(text), 1 << 25, 12, 8)
    want = rplan.estimate(terms, 0.01, 0.95, 2000, 42, 0, 0)
    req = pb.make_request(precision=0.01, pilot=2000, seed=42, n_traj=1)
    got = OracleEnsemble(orc, plan.view, plan.compile_predicate(terms), 42, 1).estimate(req)
    assert (got["estimate"], got["sample_size_used"], got["burn_in_used"]) == \
        (want["estimate"], want["sample_size"], want["burn_in"])


def test_pooled_ensembles_hit_the_exact_value(pb, orc, ref):
    # acceptance.cpp:171-196 style: exact stationary marginal vs estimate at r
    hits, total = 0, 0
    for mi in range(6):
        rm = ref.random_small_model(5001 + mi, 3 + mi % 3, 0.25, 2, 2)
        text = rm.serialize()
        truth = rm.marginal_exact([(0, 1)])
        plan = pb.prepare(pb.parse_model(text))
        pred = plan.compile_predicate([(0, 1)])
        for rep in range(4):
            req = pb.make_request(precision=0.01, pilot=500, seed=100 * mi + rep, n_traj=24)
            got = OracleEnsemble(orc, plan.view, pred, 100 * mi + rep, 24).estimate(req)
            assert not got["degenerate"]
            hits += abs(got["estimate"] - truth) <= 0.01
            total += 1
    assert hits >= 0.85 * total, (hits, total)


def test_degenerate_predicate_is_flagged(pb, orc):
    # test_estimator.cpp:112-133: a constant-1 node at tiny p never moves
    m = pb.parse_model("pbn 2\nperturbation 0.000000001\nnode a\n  f 1 1\nnode b\n  f 1 10 b\n")
    plan = pb.prepare(m)
    pred = plan.compile_predicate([(0, 1)])
    ens = OracleEnsemble(orc, plan.view, pred, 5, 2)
    ens.states[:, 0] = np.uint64(1 << int(plan.reduced()["engine_pos"][0]))
    got = ens.estimate(pb.make_request(precision=0.01, pilot=100, seed=5, n_traj=2))
    assert got["degenerate"] == 1 and got["estimate"] == 1.0


def test_request_validation(pb, orc):
    m = pb.parse_model("pbn 1\nperturbation 0.5\nnode a\n  f 1 10 a\n")
    plan = pb.prepare(m)
    ens = OracleEnsemble(orc, plan.view, plan.compile_predicate([(0, 1)]), 1, 1)
    with pytest.raises(pb.ModelError):
        ens.estimate(pb.make_request(precision=0.0, n_traj=1))
    with pytest.raises(pb.ModelError):
        ens.estimate(pb.make_request(precision=0.01, confidence=1.0, n_traj=1))


def test_inverse_normal_cdf(pb, ref):
    # test_estimator.cpp:25-40, and bitwise equal to the reference
    f = pb.lib.pbn_inverse_normal_cdf
    assert abs(f(0.5)) <= 1e-12
    assert abs(f(0.975) - 1.959963984540054) <= 1e-9
    assert abs(f(0.995) - 2.5758293035489004) <= 1e-9
    for p in np.linspace(0.001, 0.999, 97):
        assert f(float(p)) == ref.lib.ref_inverse_normal_cdf(float(p))


def test_series_stats_host_matches_numpy(pb):
    rng = np.random.default_rng(3)
    ser = rng.integers(0, 2**32, size=(5, 8), dtype=np.uint64).astype(np.uint32)
    length = 200
    bits = np.unpackbits(ser.view(np.uint8), bitorder="little").reshape(5, -1)[:, :length]
    for kappa in (1, 2, 5):
        got = pb.series_stats_host(ser, length, kappa)
        want = np.zeros(13, np.int64)
        for z in bits:
            for t in range(2 * kappa, length, kappa):
                want[(z[t - 2 * kappa] << 2) | (z[t - kappa] << 1) | z[t]] += 1
            for t in range(kappa, length, kappa):
                want[8 + ((z[t - kappa] << 1) | z[t])] += 1
            want[12] += z[1:].sum()
        assert np.array_equal(got.astype(np.int64), want)
