"""Device estimator: the pooled estimate computed on the B200 (pbn_estimate)
equals the same C++ estimator driven by the oracle restatement (bit-exact, the
device trajectories being bit-exact), and on the BASELINE c3 workload (65536
trajectories, r = 1e-3, conf 0.95) it agrees with the reference's own
high-precision estimate within |delta| <= 1e-3."""
import json
import os

import pytest

from estimator_support import OracleEnsemble
from helpers import config_text

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("stream", [0, 1])
def test_device_estimate_equals_oracle_driven_estimate(pb, orc, stream):
    text, terms = config_text("c3")
    plan = pb.prepare(pb.parse_model(text), 1 << 25, 12, 8)
    pred = plan.compile_predicate(terms)
    req = pb.make_request(precision=0.01, pilot=300, seed=11, traj_begin=7, n_traj=96,
                          stream=stream)
    dev, _ = pb.estimate(pb.GpuEnsemble(plan), pred, req)
    cpu = OracleEnsemble(orc, plan.view, pred, 11, 96, stream, traj_begin=7).estimate(req)
    for k in ("estimate", "sample_size_used", "burn_in_used", "steps_per_traj", "kappa",
              "degenerate"):
        assert dev[k] == cpu[k], k


def test_c3_pooled_estimate_matches_reference_within_1e_3(pb):
    want = json.load(open(os.path.join(HERE, "c3_steady_state.json")))
    text, terms = config_text("c3")
    plan = pb.prepare(pb.parse_model(text), 1 << 25, 12, 8)
    pred = plan.compile_predicate(terms)
    req = pb.make_request(precision=1e-3, confidence=0.95, pilot=1000, seed=42, n_traj=65536)
    got, _ = pb.estimate(pb.GpuEnsemble(plan), pred, req)
    assert not got["degenerate"]
    assert got["sample_size_used"] >= 1_000_000
    assert abs(got["estimate"] - want["estimate"]) <= 1e-3, (got, want["estimate"])


def test_c3_pooled_estimates_cover_the_reference_value_over_20_seeds(pb):
    """north star: |delta| <= 1e-3 at equal precision, as a coverage over seeds
    (cf. acceptance.cpp:171-196): 20 device estimates on the bench's c3 plan
    (k = 16, mgp = 8; 65536 trajectories, r = 1e-3, conf 0.95) against the
    reference's r = 2.5e-4 value. With nominal 95 % intervals and the
    yardstick's own error, >= 15 of 20 is expected except with probability
    < 0.5 %; tools/steady_state_coverage.py reports the distribution beside
    20 reference estimates (profiles/r02_steady_state.json)."""
    want = json.load(open(os.path.join(HERE, "c3_steady_state.json")))
    text, terms = config_text("c3")
    plan = pb.prepare(pb.parse_model(text), 1 << 25, 16, 8)
    pred = plan.compile_predicate(terms)
    eng = pb.GpuEnsemble(plan)
    deltas = []
    for s in range(20):
        req = pb.make_request(precision=1e-3, confidence=0.95, pilot=1000, seed=1000 + s,
                              n_traj=65536)
        got, _ = pb.estimate(eng, pred, req)
        assert not got["degenerate"]
        deltas.append(abs(got["estimate"] - want["estimate"]))
    assert sum(d <= 1e-3 for d in deltas) >= 15, deltas
    assert max(deltas) <= 3e-3, deltas
