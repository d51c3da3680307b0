#!/usr/bin/env python3
"""Steady-state agreement at equal precision (north star: |delta| <= 1e-3),
over many seeds, on the bench's c3 workload and plan (BASELINE config 3:
n = 96, 2-node target, r = 1e-3, confidence 0.95; plan theta 2^25, k 16,
mgp 8):

  * device: the pooled two-state Markov-chain estimate over 65536 trajectories
    (pbn_estimate, Philox stream), one per seed;
  * reference: the unmodified reference's own single-chain
    estimate_steady_state (estimator.hpp:137-244, xoshiro256, oracle/_ref), one
    per seed, at the same precision r and confidence (so both sample sizes are
    the ones the estimator itself requires for r = 1e-3);
  * truth: the reference's high-precision estimate (r = 2.5e-4, 20.2M samples,
    tests/golden/c3_steady_state.json).

Reports |estimate - truth| for both, the coverage (fraction within r) and the
sample sizes. The reference criterion is acceptance.cpp:171-196 (>= 90 of 100
estimates within r of the exact value).

  python tools/steady_state_coverage.py [--seeds 20] [--out profiles/r02_steady_state.json]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=20)
    ap.add_argument("--precision", type=float, default=1e-3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_steady_state.json"))
    ap.add_argument("--no-reference", action="store_true")
    a = ap.parse_args()

    import bench
    import paper_1605_00854_b200 as pb

    truth = json.load(open(os.path.join(ROOT, "tests", "golden", "c3_steady_state.json")))
    w, text, model, plan, terms = bench.build_workload("c3", None)
    pred = plan.compile_predicate(terms)
    eng = pb.GpuEnsemble(plan)
    dev = []
    t0 = time.perf_counter()
    for s in range(a.seeds):
        req = pb.make_request(precision=a.precision, confidence=0.95, pilot=1000, seed=1000 + s,
                              n_traj=w.n_traj)
        r, _ = pb.estimate(eng, pred, req)
        dev.append(r)
    dev_s = time.perf_counter() - t0
    out = {"workload": "c3", "plan": {"theta": w.theta, "k_max": w.k_max, "mgp": w.mgp},
           "precision": a.precision, "confidence": 0.95, "truth": truth["estimate"],
           "truth_precision": truth["precision"], "truth_sample_size": truth["sample_size"],
           "device": summarize([r["estimate"] for r in dev], truth["estimate"], a.precision)}
    out["device"].update({"trajectories": w.n_traj, "seconds_total": dev_s,
                          "sample_size": [int(r["sample_size_used"]) for r in dev],
                          "kernel": eng.last_kernel()})
    if not a.no_reference:
        import oracle

        rplan = oracle.Reference().parse(text).prepare(w.theta, w.k_max, w.mgp)

        def one(seed):
            return rplan.estimate(terms, a.precision, 0.95, 10000, seed, -1, 0)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
            ref = list(ex.map(one, range(2000, 2000 + a.seeds)))
        out["reference"] = summarize([r["estimate"] for r in ref], truth["estimate"], a.precision)
        out["reference"].update({"seconds_total": time.perf_counter() - t0,
                                 "sample_size": [int(r["sample_size"]) for r in ref],
                                 "impl": "oracle/_ref estimate_steady_state, xoshiro256"})
        out["device_minus_reference_mean"] = (out["device"]["mean"] - out["reference"]["mean"])
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k in ("truth", "device_minus_reference_mean")}
                     | {"device": {k: out["device"][k] for k in ("coverage", "abs_delta_max", "mean")},
                        "reference": {k: out.get("reference", {}).get(k) for k in ("coverage", "abs_delta_max", "mean")}}))


def summarize(est, truth, r):
    e = np.asarray(est, float)
    d = np.abs(e - truth)
    return {"estimates": e.tolist(), "mean": float(e.mean()), "std": float(e.std(ddof=1)) if len(e) > 1 else 0.0,
            "abs_delta": d.tolist(), "abs_delta_median": float(np.median(d)),
            "abs_delta_p90": float(np.quantile(d, 0.9)), "abs_delta_max": float(d.max()),
            "coverage": float((d <= r).mean()), "within_r": int((d <= r).sum()), "n": len(e)}


if __name__ == "__main__":
    main()
