#!/usr/bin/env python3
"""Regenerates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libpbnref.so, built from /root/reference/proj/include by
oracle/Makefile). Run in the development container (needs /root/reference to
build _ref); the fixtures are committed and travel to the GPU box.

Each fixture: the BASELINE-shaped model text (sha256), the reference plan's
digest, and pbn::simulate(grouped_simulator) results on the injected Philox
stream for a few trajectories (both stream kinds, predicate on, nonzero
traj_begin/step_begin)."""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from helpers import config_text, flat_of, plan_digest  # noqa: E402

FIXTURES = {
    # name: (config, k_max, mgp, n_traj, n_steps, p override)
    # the benchmarked plans (bench.py / workloads.json: theta 2^25, k 16,
    # mgp 8; c4 mgp 12) and the c5 sweep's perturbation rates
    "c1_bench": ("c1", 16, 8, 8, 600, None),
    "c2_bench": ("c2", 16, 8, 6, 300, None),
    "c3_bench": ("c3", 16, 8, 8, 600, None),
    "c4_bench": ("c4", 16, 12, 2, 60, None),
    "c5_bench": ("c5", 16, 8, 4, 200, None),
    "c5_p0.1": ("c5", 16, 8, 4, 200, 0.1),
    "c5_p0.001": ("c5", 16, 8, 4, 200, 0.001),
    "c5_p0.0001": ("c5", 16, 8, 4, 200, 0.0001),
    # the reference's default plan (engine.hpp:81-83) and a k = 12 plan
    "c2_ref_default": ("c2", 16, 18, 4, 200, None),
    "c1_k12": ("c1", 12, 8, 8, 600, None),
    "c2_k12": ("c2", 12, 8, 4, 200, None),
}
SEED, TRAJ_BEGIN, STEP_BEGIN = 42, 1000, 7


def main():
    ref = oracle.Reference()
    manifest = {}
    for name, (cfg, k, mgp, n_traj, n_steps, p) in FIXTURES.items():
        text, terms = config_text(cfg, p)
        rplan = ref.parse(text).prepare(1 << 25, k, mgp)
        pred = rplan.compile_predicate(terms)
        out = {}
        for stream in (0, 1):
            st, cnt = rplan.simulate_philox(SEED, TRAJ_BEGIN, n_traj, n_steps, pred=pred,
                                            stream=stream, step_begin=STEP_BEGIN)
            out[f"states_s{stream}"] = st
            out[f"counts_s{stream}"] = cnt
        out["pred_bits"], out["pred_vals"] = pred
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        manifest[name] = {
            "config": cfg, "p": p, "k_max": k, "mgp": mgp, "theta": 1 << 25, "n_traj": n_traj,
            "n_steps": n_steps, "seed": SEED, "traj_begin": TRAJ_BEGIN, "step_begin": STEP_BEGIN,
            "model_sha256": hashlib.sha256(text.encode()).hexdigest(),
            "plan_digest": plan_digest(flat_of(rplan.view)), "n_kept": rplan.n_kept,
            "terms": terms,
        }
        print(name, manifest[name]["n_kept"], manifest[name]["plan_digest"][:16], flush=True)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)




def steady_state_reference():
    """High-precision steady-state value of the c3 target under the reference's
    own single-chain estimator (xoshiro256, r = 2.5e-4): the yardstick the
    pooled device estimate at r = 1e-3 is compared against."""
    ref = oracle.Reference()
    text, terms = config_text("c3")
    rplan = ref.parse(text).prepare(1 << 25, 16, 8)
    est = rplan.estimate(terms, 2.5e-4, 0.95, 10000, 2024, -1, 0)
    out = {"config": "c3", "k_max": 16, "mgp": 8, "precision": 2.5e-4, "confidence": 0.95,
           "seed": 2024, "terms": terms, **est}
    with open(os.path.join(HERE, "c3_steady_state.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("c3 steady state", est, flush=True)


if __name__ == "__main__":
    main()
    steady_state_reference()
