#!/usr/bin/env python3
"""Small launches of each kernel family for compute-sanitizer (racecheck,
synccheck, memcheck): tools/sanitize.sh runs every case under every tool and
keeps the summaries in profiles/. Each case also checks the device result
against the oracle, so a sanitizer-clean run is also a correct one.

  python tools/sanitize_cases.py <case>     case in CASES
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# name: (generator args, plan (k, mgp), lanes per trajectory, trajectories, steps, flags)
CASES = {
    # c2-shaped: sub-warp kernel, register gathers + compact single-node records
    # (the headline instantiation pbn_ensemble_kernel<32, U53, tables, 2>)
    "c2_subwarp": ((1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606), (16, 8), 0, 40, 60, {}),
    # n' = 1500: two state words per lane (RG2)
    "rg2": ((1500, (1, 3), (1, 5), 0.001, 0.0, 2, False, 12), (12, 8), 0, 40, 60, {}),
    # c1-shaped: lane-per-trajectory kernel (scan-ahead), node counts on
    "c1_lane": ((100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605), (16, 8), 1, 64, 200,
                {"node_counts": True}),
    # n' > 2047: compact shared-memory-gather records (GM 4) + the exact redo
    "scl": ((2600, (1, 4), (1, 5), 0.0002, 0.0, 2, False, 21), (16, 8), 0, 24, 30,
            {"exact_alias": True}),
    # small sub-warps (LPT 8): several trajectories per warp, shared atomics
    "lpt8": ((100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605), (12, 8), 8, 64, 200, {}),
}


def main(case):
    import oracle
    import paper_1605_00854_b200 as pb

    gen, (k, mgp), lpt, n_traj, n_steps, kw = CASES[case]
    model, terms = pb.generate_model(*gen)
    plan = pb.prepare(model, 1 << 25, k, mgp)
    pred = plan.compile_predicate(terms)
    eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
    out = eng.simulate(seed=5, n_traj=n_traj, n_steps=n_steps, pred=pred, **kw)
    ref = oracle.Oracle().simulate(plan.view, 5, 0, n_traj, n_steps, pred=pred,
                                   node_counts=kw.get("node_counts", False))
    for a, b in zip(out, ref):
        assert np.array_equal(a, b), case
    print(case, "ok", eng.last_kernel())


if __name__ == "__main__":
    main(sys.argv[1])
