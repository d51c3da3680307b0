#!/usr/bin/env python3
"""Randomised device-vs-oracle parity sweep over network shapes, plan
parameters, streams and kernel choices (run on a B200; not part of the
default test suite because of its length). Usage: parity_sweep.py [cases] [seed]"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402  (checker)
import paper_1605_00854_b200 as pb  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
orc = oracle.Oracle()
fails = 0
t0 = time.time()
for case in range(n_cases):
    n = int(rng.choice([6, 20, 64, 100, 127, 200, 255, 400, 1000, 1500, 2100]))
    fmax = int(rng.integers(1, 6))
    pmax = int(rng.integers(1, 6))
    p = float(rng.choice([0.2, 0.05, 0.01, 0.001, 0.0001]))
    leaf = float(rng.choice([0.0, 0.1, 0.3]))
    k = int(rng.choice([3, 8, 12, 16]))
    mgp = int(rng.choice([4, 8, 12]))
    seed = int(rng.integers(0, 1 << 30))
    try:
        model, terms = pb.generate_model(n, (1, fmax), (1, pmax), p, leaf, 2, False, seed)
        plan = pb.prepare(model, 1 << 25, k, mgp)
    except pb.PbnError as e:  # unplannable shapes are the reference's errors too
        print(f"case {case}: skip ({type(e).__name__})")
        continue
    pred = plan.compile_predicate(terms)
    lpt = int(rng.choice([0, 0, 1, 2, 4, 8, 16, 32]))
    if lpt == 1 and plan.n_kept > 255:
        lpt = 0
    stream = int(rng.integers(0, 2))
    n_traj, n_steps = (64, 300) if plan.n_kept > 500 else (150, 800)
    placement = str(rng.choice(["auto", "auto", "global", "core", "tables", "all", "core_pert"]))
    eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
    try:
        eng.set_placement(placement)
    except pb.PbnError:
        placement = "auto"
    words = pb.state_words(plan.n_kept)
    init = rng.integers(0, 2**63, size=(n_traj, words), dtype=np.uint64)
    nk = plan.n_kept
    init[:, nk // 64] &= np.uint64((1 << (nk % 64)) - 1)
    init[:, nk // 64 + 1:] = 0
    nc = bool(rng.integers(0, 4) == 0)
    exact = bool(stream == 0 and rng.integers(0, 4) == 0)
    out = eng.simulate(seed=seed & 0xFFFF, n_traj=n_traj, n_steps=n_steps, states=init,
                       pred=pred, stream=stream, node_counts=nc, exact_alias=exact)
    ref = orc.simulate(plan.view, seed & 0xFFFF, 0, n_traj, n_steps, states=init, pred=pred,
                       stream=stream, node_counts=nc)
    ok = all(np.array_equal(a, b) for a, b in zip(out, ref))
    fails += not ok
    print(f"case {case}: n={n} n'={plan.n_kept} F<={fmax} P<={pmax} p={p} k={k} mgp={mgp} "
          f"lpt={lpt} stream={stream} nc={int(nc)} exact={int(exact)} "
          f"{eng.info()['lanes_per_traj']}/{eng.info()['placement']} "
          f"{'OK' if ok else 'MISMATCH'}", flush=True)
print(f"{n_cases} cases, {fails} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
