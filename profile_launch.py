#!/usr/bin/env python3
"""One ensemble launch of a config (for ncu):
python profile_launch.py [c2] [steps] [u53|u32] [lpt] [p] [n_traj]"""
import sys

import paper_1605_00854_b200 as pb
from paper_1605_00854_b200.configs import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
stream = pb.STREAM_U32 if (len(sys.argv) > 3 and sys.argv[3] == "u32") else pb.STREAM_U53
lpt = int(sys.argv[4]) if len(sys.argv) > 4 else 0
p = float(sys.argv[5]) if len(sys.argv) > 5 and sys.argv[5] != '-' else None
n_traj = int(sys.argv[6]) if len(sys.argv) > 6 else min(CONFIGS[cfg].n_traj, 16384)
w = CONFIGS[cfg]
model, terms = w.model(p)
plan = pb.prepare(pb.parse_model(model.serialize()), w.theta, w.k_max, w.mgp)
eng = pb.GpuEnsemble(plan, lanes_per_traj=lpt)
pred = plan.compile_predicate(terms)
eng.simulate(seed=42, n_traj=n_traj, n_steps=steps, pred=pred,
             stream=stream)
print("ok", eng.info())
