"""BASELINE.json workloads as synthetic-network + plan + ensemble parameters.

The paper's corpus and the apoptosis network are not available,
so seeded BASELINE-shaped networks stand in: model seed
1605 + 0-based config index, simulation seed 42, all-zero initial states.

Plan parameters (theta, k_max, max_group_parents) are part of the workload and
are passed identically to the oracle / reference: bit-exactness needs the same
plan. The large networks (c2, c4, c5) use the reference's default perturbation
width k_max=16 (engine.hpp:82; the paper's choice): for n' = 1000
its 64 phase-A draws are exactly one 32-lane round of 53-bit Philox draws; the
65536-cell table stays in L1/L2. The small networks (c1, c3) use k_max=16 as
well: with 53-bit draws a Philox block then covers exactly one 32-bit state
word of patterns (word-per-block phase A), and fewer, wider groups beat the
shared-memory residency of a 4096-cell k=12 table (c1 +15 %, c3 +2 %).
max_group_parents=8 keeps merged truth tables in shared memory (c4
deliberately uses 12 — "tables up to 2^12 entries per group ... spilling").
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    f_range: tuple
    p_range: tuple
    p: float
    leaf_frac: float
    n_targets: int
    targets_fixed: bool
    seed: int
    n_traj: int
    n_steps: int
    theta: int = 1 << 25
    k_max: int = 12
    mgp: int = 8
    sweep: tuple = field(default_factory=tuple)
    note: str = ""

    def model(self, p=None):
        from . import generate_model

        return generate_model(self.n, self.f_range, self.p_range, self.p if p is None else p,
                              self.leaf_frac, self.n_targets, self.targets_fixed, self.seed)


CONFIGS = {
    "c1": Workload("c1", 100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605, 131072, 100_000,
                   k_max=16,
                   note="n=100, target node0=1 AND node1=1; CPU ref 1 traj x 1e6 steps; "
                        "GPU: 131072 trajectories x 1e5 steps per bench step"),
    "c2": Workload("c2", 1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606, 4096, 100_000,
                   k_max=16, note="n=1000, 4096 trajectories x 1e5 steps, single B200 (headline)"),
    "c3": Workload("c3", 96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607, 65536, 0,
                   k_max=16,
                   note="n=96 dense, ~30% leaves; two-state MC estimate r=1e-3, conf 0.95"),
    "c4": Workload("c4", 5000, (1, 4), (1, 5), 0.0001, 0.0, 2, False, 1608, 16384, 100_000,
                   k_max=16, mgp=12,
                   note="n=5000, merged tables up to 2^12 entries (spill), 8 GPUs"),
    "c5": Workload("c5", 2000, (1, 3), (1, 4), 0.01, 0.0, 2, False, 1609, 32768, 1_000_000,
                   k_max=16, sweep=(0.1, 0.01, 0.001, 0.0001),
                   note="n=2000 perturbation sweep, 32768 traj x 1e6 steps per GPU"),
}
