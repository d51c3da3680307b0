"""Shared test helpers (test infrastructure)."""
import hashlib

import numpy as np

import paper_1605_00854_b200 as pb

PLAN_FIELDS = ["n_kept", "t", "pert_groups", "pert_k", "pert_k_prime", "pert_mask", "pert_cut",
               "pert_alias", "grp_offset", "grp_fn_begin", "grp_alias_begin", "grp_alias_size",
               "alias_cut", "alias_idx", "fn_gather_begin", "fn_table_begin", "fn_gather_count",
               "fn_gather", "fn_tables"]


def flat_of(view):
    return pb.FlatPlan.from_view(view)


def plan_diff(a, b):
    """Fields whose bytes differ (doubles compared bitwise)."""
    bad = []
    for f in PLAN_FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        if isinstance(x, np.ndarray):
            if x.dtype != y.dtype or x.shape != y.shape or x.tobytes() != y.tobytes():
                bad.append(f)
        elif np.float64(x).tobytes() != np.float64(y).tobytes():
            bad.append(f)
    return bad


def plan_digest(flat):
    h = hashlib.sha256()
    for f in PLAN_FIELDS:
        x = getattr(flat, f)
        h.update(f.encode())
        h.update(x.tobytes() if isinstance(x, np.ndarray) else np.float64(x).tobytes())
    return h.hexdigest()


def config_text(name, p=None):
    from paper_1605_00854_b200.configs import CONFIGS

    model, terms = CONFIGS[name].model(p)
    return model.serialize(), terms
