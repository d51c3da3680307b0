"""Integer form of the U53 combined-function choice (dev_plan.h a53) against
the reference's FP64 rule (engine.hpp:285-290), on the host, no GPU: random
draws, draws on and next to every cell boundary and cut point, the clamp
region at the top of the range, and degenerate cut-offs."""
import numpy as np
import pytest


def fp64_rule(cut, alias, r53):
    """engine.hpp:285-290 restated in numpy float64 (IEEE, one rounding per op)."""
    n = len(cut)
    x = (r53.astype(np.float64) * 2.0**-53) * np.float64(n)
    c = np.minimum(x.astype(np.uint64), n - 1)
    fr = x - c.astype(np.float64)
    return np.where(fr < cut[c], c, alias[c]).astype(np.uint32)


def edge_draws(cut, rng):
    """r53 values around each cell start and each cut point, plus the ends."""
    n = len(cut)
    pts = []
    width = 4096 if n <= 8 else 128
    for c in range(n):
        for base in (c / n, (c + cut[c]) / n):
            r = int(base * 2.0**53)
            pts.extend(range(max(r - width, 0), min(r + width, 2**53)))
            # the same point found at hi32 granularity
            h = int(base * 2.0**32)
            pts.extend(((h + d) << 21) + o for d in (-1, 0, 1) for o in (0, 1, 2**20, 2**21 - 1)
                       if 0 <= h + d < 2**32)
    pts.extend(range(2**53 - 5000, 2**53))
    pts.extend(range(0, 5000))
    r53 = np.array(sorted(set(pts)), np.uint64)
    low = rng.integers(0, 2**11, len(r53), dtype=np.uint64)
    return r53, (r53 << np.uint64(11)) | low


@pytest.mark.parametrize("n", [2, 3, 4, 5, 7, 8, 31, 100, 1000, 2048])
def test_integer_form_matches_fp64_rule(pb, n):
    rng = np.random.default_rng(1605 + n)
    w = rng.random(n) + 0.05
    cut, alias = pb.alias_build(w / w.sum())
    raw = rng.integers(0, 2**63, 200_000, dtype=np.uint64) * np.uint64(2) + \
        rng.integers(0, 2, 200_000, dtype=np.uint64)
    pick, fast = pb.alias53_pick(cut, alias, raw)
    assert np.array_equal(pick, fp64_rule(cut, alias, raw >> np.uint64(11)))
    assert fast.mean() > 0.999
    r53, raw = edge_draws(cut, rng)
    pick, fast = pb.alias53_pick(cut, alias, raw)
    assert np.array_equal(pick, fp64_rule(cut, alias, r53))
    assert fast.any() and not fast.all()


def test_degenerate_cutoffs(pb):
    rng = np.random.default_rng(7)
    for cut in ([1.0, 1.0, 1.0], [0.0, 1.0, 0.5], [1e-300, 1 - 2**-53, 2**-53],
                [0.5, 0.0, 1.0, 1.0, 2**-40]):
        cut = np.array(cut, np.float64)
        alias = np.array([(i + 1) % len(cut) for i in range(len(cut))], np.uint32)
        r53, raw = edge_draws(cut, rng)
        pick, _ = pb.alias53_pick(cut, alias, raw)
        assert np.array_equal(pick, fp64_rule(cut, alias, r53))


def test_rejects_out_of_range_sizes(pb):
    with pytest.raises(pb.UsageError):
        pb.alias53_pick(np.ones(1), np.zeros(1, np.uint32), np.zeros(1, np.uint64))
    with pytest.raises(pb.UsageError):
        pb.alias53_pick(np.ones(2049), np.zeros(2049, np.uint32), np.zeros(1, np.uint64))
