"""Host preprocessing parity: the product's prepare() (reduction, grouped
perturbation plan, node grouping, flattening) is byte-identical to the
unmodified reference pbn::prepare (engine.hpp:85-164) built in oracle/_ref,
on the same model text and (theta, k_max, max_group_parents)."""
import numpy as np
import pytest

from helpers import config_text, flat_of, plan_diff


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
@pytest.mark.parametrize("k,mgp", [(16, 8), (16, 18), (12, 8), (16, 12), (8, 6)])
def test_baseline_configs_identical(pb, ref, name, k, mgp):
    """(16, 8) is every bench plan but c4's; (16, 18) the reference default."""
    text, terms = config_text(name)
    mine = pb.prepare(pb.parse_model(text), 1 << 25, k, mgp)
    theirs = ref.parse(text).prepare(1 << 25, k, mgp)
    assert plan_diff(mine.flat(), flat_of(theirs.view)) == []
    # reduction bookkeeping and group membership
    n = pb.parse_model(text).n
    a, b = mine.reduced(), theirs.reduced(n)
    assert np.array_equal(a["index_map"], b["index_map"])
    assert np.array_equal(a["engine_pos"], b["engine_pos"])
    assert np.array_equal(a["removed"], b["removed"])
    ma, ca = mine.groups()
    mb, cb = theirs.groups()
    assert np.array_equal(ma, mb) and np.array_equal(ca, cb)
    # predicate compilation (engine.hpp:357-362)
    pa, pb_ = mine.compile_predicate(terms), theirs.compile_predicate(terms)
    assert np.array_equal(pa[0], pb_[0])


@pytest.mark.parametrize("seed", range(40))
def test_random_small_models_identical(pb, ref, seed):
    # the reference's own library-independent generator (oracles.hpp:175-208)
    n = 2 + seed % 7
    rm = ref.random_small_model(1000 + seed, n, 0.05 + 0.01 * (seed % 5), 3, 3)
    text = rm.serialize()
    for theta, k, mgp in [(1 << 20, 3, 18), (1 << 25, 16, 18), (64, 2, 4), (1 << 10, 1, 6)]:
        try:
            theirs = ref.parse(text).prepare(theta, k, mgp)
        except Exception as e:  # same error class on both sides
            with pytest.raises((pb.ModelError, pb.ResourceError)) as ei:
                pb.prepare(pb.parse_model(text), theta, k, mgp)
            assert ei.value.code == e.code
            continue
        mine = pb.prepare(pb.parse_model(text), theta, k, mgp)
        assert plan_diff(mine.flat(), flat_of(theirs.view)) == []


@pytest.mark.parametrize("seed", range(12))
def test_random_generated_networks_with_leaves(pb, ref, seed):
    model, _ = pb.generate_model(30 + 7 * seed, (1, 3), (1, 4), 0.02, leaf_frac=0.1 * (seed % 6),
                                 n_targets=2, seed=seed)
    text = model.serialize()
    mine = pb.prepare(pb.parse_model(text), 1 << 25, 10, 10)
    theirs = ref.parse(text).prepare(1 << 25, 10, 10)
    assert plan_diff(mine.flat(), flat_of(theirs.view)) == []


def test_unplannable_network_fails_like_the_reference(pb, ref):
    # a 5-function node with 20 distinct parents needs 5 * 2^20 > 2^22 entries
    # (grouping.hpp:42, 222-224): both sides raise resource_error
    model, _ = pb.generate_model(1000, (1, 5), (1, 4), 0.001, n_targets=3, seed=1607)
    text = model.serialize()
    with pytest.raises(Exception) as e_ref:
        ref.parse(text).prepare(1 << 25, 12, 8)
    assert e_ref.value.code == 3
    with pytest.raises(pb.ResourceError):
        pb.prepare(pb.parse_model(text), 1 << 25, 12, 8)


def test_theta_too_small_for_single_function_groups(pb, ref):
    model, _ = pb.generate_model(40, (1, 1), (3, 3), 0.01, seed=2)
    text = model.serialize()
    with pytest.raises(Exception) as e_ref:
        ref.parse(text).prepare(16, 8, 8)
    with pytest.raises(pb.ResourceError):
        pb.prepare(pb.parse_model(text), 16, 8, 8)
    assert e_ref.value.code == 3


def test_serialization_identical(pb, ref):
    for name in ["c1", "c3"]:
        text, _ = config_text(name)
        assert pb.parse_model(text).serialize() == ref.parse(text).serialize()


@pytest.mark.slow
def test_c4_bench_plan_identical(pb, ref):
    """c4's bench plan (k 16, mgp 12): the spill workload."""
    text, _ = config_text("c4")
    mine = pb.prepare(pb.parse_model(text), 1 << 25, 16, 12)
    theirs = ref.parse(text).prepare(1 << 25, 16, 12)
    assert plan_diff(mine.flat(), flat_of(theirs.view)) == []
