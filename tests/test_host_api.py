"""Host API semantics mirrored from the reference's unit tests
(test_model.cpp, test_grouping.cpp, test_core.cpp, test_engine.cpp)."""
import numpy as np
import pytest

TWO = "pbn 2\nperturbation 0.01\nnode a\n  f 1 10 b\nnode b\n  f 1 10 a\n"


def test_parse_minimal_network(pb):
    m = pb.parse_model(TWO)
    info = m.info()
    assert info["n"] == 2 and abs(info["p"] - 0.01) < 1e-15 and info["n_interest"] == 2
    assert m.serialize() == TWO


@pytest.mark.parametrize("text,line", [
    ("perturbation 0.1\n", 1),
    ("pbn 2\nperturbation 0.1\nnode a\n  f 1 1\n", 4),
    ("pbn 1\nperturbation 0.1\nnode a\n  f 1 10 nosuch\n", 4),
    ("pbn 1\nperturbation 0.1\nnode a\n  f 1 100 a\n", 4),
    ("pbn 1\nperturbation 0.1\nnode a\n  f 1 1x a\n", 4),
    ("pbn 2\nperturbation 0.1\nnode a\n  f 1 1\nnode a\n  f 1 1\n", 5),
    ("pbn 1\nperturbation 0.1\nbogus\n", 3),
])
def test_parse_errors_carry_line_numbers(pb, text, line):
    # test_model.cpp:73-94
    with pytest.raises(pb.ModelError) as e:
        pb.parse_model(text)
    assert str(e.value).startswith(f"line {line}:")


def test_probabilities_must_sum_to_one(pb):
    with pytest.raises(pb.ModelError) as e:
        pb.parse_model("pbn 1\nperturbation 0.01\nnode a\n  f 0.5 10 a\n  f 0.4 01 a\n")
    assert "sum to 0.9" in str(e.value)


def test_comments_and_table_orientation(pb, orc):
    m = pb.parse_model("# c\npbn 3   # n\n\nperturbation 0.1\nnode a\n  f 1 1000 b c\n"
                       "node b\n  f 1 10 b\nnode c\n  f 1 10 c\n")
    plan = pb.prepare(m)
    f = plan.flat()
    # AND(b, c): the only 1 sits at the highest valuation
    a_group = [i for i in range(len(f.grp_offset))]
    assert plan.n_kept == 3 and len(a_group) >= 1
    assert m.serialize().splitlines()[3] == "  f 1 1000 b c"


def test_lower_bound_and_greedy_hand_traces(pb):
    # test_grouping.cpp:19-81
    assert pb.lower_bound([2, 2, 2, 2], 16) == 1
    assert pb.lower_bound([4, 4, 4, 4], 30) == 3
    assert pb.lower_bound([5], 5) == 1
    parts = pb.greedy_partition([8, 7, 6, 5, 4], 2)
    w = [8, 7, 6, 5, 4]
    prods = sorted(int(np.prod([w[i] for i in p])) for p in parts)
    assert prods == [42, 160]
    parts = pb.greedy_partition([3, 2], 4)
    assert sum(1 for p in parts if p) == 2


def test_greedy_matches_reference_order_on_random_instances(pb):
    # the heap-based partition keeps the reference's lowest-index tie-break
    rng = np.random.default_rng(31)
    for _ in range(200):
        w = rng.integers(2, 7, size=int(rng.integers(1, 40)))
        m = int(rng.integers(1, len(w) + 3))
        order = sorted(range(len(w)), key=lambda i: (-int(w[i]), i))
        prod = [1.0] * m
        want = [[] for _ in range(m)]
        for i in order:
            j = min(range(m), key=lambda j: (prod[j], j))
            want[j].append(i)
            prod[j] *= float(w[i])
        assert pb.greedy_partition(w, m) == want


def test_alias_build_bitwise_vs_reference(pb, ref):
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(1, 40))
        p = rng.random(n) + 1e-3
        p /= p.sum()
        a = pb.alias_build(p)
        b = ref.alias_build(p)
        assert a[0].tobytes() == b[0].tobytes() and np.array_equal(a[1], b[1])
        implied = np.zeros(n)
        for i in range(n):
            implied[i] += a[0][i] / n
            implied[a[1][i]] += (1 - a[0][i]) / n
        assert np.abs(implied - p).max() <= 1e-12


def test_alias_rejects_bad_distributions(pb):
    with pytest.raises(pb.ModelError):
        pb.alias_build([])
    with pytest.raises(pb.ModelError):
        pb.alias_build([0.5, 0.4])
    with pytest.raises(pb.ModelError):
        pb.alias_build([1.5, -0.5])


def test_predicate_compilation(pb):
    # test_engine.cpp:322-359
    m = pb.parse_model("pbn 3\nperturbation 0.01\nnode a\n  f 1 10 a\nnode b\n  f 1 10 a\n"
                       "node c\n  f 1 10 b\ninterest a b\n")
    plan = pb.prepare(m)
    assert list(plan.reduced()["removed"]) == [2]
    bits, _ = plan.compile_predicate([(1, True)])
    assert bits[0] == plan.reduced()["engine_pos"][plan.reduced()["index_map"][1]]
    with pytest.raises(pb.ModelError):
        plan.compile_predicate([(2, False)])  # removed leaf
    with pytest.raises(pb.ModelError):
        plan.compile_predicate([(7, True)])  # nonexistent


def test_generator_is_deterministic_and_shaped(pb):
    a, ta = pb.generate_model(300, (1, 3), (1, 4), 0.01, leaf_frac=0.2, n_targets=3, seed=11)
    b, tb = pb.generate_model(300, (1, 3), (1, 4), 0.01, leaf_frac=0.2, n_targets=3, seed=11)
    c, _ = pb.generate_model(300, (1, 3), (1, 4), 0.01, leaf_frac=0.2, n_targets=3, seed=12)
    assert a.serialize() == b.serialize() and ta == tb
    assert a.serialize() != c.serialize()
    plan = pb.prepare(a, 1 << 25, 12, 8)
    removed = len(plan.reduced()["removed"])
    assert removed >= 60  # 20% designated leaves (plus natural ones)
    assert a.info()["n_interest"] == 3


def test_generator_fixed_targets(pb):
    m, terms = pb.generate_model(100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605)
    assert terms == [(0, 1), (1, 1)]


def test_stats_csv_matches_reference_layout(pb, orc, ref):
    """pbn simulate's CSV (pbn_main.cpp:75-85, 226-235) from one-counts of the
    reference stepper and of the oracle: identical text."""
    m = pb.parse_model(CHAIN3_CSV)
    plan = pb.prepare(m)
    rplan = ref.parse(CHAIN3_CSV).prepare()
    _, _, a = rplan.simulate_philox(9, 0, 1, 5000, node_counts=True)
    _, _, b = orc.simulate(plan.view, 9, 0, 1, 5000, node_counts=True)
    assert np.array_equal(a, b)
    csv = pb.stats_csv(plan, b, 5000)
    lines = csv.splitlines()
    assert lines[0] == "node,name,one_count,steps,frequency"
    assert [ln.split(",")[1] for ln in lines[1:]] == ["x0", "x1"]  # x2 is a removed leaf
    for ln in lines[1:]:
        v, name, ones, steps, freq = ln.split(",")
        assert int(steps) == 5000 and freq == "%.12g" % (int(ones) / 5000)


CHAIN3_CSV = ("pbn 3\nperturbation 0.05\nnode x0\n  f 1 01 x1\nnode x1\n  f 1 10 x0\n"
              "node x2\n  f 1 10 x1\ninterest x0 x1\n")
