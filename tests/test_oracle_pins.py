"""Pins the oracle before trusting it:
  * the stream's Philox4x32-10 against published known-answer vectors
    (Random123 kat_vectors) and cuRAND's host generator;
  * the oracle restatement (oracle/pbn_oracle.c) bit-for-bit against the
    UNMODIFIED reference stepper (pbn::grouped_simulator through pbn::simulate,
    oracle/_ref) on the same injected stream;
  * the reference tests' forced-draw trace (test_engine.cpp:115-153) and
    known answers (t = 0.998001, plan shapes, 96 nodes/37.5% -> 60 kept,
    pi(1) = 10/11)."""
import ctypes
import ctypes.util

import numpy as np
import pytest

from helpers import config_text, flat_of, plan_diff

KAT = [  # Random123 kat_vectors, philox4x32_10: (ctr, key) -> out
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(orc, ctr, key, want):
    assert tuple(int(x) for x in orc.philox(ctr, key)) == want


def test_philox_matches_curand_host_generator(orc):
    path = "/usr/local/cuda/lib64/libcurand.so"
    try:
        cur = ctypes.CDLL(path)
    except OSError:
        pytest.skip("libcurand not available")
    gen = ctypes.c_void_p()
    assert cur.curandCreateGeneratorHost(ctypes.byref(gen), 161) == 0  # PHILOX4_32_10
    seed = 0x0123456789ABCDEF
    assert cur.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_ulonglong(seed)) == 0
    out = (ctypes.c_uint * 4)()
    assert cur.curandGenerate(gen, out, 4) == 0
    cur.curandDestroyGenerator(gen)
    mine = orc.philox([0, 0, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
    assert [int(x) for x in out] == [int(x) for x in mine]


def test_stream_layout(orc):
    """draw d: phase A (d <= g) at block position d/4, word d%4; phase B starts
    on block position ceil((g+1)/4). U53 takes its high word from block b and
    its low word from block b | 2^31."""
    seed, traj, step = 77, 5, 123
    key = [seed, 0]
    dpb = 4
    for g in (1, 4, 7, 12, 63):
        for kind in (0, 1):
            nb0 = (g + 1 + dpb - 1) // dpb
            for d in range(g + 1 + 3 * dpb):
                if d <= g:
                    b, e = d // dpb, d % dpb
                else:
                    b, e = nb0 + (d - g - 1) // dpb, (d - g - 1) % dpb
                x = orc.philox([traj, b, step, 0], key)
                if kind == 0:
                    y = orc.philox([traj, b | 0x80000000, step, 0], key)
                    want = ((int(x[e]) << 32 | int(y[e])) >> 11) * 2.0**-53
                else:
                    want = int(x[e]) * 2.0**-32
                assert orc.draw(seed, traj, step, d, kind, g) == want


CASES = [("c1", 12, 8), ("c3", 12, 8), ("c2", 12, 8), ("c5", 12, 8), ("c1", 16, 12), ("c3", 4, 6)]


@pytest.mark.parametrize("name,k,mgp", CASES)
@pytest.mark.parametrize("stream", [0, 1])
def test_oracle_bit_exact_vs_reference_stepper(pb, orc, ref, name, k, mgp, stream):
    text, terms = config_text(name)
    rplan = ref.parse(text).prepare(1 << 25, k, mgp)
    pred = rplan.compile_predicate(terms)
    n_traj, n_steps = (6, 400) if rplan.n_kept > 500 else (16, 1500)
    a = rplan.simulate_philox(42, 3, n_traj, n_steps, pred=pred, stream=stream, node_counts=True,
                              step_begin=11)
    b = orc.simulate(rplan.view, 42, 3, n_traj, n_steps, pred=pred, stream=stream,
                     node_counts=True, step_begin=11)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # hits == t01 + t11 and the counts add up
    c = b[1]
    assert np.all(c[:, 0] == n_steps)
    assert np.array_equal(c[:, 1], c[:, 3] + c[:, 5])
    assert np.all(c[:, 2:6].sum(axis=1) == n_steps)


@pytest.mark.parametrize("seed", range(30))
def test_oracle_bit_exact_on_small_random_models(orc, ref, seed):
    rm = ref.random_small_model(500 + seed, 2 + seed % 7, 0.05 + 0.02 * (seed % 4))
    text = rm.serialize()
    rplan = ref.parse(text).prepare(1 << 20, 1 + seed % 3, 18)
    a = rplan.simulate_philox(seed, 0, 4, 500, stream=seed % 2, node_counts=True)
    b = orc.simulate(rplan.view, seed, 0, 4, 500, stream=seed % 2, node_counts=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


IDENTITY4 = ("pbn 4\nperturbation 0.2\nnode x0\n  f 1 10 x0\nnode x1\n  f 1 10 x1\n"
             "node x2\n  f 1 10 x2\nnode x3\n  f 1 10 x3\n")


def _find_uniform(cut, alias, want):
    """A single uniform that makes the table emit `want` (test_engine.cpp:133-143)."""
    n = len(cut)
    for cell in range(n):
        if cut[cell] > 0 and cell == want:
            return (cell + cut[cell] * 0.5) / n
        if cut[cell] < 1 and alias[cell] == want:
            return (cell + cut[cell] + (1 - cut[cell]) * 0.5) / n
    raise AssertionError("pattern not reachable")


def test_hand_traced_grouped_perturbation(pb, orc, ref):
    """test_engine.cpp:115-153: force c=0b01 in group 1 -> bit 2 flips,
    two draws consumed, no leaf check."""
    rplan = ref.parse(IDENTITY4).prepare(1 << 20, 2, 18)
    mine = pb.prepare(pb.parse_model(IDENTITY4), 1 << 20, 2, 18)
    assert plan_diff(mine.flat(), flat_of(rplan.view)) == []
    f = mine.flat()
    assert f.pert_groups == 2 and f.pert_k == 2
    z, o = _find_uniform(f.pert_cut, f.pert_alias, 0), _find_uniform(f.pert_cut, f.pert_alias, 1)
    s0 = np.zeros(1, np.uint64)
    for stepper in (lambda s, u: ref_step(rplan, s, u), lambda s, u: orc.step_scripted(mine.view, s, u)):
        st, used = stepper(s0, [z, o])
        assert used == 2
        assert int(st[0]) == 0b0100


def ref_step(rplan, s, u):
    return rplan.step_scripted(s, u)


def test_scripted_steps_agree_on_random_draws(pb, orc, ref):
    text, _ = config_text("c1")
    rplan = ref.parse(text).prepare(1 << 25, 12, 8)
    rng = np.random.default_rng(4)
    words = rplan.n_kept // 64 + 1
    for _ in range(200):
        s = rng.integers(0, 2**63, size=words, dtype=np.uint64)
        s[-1] &= np.uint64((1 << (rplan.n_kept % 64)) - 1)
        u = rng.random(64)
        u[: rng.integers(0, 8)] = 0.999  # make perturbation-free steps common
        a = rplan.step_scripted(s, u)
        b = orc.step_scripted(rplan.view, s, u)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]


CHAIN3 = ("pbn 3\nperturbation 0.001\nnode x0\n  f 1 1\nnode x1\n  f 1 10 x0\n"
          "node x2\n  f 1 10 x1\ninterest x0\n")


def test_two_leaves_give_t_0_998001(pb):
    # test_reduction.cpp:113-121: chain x0 -> x1 -> x2, interest {x0}
    plan = pb.prepare(pb.parse_model(CHAIN3), 1 << 25, 16, 18)
    red = plan.reduced()
    assert list(red["removed"]) == [2, 1]
    assert abs(plan.t - 0.998001) <= 1e-12 * 0.998001
    assert plan.n_kept == 1
    assert list(red["index_map"]) == [0, -1, -1]


def test_perturbation_plan_shapes(pb):
    # test_grouping.cpp:126-145: n'=10, k=4 -> g=3, k=4, k'=2, mask=0b11
    text = "pbn 10\nperturbation 0.01\n" + "".join(f"node v{i}\n  f 1 10 v{i}\n" for i in range(10))
    f = pb.prepare(pb.parse_model(text), 1 << 25, 4, 18).flat()
    assert (f.pert_groups, f.pert_k, f.pert_k_prime, f.pert_mask) == (3, 4, 2, 0b11)
    text4 = "pbn 4\nperturbation 0.01\n" + "".join(f"node v{i}\n  f 1 10 v{i}\n" for i in range(4))
    f = pb.prepare(pb.parse_model(text4), 1 << 25, 16, 18).flat()
    assert (f.pert_groups, f.pert_k, f.pert_k_prime, f.pert_mask) == (1, 4, 4, 0b1111)


def test_masked_perturbation_keeps_rate_p(pb):
    """Theorem 1 (test_grouping.cpp:147-174): the masked last-group draw keeps
    each node's flip rate at p and the bits independent (exact enumeration
    of the alias table's implied distribution)."""
    for k in range(1, 6):
        for p in (0.1, 0.25, 0.5):
            cut, alias = pb.alias_build([p ** bin(c).count("1") * (1 - p) ** (k - bin(c).count("1"))
                                         for c in range(1 << k)])
            n = 1 << k
            cell = np.zeros(n)
            for i in range(n):
                cell[i] += cut[i] / n
                cell[alias[i]] += (1 - cut[i]) / n
            for kp in range(1, k + 1):
                folded = np.zeros(1 << kp)
                for c in range(n):
                    folded[c & ((1 << kp) - 1)] += cell[c]
                for c in range(1 << kp):
                    ones = bin(c).count("1")
                    assert abs(folded[c] - p ** ones * (1 - p) ** (kp - ones)) <= 1e-12


def test_96_nodes_37_5_percent_leaves_keep_60(pb, ref):
    # test_engine.cpp:164-172, on the reference generator's network
    m = ref.generate(96, 1.78, 0.375, 3, 5, 9, 0.001)
    plan = pb.prepare(pb.parse_model(m.serialize()))
    assert plan.n_kept == 60


def test_constant_node_steady_state_10_over_11(orc, pb):
    # test_engine.cpp:58-64: constant-1 node at p = 0.1 has pi(1) = 10/11
    plan = pb.prepare(pb.parse_model("pbn 1\nperturbation 0.1\nnode a\n  f 1 1\n"))
    _, cnt = orc.simulate(plan.view, 1, 0, 1, 400_000, pred=(np.array([0], np.uint32),
                                                               np.array([1], np.uint8)))
    freq = cnt[0, 1] / 400_000
    assert abs(freq - 10 / 11) < 0.003


def test_reference_grouped_rows_match_exact_matrix(ref):
    """The reference's exact one-step distribution of the grouped stepper
    equals the exact chain (test_engine.cpp:239-258) — pins the reference
    build the parity tests run against."""
    rng = np.random.default_rng(82)
    for trial in range(6):
        n = int(2 + rng.integers(0, 4))
        p = 0.25 if trial % 2 else 0.01
        m = ref.random_small_model(900 + trial, n, p)
        mat = m.exact_matrix(n)
        plan = m.prepare(1 << 20, 3, 18)
        red = plan.reduced(n)
        epos = red["engine_pos"]
        to_e = lambda s: sum(1 << int(epos[i]) for i in range(n) if (s >> i) & 1)
        for s in range(1 << n):
            row = plan.grouped_row(to_e(s))
            for sp in range(1 << n):
                assert abs(row[to_e(sp)] - mat[s, sp]) <= 1e-10
