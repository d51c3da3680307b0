"""The model text parser (csrc/host/model.cpp) against the unmodified
reference parser (io.hpp:74-226, model.hpp:81-117, through oracle/_ref) on
valid and systematically corrupted texts: the same accept/reject decision,
the same error class and message (line numbers included), and byte-identical
serialisation of what both accept."""
import random

import pytest

BASE = ("# net\npbn 4\nperturbation 0.01\n"
        "node a\n  f 0.6 1000 b c\n  f 0.4 10 d\n"
        "node b\n  f 1 01 a\n"
        "node c\n  f 0.5 0110 a b\n  f 0.5 1 \n"
        "node d\n  f 1 10 c\n"
        "interest a c\n")


def mutations(text, rng, n):
    lines = text.split("\n")
    out = [text, text.replace("\n", "\r\n"), text.rstrip("\n"), text.replace("interest a c\n", "")]
    edits = [
        lambda L, i: L[:i] + L[i + 1:],                                   # drop a line
        lambda L, i: L[:i] + [L[i]] + L[i:],                              # duplicate a line
        lambda L, i: L[:i] + ["bogus x"] + L[i:],                         # unknown directive
        lambda L, i: L[:i] + ["  # only a comment"] + L[i:],
        lambda L, i: L[:i] + [L[i].replace("1", "2", 1)] + L[i + 1:],     # non-binary / numbers
        lambda L, i: L[:i] + [L[i].replace("0", "x", 1)] + L[i + 1:],
        lambda L, i: L[:i] + [L[i] + " a"] + L[i + 1:],                   # extra parent/token
        lambda L, i: L[:i] + [L[i].replace("0.5", "0.25", 1)] + L[i + 1:],  # bad sums
        lambda L, i: L[:i] + [L[i].replace("b", "zz", 1)] + L[i + 1:],    # unknown names
        lambda L, i: L[:i] + [L[i].replace("0.01", "1e-400", 1)] + L[i + 1:],
        lambda L, i: L[:i] + [L[i].replace("4", "-1", 1)] + L[i + 1:],
        lambda L, i: L[:i] + [L[i].replace("node d", "node a", 1)] + L[i + 1:],
    ]
    for _ in range(n):
        L = list(lines)
        for _ in range(rng.randint(1, 2)):
            i = rng.randrange(len(L))
            L = rng.choice(edits)(L, i)
        out.append("\n".join(L))
    return out


def outcome_mine(pb, text):
    try:
        return ("ok", pb.parse_model(text).serialize())
    except pb.PbnError as e:
        return (type(e).__name__, str(e))


def outcome_ref(ref, text):
    import oracle

    try:
        return ("ok", ref.parse(text).serialize())
    except oracle.RefError as e:
        return ({2: "ModelError", 3: "ResourceError"}.get(e.code, str(e.code)), str(e))


@pytest.mark.parametrize("seed", range(4))
def test_parser_matches_reference_on_corrupted_texts(pb, ref, seed):
    rng = random.Random(seed)
    texts = mutations(BASE, rng, 150)
    ok = 0
    for t in texts:
        mine, theirs = outcome_mine(pb, t), outcome_ref(ref, t)
        assert mine == theirs, (t, mine, theirs)
        ok += mine[0] == "ok"
    assert 0 < ok < len(texts)  # both accepted and rejected inputs were exercised
