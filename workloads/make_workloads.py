#!/usr/bin/env python3
"""Regenerate the committed workload model texts (workloads/<name>.pbn.gz) and
their predicate terms from the engine's BASELINE-shaped generator
(csrc/host/generator.cpp) with the parameters of workloads.json.

The texts are the interchange format both libraries parse (io.hpp:74-197):
bench.py's reference arm reads them with the reference's own parser and never
loads the engine. tests/test_workloads.py checks the committed files against
the generator.
"""
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def reference_text(d):
    import oracle

    ref = oracle.Reference()
    m = ref.generate(d["n"], d["density"], d["leaf_frac"], d["f_range"][1], d["p_range"][1],
                     d["seed"], d["p"])
    return m.serialize()


def main():
    from paper_1605_00854_b200.configs import CONFIGS

    path = os.path.join(HERE, "workloads.json")
    table = json.load(open(path))
    for name, w in CONFIGS.items():
        if table[name].get("generator") == "reference":
            # the acceptance profiles (acceptance.cpp:202): the reference's own
            # generator (generate.hpp:34-176) through oracle/_ref, exactly as
            # run_benchmark (bench.hpp:170-185) calls it
            text = reference_text(table[name])
            terms = []
        else:
            model, terms = w.model()
            text = model.serialize()
        with gzip.GzipFile(os.path.join(HERE, f"{name}.pbn.gz"), "wb", mtime=0) as f:
            f.write(text.encode())
        table[name]["terms"] = [[int(a), int(b)] for a, b in terms]
    with open(path, "w") as f:
        json.dump(table, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
