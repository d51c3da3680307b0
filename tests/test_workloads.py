"""The committed workload texts (workloads/<name>.pbn.gz, read by both bench
arms) are exactly what the engine's BASELINE-shaped generator produces for
workloads.json, also for the c5 sweep's perturbation rates; and
the reference arm of bench.py never loads the engine library."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("name", sorted(bench.WORKLOADS))
def test_committed_text_is_the_generator_output(pb, name):
    from paper_1605_00854_b200.configs import CONFIGS

    w = CONFIGS[name]
    if bench.WORKLOADS[name].get("generator") == "reference":
        import oracle

        if not os.path.exists(oracle.REF_SO):
            pytest.skip("oracle/_ref not built")
        sys.path.insert(0, os.path.join(ROOT, "workloads"))
        from make_workloads import reference_text

        assert bench.workload_text(name) == reference_text(bench.WORKLOADS[name])
        return
    model, terms = w.model()
    assert bench.workload_text(name) == model.serialize()
    assert [list(t) for t in terms] == bench.WORKLOADS[name]["terms"]
    for p in w.sweep:
        m2, _ = w.model(p)
        assert bench.workload_text(name, p) == m2.serialize()


def test_reference_arm_never_maps_the_engine():
    code = (
        "import sys, runpy; sys.argv=['bench.py']; import bench\n"
        "import oracle\n"
        "assert 'paper_1605_00854_b200' not in sys.modules, sorted(sys.modules)\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libpbn_b200' not in maps\n"
        "print('ok')\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    src = open(os.path.join(ROOT, "bench.py")).read()
    arm = src[src.index("def run_reference_arm("):src.index("def run_estimate_mode(")]
    assert "paper_1605_00854_b200" not in arm and "build_workload" not in arm
