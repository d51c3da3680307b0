"""The reference-side binding (integration/pbn_gpu.hpp, shown in INTEGRATION.md)
compiled against the UNMODIFIED reference headers (oracle/_ref/shim_check,
oracle/Makefile target `shim`), and the reference's own plan fed to the device.

* CPU: the shim builds a view of a `pbn::prepare` plan (engine.hpp:85-164) that
  pbn_gpu_create accepts (it gets as far as the device: PBN_ECUDA here), and a
  view with the leaf draw switched off is refused (PBN_EUSAGE) instead of
  silently shifting the stream (engine.hpp:268).
* GPU: pbn::gpu_ensemble::simulate over the reference plan equals the
  reference's own pbn::simulate(grouped_simulator, ...) (engine.hpp:371-384) on
  the same injected stream, state for state and hit for hit — at the bench
  plans (k = 16) — and the same through the Python mirror (GpuEnsemble over
  oracle.Reference()'s view).
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "shim_check")


def _model_file(pb, tmp_path, n, f, p, pp, leaf, nt, fixed, seed):
    model, terms = pb.generate_model(n, f, p, pp, leaf, nt, fixed, seed)
    path = tmp_path / f"m{seed}.pbn"
    path.write_text(model.serialize())
    return str(path), ",".join(f"{a}={b}" for a, b in terms)


def _shim():
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/shim_check not built (needs /root/reference)")
    return SHIM


def test_shim_view_accepted_and_leafless_view_refused(pb, tmp_path):
    shim = _shim()
    path, pred = _model_file(pb, tmp_path, 100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605)
    out = subprocess.run([shim, path, str(1 << 25), "16", "8", "4", "10", "42", pred,
                          "--no-device"], capture_output=True, text=True, check=True)
    r = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert r["create_rc_without_leaf"] == 1  # PBN_EUSAGE, plan never runs
    if pb.device_count() == 0:
        assert r["create_rc"] == 4  # validated + encoded, then no device
    else:
        assert r["create_rc"] == 0


SHIM_CASES = {
    # name: (n, F, P, p, leaf, n_targets, fixed, seed, k, mgp, n_traj, steps)
    "c1_bench_plan": (100, (1, 3), (1, 3), 0.01, 0.2, 2, True, 1605, 16, 8, 64, 3000),
    "c2_bench_plan": (1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606, 16, 8, 32, 1500),
    "c3_bench_plan": (96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607, 16, 8, 64, 3000),
    "c2_reference_default_plan": (1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606, 16, 18, 16,
                                  800),
}


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(SHIM_CASES))
def test_shim_device_equals_reference_simulate(pb, tmp_path, case):
    shim = _shim()
    n, f, p, pp, leaf, nt, fixed, seed, k, mgp, n_traj, steps = SHIM_CASES[case]
    path, pred = _model_file(pb, tmp_path, n, f, p, pp, leaf, nt, fixed, seed)
    out = subprocess.run([shim, path, str(1 << 25), str(k), str(mgp), str(n_traj), str(steps),
                          "42", pred], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert r["state_mismatches"] == 0 and r["hit_mismatches"] == 0
    # the same job through the C-ABI device group (one ncclAllReduce)
    assert r["group_rc"] == 0 and r["group_state_mismatch"] == 0 and r["group_hits"] == r["hits"]
    assert r["fn_phase_steps"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("k,mgp", [(16, 8), (16, 18)])
def test_reference_plan_view_through_python_mirror(pb, ref, k, mgp):
    model, terms = pb.generate_model(1000, (1, 5), (1, 4), 0.001, 0.0, 3, False, 1606)
    rplan = ref.parse(model.serialize()).prepare(1 << 25, k, mgp)
    pred = rplan.compile_predicate(terms)
    eng = pb.GpuEnsemble(rplan.view)  # the reference's own prepared_simulation, flat view
    n_traj, steps = 24, 600
    st, cnt = eng.simulate(seed=42, n_traj=n_traj, n_steps=steps, pred=pred)
    rst, rcnt = rplan.simulate_philox(42, 0, n_traj, steps, pred=pred)
    assert np.array_equal(st, rst)
    assert np.array_equal(cnt, rcnt)
