"""The C-ABI library loads without a GPU and exports every symbol declared in
include/pbn_b200.h; device entry points fail loudly (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    hdr = open(os.path.join(ROOT, "include", "pbn_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(pbn_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["pbn_model_parse", "pbn_prepare", "pbn_plan_get_view", "pbn_gpu_create",
                 "pbn_gpu_run", "pbn_gpu_run_device", "pbn_gpu_run_scripted", "pbn_compile_predicate", "pbn_estimate",
                 "pbn_last_error"]:
        assert must in names


def test_every_declared_symbol_is_exported(pb):
    out = subprocess.run(["nm", "-D", "--defined-only", pb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_python_mirror_binds_every_symbol(pb):
    for n in declared_functions():
        assert getattr(pb.lib, n) is not None


def test_state_words_matches_reference_layout(pb):
    # bitstate.hpp:19 -- nbits/64 + 1 words, one slack word
    for n in [1, 63, 64, 65, 1000, 4998]:
        assert pb.lib.pbn_state_words(n) == n // 64 + 1 == pb.state_words(n)


def test_device_path_fails_loudly_without_gpu(pb):
    if pb.device_count() > 0:
        pytest.skip("a GPU is visible")
    model, _ = pb.generate_model(20, (1, 2), (1, 2), 0.05, seed=3)
    plan = pb.prepare(model, 1 << 25, 8, 8)
    with pytest.raises(pb.CudaError):
        pb.GpuEnsemble(plan)


def test_error_codes_mirror_reference_classes(pb):
    with pytest.raises(pb.ModelError):
        pb.parse_model("pbn 1\nperturbation 2\nnode a\n  f 1 1\n")
    model, _ = pb.generate_model(20, (1, 2), (1, 2), 0.05, seed=3)
    with pytest.raises(pb.ResourceError):
        pb.prepare(model, 1 << 25, 25, 8)  # k_max > 24 (perturbation.hpp:30)
    assert pb.ModelError.code == 2 and pb.ResourceError.code == 3


def test_view_arrays_are_consistent(pb):
    model, _ = pb.generate_model(60, (1, 3), (1, 3), 0.01, leaf_frac=0.2, seed=5)
    plan = pb.prepare(model, 1 << 25, 8, 8)
    f = plan.flat()
    assert len(f.pert_cut) == 1 << f.pert_k
    assert np.all(np.diff(f.grp_offset.astype(np.int64)) > 0)
    assert int(f.grp_offset[0]) == 0
    assert np.all(f.fn_gather_count <= 30)
    assert f.pert_groups * f.pert_k >= f.n_kept


def test_null_arguments_are_errors_not_crashes(pb):
    import ctypes as C

    lib = pb.lib
    assert lib.pbn_model_parse(None, 0, C.byref(C.c_void_p())) == 1
    assert lib.pbn_prepare(None, 1 << 25, 16, 18, C.byref(C.c_void_p())) == 1
    m, _ = pb.generate_model(20, (1, 2), (1, 2), 0.05, seed=3)
    plan = pb.prepare(m, 1 << 25, 8, 8)
    assert lib.pbn_compile_predicate(plan._h, None, None, 2, None) == 1
    assert lib.pbn_gpu_create(None, 0, 0, C.byref(C.c_void_p())) == 1
    v = pb.PlanView()
    v.n_groups = 3  # arrays missing
    assert lib.pbn_gpu_create(C.byref(v), 0, 0, C.byref(C.c_void_p())) == 1
    assert b"missing" in lib.pbn_last_error()
    assert lib.pbn_gpu_create(C.byref(plan.view), 0, 3, C.byref(C.c_void_p())) == 1  # bad LPT


def test_inverse_normal_cdf_domain_error_is_reported(pb):
    f = pb.lib.pbn_inverse_normal_cdf
    assert abs(f(0.5)) < 1e-12
    assert f(1.5) != f(1.5)  # NaN outside (0,1), error recorded
    assert b"normal quantile" in pb.lib.pbn_last_error()
