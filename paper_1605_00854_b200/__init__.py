"""pbn_b200 — B200-native PBN trajectory engine (arxiv 1605.00854 hot path).

Python mirror of the reference's host interface over the C-ABI in
``include/pbn_b200.h`` (``libpbn_b200.so``, built in-tree). Names follow the
reference (``/root/reference/proj/include/pbn``):

==============================  =================================================
reference                       here
==============================  =================================================
``parse_model`` io.hpp:74       :func:`parse_model` -> :class:`Model`
``serialize_model`` io.hpp:205  :meth:`Model.serialize`
``prepare`` engine.hpp:85       :func:`prepare` -> :class:`PreparedSimulation`
``compile_predicate`` :357      :meth:`PreparedSimulation.compile_predicate`
``simulate`` engine.hpp:371     :meth:`GpuEnsemble.simulate` (ensemble of trajectories)
==============================  =================================================

Errors mirror the reference's exception classes (errors.hpp:10-32):
:class:`ModelError` (exit code 2), :class:`ResourceError` (3); device
failures raise :class:`CudaError`. There is no CPU fallback: if the shared
library is missing, importing this package raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PBN_B200_LIB selects an alternative in-tree build (A/B measurements of
# compile-time variants, see Makefile `variant`)
LIB_PATH = os.environ.get("PBN_B200_LIB") or os.path.join(_HERE, "libpbn_b200.so")

STREAM_U53 = 0
STREAM_U32 = 1
RUN_NODE_COUNTS = 1
RUN_EXACT_ALIAS = 2
COUNT_FIELDS = 8
C_STEPS, C_HITS, C_T00, C_T01, C_T10, C_T11, C_FNSTEPS, C_PERTSTEPS = range(8)
DEFAULT_THETA = 1 << 25  # engine.hpp:81
DEFAULT_K = 16  # engine.hpp:82
DEFAULT_MGP = 18  # engine.hpp:83


class PbnError(RuntimeError):
    code = 1


class UsageError(PbnError):
    code = 1


class ModelError(PbnError):
    code = 2


class ResourceError(PbnError):
    code = 3


class CudaError(PbnError):
    code = 4


_ERRORS = {1: UsageError, 2: ModelError, 3: ResourceError, 4: CudaError}


class PlanView(C.Structure):
    _fields_ = [
        ("n_kept", C.c_uint32), ("t", C.c_double),
        ("pert_groups", C.c_uint32), ("pert_k", C.c_uint32), ("pert_k_prime", C.c_uint32),
        ("pert_size", C.c_uint32), ("pert_mask", C.c_uint64),
        ("pert_cut", C.POINTER(C.c_double)), ("pert_alias", C.POINTER(C.c_uint32)),
        ("n_groups", C.c_uint32),
        ("grp_offset", C.POINTER(C.c_uint32)), ("grp_fn_begin", C.POINTER(C.c_uint32)),
        ("grp_alias_begin", C.POINTER(C.c_uint32)), ("grp_alias_size", C.POINTER(C.c_uint32)),
        ("n_alias", C.c_uint64), ("alias_cut", C.POINTER(C.c_double)),
        ("alias_idx", C.POINTER(C.c_uint32)),
        ("n_fns", C.c_uint32), ("fn_gather_begin", C.POINTER(C.c_uint64)),
        ("fn_table_begin", C.POINTER(C.c_uint64)), ("fn_gather_count", C.POINTER(C.c_uint32)),
        ("n_gather", C.c_uint64), ("fn_gather", C.POINTER(C.c_uint32)),
        ("n_table", C.c_uint64), ("fn_tables", C.POINTER(C.c_uint64)),
        ("pert_mode", C.c_uint32), ("has_leaf", C.c_uint32), ("pert_p", C.c_double),
        ("grp_members", C.POINTER(C.c_uint32)),
    ]


class GenParams(C.Structure):
    _fields_ = [
        ("n", C.c_uint32), ("f_min", C.c_uint32), ("f_max", C.c_uint32),
        ("p_min", C.c_uint32), ("p_max", C.c_uint32), ("leaf_frac", C.c_double),
        ("perturbation", C.c_double), ("n_targets", C.c_uint32),
        ("targets_fixed", C.c_uint32), ("seed", C.c_uint64),
    ]


class RunArgs(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("traj_begin", C.c_uint64), ("n_traj", C.c_uint32),
        ("stream", C.c_uint32), ("step_begin", C.c_uint64), ("n_steps", C.c_uint64),
        ("pred_bits", C.POINTER(C.c_uint32)), ("pred_vals", C.POINTER(C.c_uint8)),
        ("n_pred", C.c_uint32), ("flags", C.c_uint32),
        ("kappa", C.c_uint32), ("thin_mode", C.c_uint32), ("tprev", C.POINTER(C.c_uint8)),
        ("series", C.POINTER(C.c_uint32)), ("series_stride", C.c_uint64),
        ("series_bit0", C.c_uint64), ("series_init", C.c_uint32), ("reserved", C.c_uint32),
    ]


class EstimateRequest(C.Structure):
    _fields_ = [
        ("precision", C.c_double), ("confidence", C.c_double), ("pilot", C.c_uint64),
        ("burn_epsilon", C.c_double), ("max_refinements", C.c_uint32),
        ("sample_inflation", C.c_double), ("seed", C.c_uint64), ("traj_begin", C.c_uint64),
        ("n_traj", C.c_uint32), ("stream", C.c_uint32),
    ]


class EstimateResult(C.Structure):
    _fields_ = [
        ("estimate", C.c_double), ("sample_size_used", C.c_uint64), ("burn_in_used", C.c_uint64),
        ("steps_per_traj", C.c_uint64), ("kappa", C.c_uint32), ("degenerate", C.c_uint32),
        ("alpha", C.c_double), ("beta", C.c_double), ("wall_seconds", C.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


RUN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                     C.c_uint64, C.c_uint32, C.POINTER(C.c_uint64))
STATS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint64))


class EstimatorBackend(C.Structure):
    _fields_ = [("user", C.c_void_p), ("n_traj", C.c_uint32), ("reserved", C.c_uint32),
                ("series_capacity", C.c_uint64), ("run", RUN_FN), ("series_stats", STATS_FN)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, U32, U64, I = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    sig = {
        "pbn_last_error": (C.c_char_p, []),
        "pbn_version": (C.c_char_p, []),
        "pbn_state_words": (U32, [U32]),
        "pbn_model_parse": (I, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
        "pbn_model_serialize": (I, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
        "pbn_model_generate": (I, [C.POINTER(GenParams), C.POINTER(P), C.POINTER(U32),
                                   C.POINTER(C.c_uint8), C.POINTER(U32)]),
        "pbn_model_info": (I, [P, C.POINTER(U32), C.POINTER(C.c_double), C.POINTER(U32),
                               C.POINTER(C.c_double)]),
        "pbn_model_node_index": (I, [P, C.c_char_p, C.POINTER(U32)]),
        "pbn_model_node_name": (I, [P, U32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
        "pbn_model_free": (None, [P]),
        "pbn_prepare": (I, [P, U64, U32, U32, C.POINTER(P)]),
        "pbn_plan_get_view": (I, [P, C.POINTER(PlanView)]),
        "pbn_prepare_nodewise": (I, [P, I, C.POINTER(P)]),
        "pbn_plan_reduced": (I, [P, C.POINTER(U32), C.POINTER(U32), C.POINTER(C.c_int32),
                                 C.POINTER(U32), C.POINTER(U32)]),
        "pbn_plan_groups": (I, [P, C.POINTER(U32), C.POINTER(U32)]),
        "pbn_compile_predicate": (I, [P, C.POINTER(U32), C.POINTER(C.c_uint8), U32,
                                      C.POINTER(U32)]),
        "pbn_plan_free": (None, [P]),
        "pbn_device_count": (I, [C.POINTER(I)]),
        "pbn_gpu_create": (I, [C.POINTER(PlanView), I, U32, C.POINTER(P)]),
        "pbn_gpu_set_placement": (I, [P, U32]),
        "pbn_gpu_info": (I, [P, C.POINTER(U32), C.POINTER(U32), C.POINTER(U64), C.POINTER(U64),
                             C.POINTER(U32)]),
        "pbn_gpu_run": (I, [P, C.POINTER(RunArgs), C.POINTER(U64), C.POINTER(U64),
                            C.POINTER(U64)]),
        "pbn_gpu_run_device": (I, [P, C.POINTER(RunArgs), P, P, P, P]),
        "pbn_gpu_run_scripted": (I, [P, C.POINTER(RunArgs), C.POINTER(C.c_double), U64,
                                     C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]),
        "pbn_gpu_last_launches": (U32, [P]),
        "pbn_gpu_last_kernel": (I, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
        "pbn_gpu_plan_launch": (I, [P, U32, U32, U32, C.c_char_p, C.c_size_t,
                                    C.POINTER(C.c_size_t)]),
        "pbn_gpu_destroy": (None, [P]),
        "pbn_philox_kat": (I, [C.POINTER(U32), U32, U64, C.POINTER(U32)]),
        "pbn_estimate": (I, [P, C.POINTER(EstimateRequest), C.POINTER(U32), C.POINTER(C.c_uint8),
                             U32, C.POINTER(U64), C.POINTER(EstimateResult)]),
        "pbn_estimate_with_backend": (I, [C.POINTER(EstimateRequest), C.POINTER(EstimatorBackend),
                                          C.POINTER(EstimateResult)]),
        "pbn_series_stats_host": (I, [C.POINTER(U32), U32, U64, U64, U32, C.POINTER(U64)]),
        "pbn_inverse_normal_cdf": (C.c_double, [C.c_double]),
        "pbn_series_stats_device": (I, [I, P, U32, U64, U64, U32, C.POINTER(U64)]),
        "pbn_group_create": (I, [C.POINTER(PlanView), C.POINTER(I), U32, U32, C.POINTER(P)]),
        "pbn_nccl_unique_id": (I, [C.POINTER(C.c_uint8)]),
        "pbn_group_create_rank": (I, [C.POINTER(PlanView), I, U32, U32, C.POINTER(C.c_uint8), U32,
                                      C.POINTER(P)]),
        "pbn_group_info": (I, [P, C.POINTER(U32), C.POINTER(U32), C.POINTER(U32)]),
        "pbn_group_shard": (I, [P, U64, U32, C.POINTER(U64), C.POINTER(U64)]),
        "pbn_group_member": (I, [P, U32, C.POINTER(P)]),
        "pbn_group_run": (I, [P, C.POINTER(RunArgs), C.POINTER(U64), C.POINTER(U64),
                              C.POINTER(U64), C.POINTER(U64)]),
        "pbn_group_destroy": (None, [P]),
        "pbn_internal_plan_layout": (I, [C.POINTER(PlanView), C.POINTER(U64), U32]),
        "pbn_internal_lower_bound": (U32, [C.POINTER(U32), U32, U64]),
        "pbn_internal_greedy_partition": (I, [C.POINTER(U32), U32, U32, C.POINTER(U32)]),
        "pbn_internal_alias_build": (I, [C.POINTER(C.c_double), U32, C.POINTER(C.c_double),
                                         C.POINTER(U32)]),
        "pbn_internal_alias53_pick": (I, [C.POINTER(C.c_double), C.POINTER(U32), U32,
                                          C.POINTER(U64), U64, C.POINTER(U32),
                                          C.POINTER(C.c_uint8)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
EXPORTED_SYMBOLS = (
    "pbn_last_error", "pbn_version", "pbn_state_words", "pbn_model_parse", "pbn_model_serialize",
    "pbn_model_generate", "pbn_model_info", "pbn_model_node_index", "pbn_model_node_name",
    "pbn_model_free", "pbn_prepare", "pbn_prepare_nodewise",
    "pbn_plan_get_view", "pbn_plan_reduced", "pbn_plan_groups", "pbn_compile_predicate",
    "pbn_plan_free", "pbn_device_count", "pbn_gpu_create", "pbn_gpu_set_placement", "pbn_gpu_info", "pbn_gpu_run",
    "pbn_gpu_run_device", "pbn_gpu_run_scripted", "pbn_gpu_last_launches", "pbn_gpu_last_kernel", "pbn_gpu_plan_launch",
    "pbn_gpu_destroy", "pbn_estimate",
    "pbn_estimate_with_backend", "pbn_series_stats_host", "pbn_inverse_normal_cdf",
    "pbn_series_stats_device", "pbn_group_create", "pbn_nccl_unique_id", "pbn_group_create_rank",
    "pbn_group_info", "pbn_group_shard", "pbn_group_member", "pbn_group_run", "pbn_group_destroy",
)


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.pbn_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, PbnError)(msg)


def _u32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def state_words(n_kept: int) -> int:
    """Words per trajectory state (bitstate.hpp:19: n/64 + 1, one slack word)."""
    return n_kept // 64 + 1


# ----------------------------------------------------------------------------
class Model:
    """Parsed, validated PBN (model.hpp:57-69)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if lib is not None and getattr(self, "_h", None) and self._h.value:
            lib.pbn_model_free(self._h)
            self._h = C.c_void_p(None)

    def serialize(self) -> str:
        n = C.c_size_t(0)
        _check(lib.pbn_model_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.pbn_model_serialize(self._h, buf, n.value + 1, C.byref(n)))
        return buf.raw[: n.value].decode()

    def info(self):
        n, ni = C.c_uint32(), C.c_uint32()
        p, d = C.c_double(), C.c_double()
        _check(lib.pbn_model_info(self._h, C.byref(n), C.byref(p), C.byref(ni), C.byref(d)))
        return {"n": n.value, "p": p.value, "n_interest": ni.value, "density": d.value}

    @property
    def n(self) -> int:
        return self.info()["n"]

    def node_name(self, i: int) -> str:
        n = C.c_size_t()
        _check(lib.pbn_model_node_name(self._h, i, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.pbn_model_node_name(self._h, i, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def node_index(self, name: str) -> int:
        out = C.c_uint32()
        _check(lib.pbn_model_node_index(self._h, name.encode(), C.byref(out)))
        return out.value


def parse_model(text: str) -> Model:
    """io.hpp:74-197: parse + validate a PBN text model."""
    h = C.c_void_p()
    raw = text.encode()
    _check(lib.pbn_model_parse(raw, len(raw), C.byref(h)))
    return Model(h.value)


def generate_model(n, f_range, p_range, p, leaf_frac=0.0, n_targets=2, targets_fixed=False,
                   seed=1605):
    """BASELINE-shaped synthetic network. Returns (model, predicate terms)."""
    gp = GenParams(n, f_range[0], f_range[1], p_range[0], p_range[1], leaf_frac, p, n_targets,
                   1 if targets_fixed else 0, seed)
    h = C.c_void_p()
    nodes = (C.c_uint32 * max(1, n_targets))()
    vals = (C.c_uint8 * max(1, n_targets))()
    cnt = C.c_uint32()
    _check(lib.pbn_model_generate(C.byref(gp), C.byref(h), nodes, vals, C.byref(cnt)))
    return Model(h.value), [(int(nodes[i]), int(vals[i])) for i in range(cnt.value)]


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


@dataclass
class FlatPlan:
    """Copy of the flat hot-loop arrays (engine.hpp:22-79)."""

    n_kept: int
    t: float
    pert_groups: int
    pert_k: int
    pert_k_prime: int
    pert_mask: int
    pert_cut: np.ndarray
    pert_alias: np.ndarray
    grp_offset: np.ndarray
    grp_fn_begin: np.ndarray
    grp_alias_begin: np.ndarray
    grp_alias_size: np.ndarray
    alias_cut: np.ndarray
    alias_idx: np.ndarray
    fn_gather_begin: np.ndarray
    fn_table_begin: np.ndarray
    fn_gather_count: np.ndarray
    fn_gather: np.ndarray
    fn_tables: np.ndarray

    @staticmethod
    def from_view(v: PlanView) -> "FlatPlan":
        return FlatPlan(
            v.n_kept, v.t, v.pert_groups, v.pert_k, v.pert_k_prime, v.pert_mask,
            _arr(v.pert_cut, v.pert_size, np.float64), _arr(v.pert_alias, v.pert_size, np.uint32),
            _arr(v.grp_offset, v.n_groups, np.uint32), _arr(v.grp_fn_begin, v.n_groups, np.uint32),
            _arr(v.grp_alias_begin, v.n_groups, np.uint32),
            _arr(v.grp_alias_size, v.n_groups, np.uint32),
            _arr(v.alias_cut, v.n_alias, np.float64), _arr(v.alias_idx, v.n_alias, np.uint32),
            _arr(v.fn_gather_begin, v.n_fns, np.uint64), _arr(v.fn_table_begin, v.n_fns, np.uint64),
            _arr(v.fn_gather_count, v.n_fns, np.uint32), _arr(v.fn_gather, v.n_gather, np.uint32),
            _arr(v.fn_tables, v.n_table, np.uint64))

    def expected_lookups(self, fn_steps: int, steps: int) -> int:
        """Algorithmic table probes: g per step + (A + G) per function-phase step."""
        a = int(np.count_nonzero(self.grp_alias_size))
        return self.pert_groups * steps + fn_steps * (a + len(self.grp_offset))


class PreparedSimulation:
    """engine.hpp:22-79 — immutable plan built by :func:`prepare`."""

    def __init__(self, handle, model: Model, theta, k_max, mgp):
        self._h = C.c_void_p(handle)
        self.model = model
        self.theta, self.k_max, self.max_group_parents = theta, k_max, mgp
        self._view = PlanView()
        _check(lib.pbn_plan_get_view(self._h, C.byref(self._view)))

    def __del__(self):
        if lib is not None and getattr(self, "_h", None) and self._h.value:
            lib.pbn_plan_free(self._h)
            self._h = C.c_void_p(None)

    @property
    def view(self) -> PlanView:
        return self._view

    @property
    def n_kept(self) -> int:
        return self._view.n_kept

    @property
    def t(self) -> float:
        return self._view.t

    def flat(self) -> FlatPlan:
        return FlatPlan.from_view(self._view)

    def reduced(self):
        on, nr = C.c_uint32(), C.c_uint32()
        _check(lib.pbn_plan_reduced(self._h, C.byref(on), C.byref(nr), None, None, None))
        imap = np.zeros(on.value, np.int32)
        epos = np.zeros(self.n_kept, np.uint32)
        rem = np.zeros(max(1, nr.value), np.uint32)
        _check(lib.pbn_plan_reduced(self._h, None, None, imap.ctypes.data_as(C.POINTER(C.c_int32)),
                                    _u32p(epos), _u32p(rem)))
        return {"original_n": on.value, "removed": rem[: nr.value], "index_map": imap,
                "engine_pos": epos}

    def groups(self):
        cum = np.zeros(self._view.n_groups + 1, np.uint32)
        mem = np.zeros(self.n_kept, np.uint32)
        _check(lib.pbn_plan_groups(self._h, _u32p(mem), _u32p(cum)))
        return mem, cum

    def compile_predicate(self, terms):
        """engine.hpp:357-362: [(node, value)] over original indices -> engine bits."""
        nodes = np.array([t[0] for t in terms], np.uint32)
        vals = np.array([1 if t[1] else 0 for t in terms], np.uint8)
        bits = np.zeros(len(terms), np.uint32)
        _check(lib.pbn_compile_predicate(self._h, _u32p(nodes),
                                         vals.ctypes.data_as(C.POINTER(C.c_uint8)), len(terms),
                                         _u32p(bits)))
        return bits, vals


def prepare(model: Model, theta=DEFAULT_THETA, k_max=DEFAULT_K, max_group_parents=DEFAULT_MGP):
    """engine.hpp:85-164: reduce -> perturbation plan -> partition -> flatten."""
    h = C.c_void_p()
    _check(lib.pbn_prepare(model._h, theta, k_max, max_group_parents, C.byref(h)))
    return PreparedSimulation(h.value, model, theta, k_max, max_group_parents)


PLAN_LAYOUT_FIELDS = ("off_pert53", "off_pert32", "off_groups", "off_fns", "off_grec", "off_acut",
                      "off_aidx", "off_acell", "off_arec", "off_scol", "off_arec4", "off_tables",
                      "off_fns_s", "off_acell_s", "core_bytes", "table_bytes", "blob_bytes",
                      "total_bytes", "n_alias_groups", "n_single_alias", "n_groups", "sw32",
                      "rg_ok", "single_compact")


def plan_layout(plan) -> dict:
    """Device encoding sizes/offsets of a plan (no device needed)."""
    out = np.zeros(len(PLAN_LAYOUT_FIELDS), np.uint64)
    view = plan.view if isinstance(plan, PreparedSimulation) else plan
    _check(lib.pbn_internal_plan_layout(C.byref(view), _u64p(out), len(out)))
    return {k: int(v) for k, v in zip(PLAN_LAYOUT_FIELDS, out)}


def lower_bound(weights, theta):
    """grouping.hpp:50-57 (test hook)."""
    w = np.ascontiguousarray(weights, np.uint32)
    return int(lib.pbn_internal_lower_bound(_u32p(w), len(w), theta))


def greedy_partition(weights, m):
    """grouping.hpp:63-82 (test hook): list of m lists of item indices."""
    w = np.ascontiguousarray(weights, np.uint32)
    part = np.zeros(len(w), np.uint32)
    _check(lib.pbn_internal_greedy_partition(_u32p(w), len(w), m, _u32p(part)))
    out = [[] for _ in range(m)]
    order = sorted(range(len(w)), key=lambda i: (-int(w[i]), i))
    for i in order:  # insertion order of the greedy pass
        out[int(part[i])].append(i)
    return out


def alias_build(probs):
    """alias.hpp:18-56 (test hook): (cut-offs, aliases)."""
    p = np.ascontiguousarray(probs, np.float64)
    cut = np.zeros(len(p), np.float64)
    al = np.zeros(len(p), np.uint32)
    _check(lib.pbn_internal_alias_build(p.ctypes.data_as(C.POINTER(C.c_double)), len(p),
                                        cut.ctypes.data_as(C.POINTER(C.c_double)), _u32p(al)))
    return cut, al


def alias53_pick(cut, alias, raw):
    """Test hook: the kernel's integer U53 combined-function choice (dev_plan.h
    a53) on raw draw words; returns (picks, took_fast_path)."""
    cut = np.ascontiguousarray(cut, np.float64)
    alias = np.ascontiguousarray(alias, np.uint32)
    raw = np.ascontiguousarray(raw, np.uint64)
    pick = np.zeros(len(raw), np.uint32)
    fast = np.zeros(len(raw), np.uint8)
    _check(lib.pbn_internal_alias53_pick(cut.ctypes.data_as(C.POINTER(C.c_double)), _u32p(alias),
                                         len(cut), _u64p(raw), len(raw), _u32p(pick),
                                         fast.ctypes.data_as(C.POINTER(C.c_uint8))))
    return pick, fast.astype(bool)


def prepare_nodewise(model: Model, reduced: bool):
    """Plan of the reference's node-by-node steppers: Method_old
    (reference_simulator, engine.hpp:168-221) on the full model, or
    Method_reduction (reduced_simulator, engine.hpp:225-242)."""
    h = C.c_void_p()
    _check(lib.pbn_prepare_nodewise(model._h, 1 if reduced else 0, C.byref(h)))
    return PreparedSimulation(h.value, model, None, None, None)


def device_count() -> int:
    c = C.c_int(0)
    _check(lib.pbn_device_count(C.byref(c)))
    return c.value


def philox_kat_device(ctrs: np.ndarray, seed: int) -> np.ndarray:
    """Run Philox4x32-10 on the device for (n,4) uint32 counters (stream known-answer tests)."""
    ctrs = np.ascontiguousarray(ctrs, dtype=np.uint32)
    out = np.zeros_like(ctrs)
    _check(lib.pbn_philox_kat(_u32p(ctrs), ctrs.shape[0], seed, _u32p(out)))
    return out


class GpuEnsemble:
    """Device-resident plan + ensemble stepping: the drop-in for
    ``simulate(grouped_simulator, ...)`` (engine.hpp:371-384) over many
    trajectories, keyed by (seed, global trajectory id, step)."""

    def __init__(self, plan, device: int = 0, lanes_per_traj: int = 0, placement: str = "auto"):
        view = plan.view if isinstance(plan, PreparedSimulation) else plan
        if not isinstance(view, PlanView):
            # any structure with the pbn_plan_view layout (e.g. a reference-side
            # view of pbn::prepare's plan, oracle/_ref): reinterpret, no copy
            if C.sizeof(view) != C.sizeof(PlanView):
                raise UsageError("plan view layout does not match pbn_plan_view")
            view = C.cast(C.pointer(view), C.POINTER(PlanView)).contents
        self._keep = plan  # the view's arrays must outlive creation
        self.n_kept = view.n_kept
        self.words = state_words(self.n_kept)
        h = C.c_void_p()
        _check(lib.pbn_gpu_create(C.byref(view), device, lanes_per_traj, C.byref(h)))
        self._h = h
        self._device = device
        if placement != "auto":
            self.set_placement(placement)

    def __del__(self):
        if lib is not None and getattr(self, "_h", None) and self._h.value:
            lib.pbn_gpu_destroy(self._h)
            self._h = C.c_void_p(None)

    def set_placement(self, placement: str) -> None:
        """'auto' | 'global' | 'core' | 'tables' | 'all' (staged prefix of the plan)."""
        code = {"auto": 0, "global": 1, "core": 2, "tables": 3, "all": 4, "core_pert": 5}[placement]
        _check(lib.pbn_gpu_set_placement(self._h, code))

    def info(self):
        lpt, place, wpc = C.c_uint32(), C.c_uint32(), C.c_uint32()
        sm, pb = C.c_uint64(), C.c_uint64()
        _check(lib.pbn_gpu_info(self._h, C.byref(lpt), C.byref(place), C.byref(sm), C.byref(pb),
                                C.byref(wpc)))
        return {"lanes_per_traj": lpt.value, "placement": ("global", "core", "tables", "all", "core_pert")[place.value],
                "staged_smem_bytes": sm.value, "plan_bytes": pb.value,
                "warps_per_cta": wpc.value, "kernel": self.last_kernel()}

    def _args(self, seed, traj_begin, n_traj, n_steps, step_begin, pred, stream):
        a = RunArgs()
        a.seed, a.traj_begin, a.n_traj = seed, traj_begin, n_traj
        a.stream, a.step_begin, a.n_steps = stream, step_begin, n_steps
        if pred is not None and len(pred[0]):
            bits = np.ascontiguousarray(pred[0], np.uint32)
            vals = np.ascontiguousarray(pred[1], np.uint8)
            self._pred_keep = (bits, vals)
            a.pred_bits = _u32p(bits)
            a.pred_vals = vals.ctypes.data_as(C.POINTER(C.c_uint8))
            a.n_pred = len(bits)
        return a

    def simulate(self, seed, n_traj, n_steps, traj_begin=0, step_begin=0, states=None,
                 pred=None, stream=STREAM_U53, kappa=1, thin_mode=0, tprev=None, series=None,
                 series_bit0=0, series_init=False, node_counts=False, exact_alias=False):
        """HOST buffers in/out. states: (n_traj, words) uint64 engine-order (zeros if None).
        pred: (engine bits, values) from PreparedSimulation.compile_predicate.
        kappa/thin_mode/tprev: sampled predicate transitions (see pbn_run_args);
        series: (n_traj, stride) uint32 bit rows updated in place.
        exact_alias: every U53 combined-function choice takes the FP64 path
        (checks the integer fast path against it; same results, slower).
        Returns (states, counts[n_traj, 8])."""
        if states is None:
            states = np.zeros((n_traj, self.words), np.uint64)
        states = np.ascontiguousarray(states, np.uint64).copy()
        assert states.shape == (n_traj, self.words)
        counts = np.zeros((n_traj, COUNT_FIELDS), np.uint64)
        a = self._args(seed, traj_begin, n_traj, n_steps, step_begin, pred, stream)
        a.kappa, a.thin_mode = kappa, thin_mode
        if tprev is not None:
            assert tprev.dtype == np.uint8 and tprev.flags.c_contiguous and len(tprev) == n_traj
            a.tprev = tprev.ctypes.data_as(C.POINTER(C.c_uint8))
        if series is not None:
            assert series.dtype == np.uint32 and series.flags.c_contiguous
            a.series = _u32p(series)
            a.series_stride = series.shape[1]
            a.series_bit0, a.series_init = series_bit0, 1 if series_init else 0
        if exact_alias:
            a.flags |= RUN_EXACT_ALIAS
        nc = None
        if node_counts:
            a.flags |= RUN_NODE_COUNTS
            nc = np.zeros((n_traj, self.n_kept), np.uint64)
        _check(lib.pbn_gpu_run(self._h, C.byref(a), _u64p(states), _u64p(counts),
                               _u64p(nc) if nc is not None else None))
        return (states, counts, nc) if node_counts else (states, counts)

    def simulate_device(self, seed, n_traj, n_steps, d_states, d_counts, traj_begin=0,
                        step_begin=0, pred=None, stream=STREAM_U53, cuda_stream=0, kappa=1,
                        thin_mode=0, d_tprev=None, d_series=None, series_stride=0,
                        series_bit0=0, series_init=False, d_node_counts=None):
        """DEVICE pointers (ints, e.g. torch tensor .data_ptr()), asynchronous."""
        a = self._args(seed, traj_begin, n_traj, n_steps, step_begin, pred, stream)
        a.kappa, a.thin_mode = kappa, thin_mode
        if d_tprev is not None:
            a.tprev = C.cast(C.c_void_p(d_tprev), C.POINTER(C.c_uint8))
        if d_series is not None:
            a.series = C.cast(C.c_void_p(d_series), C.POINTER(C.c_uint32))
            a.series_stride, a.series_bit0 = series_stride, series_bit0
            a.series_init = 1 if series_init else 0
        if d_node_counts is not None:
            a.flags |= RUN_NODE_COUNTS
        _check(lib.pbn_gpu_run_device(self._h, C.byref(a), C.c_void_p(d_states),
                                      C.c_void_p(d_counts),
                                      C.c_void_p(d_node_counts) if d_node_counts else None,
                                      C.c_void_p(cuda_stream)))

    def simulate_scripted(self, draws, n_steps, states=None, pred=None):
        """Forced-draw replay (pbn_gpu_run_scripted; the reference tests'
        scripted_rng, tests/oracles.hpp:235-254): draws is (n_traj, n_draws)
        float64 — or one row for one trajectory — consumed in the reference's
        call order, wrapping around. Returns (states, counts, consumed)."""
        draws = np.ascontiguousarray(np.atleast_2d(np.asarray(draws, np.float64)))
        n_traj = draws.shape[0]
        if states is None:
            states = np.zeros((n_traj, self.words), np.uint64)
        states = np.ascontiguousarray(states, np.uint64).copy()
        assert states.shape == (n_traj, self.words)
        counts = np.zeros((n_traj, COUNT_FIELDS), np.uint64)
        consumed = np.zeros(n_traj, np.uint64)
        a = self._args(0, 0, n_traj, n_steps, 0, pred, STREAM_U53)
        _check(lib.pbn_gpu_run_scripted(self._h, C.byref(a),
                                        draws.ctypes.data_as(C.POINTER(C.c_double)),
                                        draws.shape[1], _u64p(states), _u64p(counts),
                                        _u64p(consumed)))
        return states, counts, consumed

    @property
    def device(self) -> int:
        return self._device

    def last_launches(self) -> int:
        return int(lib.pbn_gpu_last_launches(self._h))

    def last_kernel(self) -> str:
        """The kernel instantiation the last run launched (pbn_gpu_last_kernel)."""
        buf = C.create_string_buffer(256)
        _check(lib.pbn_gpu_last_kernel(self._h, buf, 256, None))
        return buf.value.decode()

    def plan_launch(self, n_traj: int, stream: int = STREAM_U53, node_counts: bool = False) -> str:
        """The kernel a run of n_traj trajectories would launch (pbn_gpu_plan_launch)."""
        buf = C.create_string_buffer(256)
        _check(lib.pbn_gpu_plan_launch(self._h, n_traj, stream,
                                       RUN_NODE_COUNTS if node_counts else 0, buf, 256, None))
        return buf.value.decode()


class GpuGroup:
    """One ensemble over several GPUs through the C-ABI device group
    (pbn_group_*): contiguous per-rank trajectory ranges, the plan
    replicated, ONE ncclAllReduce of the pooled counts (+ per-node one-counts).

    GpuGroup(plan, devices=[0, 1, ...])            one process, every device
    GpuGroup(plan, device=d, nranks=R, rank=r, nccl_id=id)   one process per device
    (nccl_id: 128 bytes from nccl_unique_id() on one rank, shared by the caller)."""

    def __init__(self, plan, devices=None, lanes_per_traj=0, device=None, nranks=None,
                 rank=None, nccl_id=None):
        view = plan.view if isinstance(plan, PreparedSimulation) else plan
        self._keep = plan
        self.n_kept = view.n_kept
        self.words = state_words(self.n_kept)
        h = C.c_void_p()
        if nranks is None:
            devs = list(range(device_count())) if devices is None else list(devices)
            arr = (C.c_int * len(devs))(*devs)
            _check(lib.pbn_group_create(C.byref(view), arr, len(devs), lanes_per_traj, C.byref(h)))
        else:
            idb = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
            _check(lib.pbn_group_create_rank(C.byref(view), device, nranks, rank, idb,
                                             lanes_per_traj, C.byref(h)))
        self._h = h
        n, r, f = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib.pbn_group_info(h, C.byref(n), C.byref(r), C.byref(f)))
        self.n_members, self.nranks, self.first_rank = n.value, r.value, f.value

    def __del__(self):
        if lib is not None and getattr(self, "_h", None) and self._h.value:
            lib.pbn_group_destroy(self._h)
            self._h = C.c_void_p(None)

    def shard(self, n_total: int, rank: int):
        b, c = C.c_uint64(), C.c_uint64()
        _check(lib.pbn_group_shard(self._h, n_total, rank, C.byref(b), C.byref(c)))
        return b.value, c.value

    def local_rows(self, n_total: int):
        """[begin, end) of the global rows this process's members own."""
        b0, _ = self.shard(n_total, self.first_rank)
        bl, cl = self.shard(n_total, self.first_rank + self.n_members - 1)
        return b0, bl + cl

    def member_kernel(self, i: int = 0) -> str:
        eng = C.c_void_p()
        _check(lib.pbn_group_member(self._h, i, C.byref(eng)))
        buf = C.create_string_buffer(256)
        _check(lib.pbn_gpu_last_kernel(eng, buf, 256, None))
        return buf.value.decode()

    def simulate(self, seed, n_traj, n_steps, traj_begin=0, step_begin=0, states=None, pred=None,
                 stream=STREAM_U53, node_counts=False):
        """The whole job of n_traj trajectories (collective over the ranks).
        states: this process's rows (local_rows) or None (zeros).
        Returns (states, per-trajectory counts, job totals (8,), job node totals or None)."""
        b, e = self.local_rows(n_traj)
        rows = e - b
        st = (np.zeros((rows, self.words), np.uint64) if states is None
              else np.ascontiguousarray(states, np.uint64).copy())
        if st.shape != (rows, self.words):
            raise UsageError(f"states must be ({rows}, {self.words}) for this process's rows")
        cnt = np.zeros((rows, COUNT_FIELDS), np.uint64)
        tot = np.zeros(COUNT_FIELDS, np.uint64)
        ntot = np.zeros(self.n_kept, np.uint64) if node_counts else None
        a = GpuEnsemble._args(self, seed, traj_begin, n_traj, n_steps, step_begin, pred, stream)
        a.flags = RUN_NODE_COUNTS if node_counts else 0
        _check(lib.pbn_group_run(self._h, C.byref(a), _u64p(st), _u64p(cnt), _u64p(tot),
                                 _u64p(ntot) if node_counts else None))
        return st, cnt, tot, ntot


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for GpuGroup(..., nranks=R, rank=r, nccl_id=id)."""
    buf = (C.c_uint8 * 128)()
    _check(lib.pbn_nccl_unique_id(buf))
    return bytes(buf)


# ----------------------------------------------------------------------------
# Pooled two-state Markov chain steady-state estimate (estimator.hpp:137-244)

def make_request(precision=1e-3, confidence=0.95, pilot=10000, burn_epsilon=0.0,
                 max_refinements=20, sample_inflation=1.3, seed=42, traj_begin=0, n_traj=1,
                 stream=STREAM_U53):
    """estimation_request (estimator.hpp:59-70) + ensemble fields."""
    return EstimateRequest(precision, confidence, pilot, burn_epsilon, max_refinements,
                           sample_inflation, seed, traj_begin, n_traj, stream)


def estimate(engine: "GpuEnsemble", pred, req: EstimateRequest, states=None):
    """Device ensemble estimate of P(predicate) under the stationary law.
    pred: (engine bits, values); states: (n_traj, words) initial states (zeros)."""
    n = req.n_traj
    st = (np.zeros((n, engine.words), np.uint64) if states is None
          else np.ascontiguousarray(states, np.uint64).copy())
    bits = np.ascontiguousarray(pred[0], np.uint32)
    vals = np.ascontiguousarray(pred[1], np.uint8)
    res = EstimateResult()
    _check(lib.pbn_estimate(engine._h, C.byref(req), _u32p(bits),
                            vals.ctypes.data_as(C.POINTER(C.c_uint8)), len(bits), _u64p(st),
                            C.byref(res)))
    return res.as_dict(), st


def estimate_with_backend(req: EstimateRequest, n_traj, run, series_stats, series_capacity):
    """The same C++ estimator over Python callbacks (tests: the oracle as stepper).
    run(step_begin, n_steps, kappa, thin_mode, series_bit0|None, series_init) -> totals[8];
    series_stats(kappa, length) -> 13 pooled counters."""

    def _run(user, s0, n, kappa, mode, bit0, init, out):
        try:
            tot = run(s0, n, kappa, mode, None if bit0 == (1 << 64) - 1 else bit0, bool(init))
            for i in range(8):
                out[i] = int(tot[i])
            return 0
        except Exception:  # noqa: BLE001  (reported as a backend failure)
            import traceback
            traceback.print_exc()
            return 1

    def _stats(user, kappa, length, out):
        try:
            v = series_stats(kappa, length)
            for i in range(13):
                out[i] = int(v[i])
            return 0
        except Exception:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1

    be = EstimatorBackend(None, n_traj, 0, series_capacity, RUN_FN(_run), STATS_FN(_stats))
    res = EstimateResult()
    _check(lib.pbn_estimate_with_backend(C.byref(req), C.byref(be), C.byref(res)))
    return res.as_dict()


def series_stats_host(series: np.ndarray, length: int, kappa: int):
    out = np.zeros(13, np.uint64)
    ser = np.ascontiguousarray(series, np.uint32)
    _check(lib.pbn_series_stats_host(_u32p(ser), ser.shape[0], ser.shape[1], length, kappa,
                                     _u64p(out)))
    return out


def stats_csv(plan: "PreparedSimulation", one_counts, steps: int) -> str:
    """The reference CLI's per-node statistics (pbn_main.cpp:75-85, 207-245):
    one row per kept node in model order, one_counts in engine order (pooled
    over trajectories if 2-D), frequency printed with %.12g."""
    oc = np.asarray(one_counts, dtype=np.uint64)
    if oc.ndim == 2:
        oc = oc.sum(axis=0, dtype=np.uint64)
    red = plan.reduced()
    rows = ["node,name,one_count,steps,frequency"]
    for v in range(red["original_n"]):
        r = int(red["index_map"][v])
        if r < 0:
            continue
        ones = int(oc[int(red["engine_pos"][r])])
        freq = 0.0 if steps == 0 else ones / steps
        rows.append(f"{v},{plan.model.node_name(v)},{ones},{steps},{freq:.12g}")
    return "\n".join(rows) + "\n"


def series_stats_device(device: int, d_series: int, n_traj: int, stride: int, length: int,
                        kappa: int):
    out = np.zeros(13, np.uint64)
    _check(lib.pbn_series_stats_device(device, C.c_void_p(d_series), n_traj, stride, length, kappa,
                                       _u64p(out)))
    return out
