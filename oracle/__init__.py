"""oracle — TEST INFRASTRUCTURE ONLY (the checker, never the product).

Python bindings of
  * ``oracle/liboracle.so``      — plain-C restatement of the grouped stepper
    (pbn_oracle.c, citing engine.hpp:255-384 line by line), and
  * ``oracle/_ref/libpbnref.so`` — the UNMODIFIED reference library compiled
    from /root/reference/proj/include by oracle/Makefile (ref_driver.cpp),
    running pbn::grouped_simulator through pbn::simulate on the injected
    Philox stream, plus its CPU baseline (xoshiro256, std::thread fan-out).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libpbnref.so")


class PlanView(C.Structure):
    """Same layout as pbn_plan_view (include/pbn_b200.h)."""

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


def _u32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _as_view(view):
    """Accept any ctypes structure with the pbn_plan_view layout."""
    return C.cast(C.pointer(view), C.POINTER(PlanView))


# ---------------------------------------------------------------------------
class Oracle:
    """The plain-C restatement (liboracle.so)."""

    def __init__(self, path=ORACLE_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_simulate.restype = C.c_int
        L.orc_simulate.argtypes = [C.POINTER(PlanView), C.c_uint64, C.c_uint64, C.c_uint32, C.c_int,
                                   C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32),
                                   C.POINTER(C.c_uint8), C.c_uint32, C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.orc_simulate_ex.restype = C.c_int
        L.orc_simulate_ex.argtypes = L.orc_simulate.argtypes + [
            C.c_uint32, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.c_uint64,
            C.c_uint64, C.c_int]
        L.orc_step_scripted.restype = C.c_int
        L.orc_step_scripted.argtypes = [C.POINTER(PlanView), C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_double), C.c_uint32, C.POINTER(C.c_uint32)]
        L.orc_philox_block.restype = None
        L.orc_philox_block.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint32)]
        L.orc_draw.restype = C.c_double
        L.orc_draw.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.c_uint32]

    def simulate(self, view, seed, traj_begin, n_traj, n_steps, states=None, step_begin=0,
                 pred=None, stream=0, node_counts=False):
        words = view.n_kept // 64 + 1
        st = (np.zeros((n_traj, words), np.uint64) if states is None
              else np.ascontiguousarray(states, np.uint64).copy())
        counts = np.zeros((n_traj, 8), np.uint64)
        nc = np.zeros((n_traj, view.n_kept), np.uint64) if node_counts else None
        bits = np.zeros(1, np.uint32) if pred is None else np.ascontiguousarray(pred[0], np.uint32)
        vals = np.zeros(1, np.uint8) if pred is None else np.ascontiguousarray(pred[1], np.uint8)
        npred = 0 if pred is None else len(pred[0])
        rc = self.lib.orc_simulate(_as_view(view), seed, traj_begin, n_traj, stream, step_begin,
                                   n_steps, _u32p(bits), _u8p(vals), npred, _u64p(st),
                                   _u64p(counts), _u64p(nc) if nc is not None else None)
        assert rc == 0
        return (st, counts, nc) if node_counts else (st, counts)

    def simulate_ex(self, view, seed, traj_begin, n_traj, n_steps, states=None, step_begin=0,
                    pred=None, stream=0, kappa=1, thin_mode=0, tprev=None, series=None,
                    series_bit0=0, series_init=False):
        """orc_simulate_ex: sampled transitions (kappa/thin_mode/tprev) and an
        optional predicate series (updated in place)."""
        words = view.n_kept // 64 + 1
        st = (np.zeros((n_traj, words), np.uint64) if states is None
              else np.ascontiguousarray(states, np.uint64).copy())
        counts = np.zeros((n_traj, 8), np.uint64)
        bits = np.zeros(1, np.uint32) if pred is None else np.ascontiguousarray(pred[0], np.uint32)
        vals = np.zeros(1, np.uint8) if pred is None else np.ascontiguousarray(pred[1], np.uint8)
        npred = 0 if pred is None else len(pred[0])
        rc = self.lib.orc_simulate_ex(
            _as_view(view), seed, traj_begin, n_traj, stream, step_begin, n_steps, _u32p(bits),
            _u8p(vals), npred, _u64p(st), _u64p(counts), None, kappa, thin_mode,
            _u8p(tprev) if tprev is not None else None,
            _u32p(series) if series is not None else None,
            series.shape[1] if series is not None else 0, series_bit0, 1 if series_init else 0)
        assert rc == 0
        return st, counts

    def step_scripted(self, view, state_words, uniforms):
        st = np.ascontiguousarray(state_words, np.uint64).copy()
        u = np.ascontiguousarray(uniforms, np.float64)
        used = C.c_uint32()
        rc = self.lib.orc_step_scripted(_as_view(view), _u64p(st), _dp(u), len(u), C.byref(used))
        assert rc == 0
        return st, used.value

    def philox(self, ctr, key):
        c = np.ascontiguousarray(ctr, np.uint32)
        k = np.ascontiguousarray(key, np.uint32)
        out = np.zeros(4, np.uint32)
        self.lib.orc_philox_block(_u32p(c), _u32p(k), _u32p(out))
        return out

    def draw(self, seed, traj, step, d, stream=0, g=0):
        return self.lib.orc_draw(seed, traj, step, d, stream, g)


# ---------------------------------------------------------------------------
class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Reference:
    """The unmodified reference library (oracle/_ref/libpbnref.so)."""

    def __init__(self, path=REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        P, U32, U64, I, D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
        PU32, PU64, PU8, PD = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint8), C.POINTER(C.c_double))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_model_parse": (I, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
            "ref_model_free": (None, [P]),
            "ref_model_serialize": (I, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
            "ref_generate_random": (I, [U32, D, D, U32, U32, U64, D, C.POINTER(P)]),
            "ref_prepare": (I, [P, U64, U32, U32, C.POINTER(P)]),
            "ref_plan_free": (None, [P]),
            "ref_plan_view": (I, [P, C.POINTER(PlanView)]),
            "ref_plan_reduced": (I, [P, PU32, PU32, C.POINTER(C.c_int32), PU32, PU32]),
            "ref_plan_groups": (I, [P, PU32, PU32]),
            "ref_compile_predicate": (I, [P, PU32, PU8, U32, PU32]),
            "ref_simulate_philox": (I, [P, U64, U64, U32, I, U64, U64, PU32, PU8, U32, PU64,
                                        PU64, PU64]),
            "ref_step_scripted": (I, [P, PU64, PD, U32, PU32]),
            "ref_simulate_nodewise": (I, [P, I, U64, U64, U32, I, U64, U64, PU32, PU8, U32, PU64,
                                          PU64, PU64]),
            "ref_bench_xoshiro": (I, [P, U64, U32, U64, PU32, PU8, U32, I, P, PD, PU64]),
            "ref_bench_ensemble": (I, [P, U64, U32, U32, U64, PU32, PU8, U32, I, P, PD, PU64]),
            "ref_estimate": (I, [P, PU32, PU8, U32, D, D, U64, U64, I, U32, PD, PU64, PU64,
                                 C.POINTER(C.c_int)]),
            "ref_exact_matrix": (I, [P, D, PD]),
            "ref_grouped_row": (I, [P, U64, PD]),
            "ref_marginal_exact": (I, [P, PU32, PU8, U32, PD]),
            "ref_random_small_model": (I, [U64, U32, D, U32, U32, C.POINTER(P)]),
            "ref_alias_build": (I, [PD, U32, PD, PU32]),
            "ref_inverse_normal_cdf": (D, [D]),
            "ref_last_estimate_steps": (U64, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args

    def _ck(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode(errors="replace"))

    # models
    def parse(self, text):
        h = C.c_void_p()
        raw = text.encode()
        self._ck(self.lib.ref_model_parse(raw, len(raw), C.byref(h)))
        return RefModel(self, h)

    def generate(self, n, density, leaf_pct, max_f, max_p, seed, p):
        h = C.c_void_p()
        self._ck(self.lib.ref_generate_random(n, density, leaf_pct, max_f, max_p, seed, p,
                                              C.byref(h)))
        return RefModel(self, h)

    def random_small_model(self, seed, n, p, max_f=3, max_p=3):
        h = C.c_void_p()
        self._ck(self.lib.ref_random_small_model(seed, n, p, max_f, max_p, C.byref(h)))
        return RefModel(self, h)

    def alias_build(self, probs):
        pr = np.ascontiguousarray(probs, np.float64)
        cut = np.zeros(len(pr), np.float64)
        al = np.zeros(len(pr), np.uint32)
        self._ck(self.lib.ref_alias_build(_dp(pr), len(pr), _dp(cut), _u32p(al)))
        return cut, al


class RefModel:
    def __init__(self, ref, h):
        self.ref, self._h = ref, h

    def __del__(self):
        if self._h and self._h.value:
            self.ref.lib.ref_model_free(self._h)
            self._h = C.c_void_p(None)

    def serialize(self):
        n = C.c_size_t()
        self.ref._ck(self.ref.lib.ref_model_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.ref._ck(self.ref.lib.ref_model_serialize(self._h, buf, n.value + 1, C.byref(n)))
        return buf.raw[: n.value].decode()

    def prepare(self, theta=1 << 25, k_max=16, mgp=18):
        h = C.c_void_p()
        self.ref._ck(self.ref.lib.ref_prepare(self._h, theta, k_max, mgp, C.byref(h)))
        return RefPlan(self.ref, h, self)

    def simulate_nodewise(self, reduced, n_state, seed, traj_begin, n_traj, n_steps,
                          states=None, step_begin=0, pred=None, stream=0, node_counts=False):
        """Method_old (reduced=0) / Method_reduction (1) through pbn::simulate;
        counts carry steps and hits only."""
        words = n_state // 64 + 1
        st = (np.zeros((n_traj, words), np.uint64) if states is None
              else np.ascontiguousarray(states, np.uint64).copy())
        counts = np.zeros((n_traj, 8), np.uint64)
        nc = np.zeros((n_traj, n_state), np.uint64) if node_counts else None
        bits = np.zeros(1, np.uint32) if pred is None else np.ascontiguousarray(pred[0], np.uint32)
        vals = np.zeros(1, np.uint8) if pred is None else np.ascontiguousarray(pred[1], np.uint8)
        npred = 0 if pred is None else len(pred[0])
        self.ref._ck(self.ref.lib.ref_simulate_nodewise(
            self._h, reduced, seed, traj_begin, n_traj, stream, step_begin, n_steps, _u32p(bits),
            _u8p(vals), npred, _u64p(st), _u64p(counts), _u64p(nc) if nc is not None else None))
        return (st, counts, nc) if node_counts else (st, counts)

    def exact_matrix(self, n, t=1.0):
        out = np.zeros((1 << n) * (1 << n), np.float64)
        self.ref._ck(self.ref.lib.ref_exact_matrix(self._h, t, _dp(out)))
        return out.reshape(1 << n, 1 << n)

    def marginal_exact(self, terms):
        nodes = np.array([t[0] for t in terms], np.uint32)
        vals = np.array([t[1] for t in terms], np.uint8)
        out = C.c_double()
        self.ref._ck(self.ref.lib.ref_marginal_exact(self._h, _u32p(nodes), _u8p(vals),
                                                     len(terms), C.byref(out)))
        return out.value


class RefPlan:
    def __init__(self, ref, h, model):
        self.ref, self._h, self.model = ref, h, model
        self.view = PlanView()
        self.ref._ck(self.ref.lib.ref_plan_view(self._h, C.byref(self.view)))

    def __del__(self):
        if self._h and self._h.value:
            self.ref.lib.ref_plan_free(self._h)
            self._h = C.c_void_p(None)

    @property
    def n_kept(self):
        return self.view.n_kept

    def reduced(self, original_n):
        on, nr = C.c_uint32(), C.c_uint32()
        self.ref._ck(self.ref.lib.ref_plan_reduced(self._h, C.byref(on), C.byref(nr), None, None,
                                                   None))
        imap = np.zeros(original_n, np.int32)
        epos = np.zeros(self.n_kept, np.uint32)
        rem = np.zeros(max(1, nr.value), np.uint32)
        self.ref._ck(self.ref.lib.ref_plan_reduced(self._h, None, None,
                                                   imap.ctypes.data_as(C.POINTER(C.c_int32)),
                                                   _u32p(epos), _u32p(rem)))
        return {"original_n": on.value, "removed": rem[: nr.value], "index_map": imap,
                "engine_pos": epos}

    def groups(self):
        cum = np.zeros(self.view.n_groups + 1, np.uint32)
        mem = np.zeros(self.n_kept, np.uint32)
        self.ref._ck(self.ref.lib.ref_plan_groups(self._h, _u32p(mem), _u32p(cum)))
        return mem, cum

    def compile_predicate(self, terms):
        nodes = np.array([t[0] for t in terms], np.uint32)
        vals = np.array([1 if t[1] else 0 for t in terms], np.uint8)
        bits = np.zeros(len(terms), np.uint32)
        self.ref._ck(self.ref.lib.ref_compile_predicate(self._h, _u32p(nodes), _u8p(vals),
                                                        len(terms), _u32p(bits)))
        return bits, vals

    def simulate_philox(self, seed, traj_begin, n_traj, n_steps, states=None, step_begin=0,
                        pred=None, stream=0, node_counts=False):
        words = self.n_kept // 64 + 1
        st = (np.zeros((n_traj, words), np.uint64) if states is None
              else np.ascontiguousarray(states, np.uint64).copy())
        counts = np.zeros((n_traj, 8), np.uint64)
        nc = np.zeros((n_traj, self.n_kept), np.uint64) if node_counts else None
        bits = np.zeros(1, np.uint32) if pred is None else np.ascontiguousarray(pred[0], np.uint32)
        vals = np.zeros(1, np.uint8) if pred is None else np.ascontiguousarray(pred[1], np.uint8)
        npred = 0 if pred is None else len(pred[0])
        self.ref._ck(self.ref.lib.ref_simulate_philox(
            self._h, seed, traj_begin, n_traj, stream, step_begin, n_steps, _u32p(bits),
            _u8p(vals), npred, _u64p(st), _u64p(counts), _u64p(nc) if nc is not None else None))
        return (st, counts, nc) if node_counts else (st, counts)

    def step_scripted(self, state_words, uniforms):
        st = np.ascontiguousarray(state_words, np.uint64).copy()
        u = np.ascontiguousarray(uniforms, np.float64)
        used = C.c_uint32()
        self.ref._ck(self.ref.lib.ref_step_scripted(self._h, _u64p(st), _dp(u), len(u),
                                                    C.byref(used)))
        return st, used.value

    def bench_xoshiro(self, seed, n_threads, steps_per_thread, pred=None, method=0):
        """CPU baseline: reference grouped stepper (method 0) or Method_old (1)."""
        bits = np.zeros(1, np.uint32) if pred is None else np.ascontiguousarray(pred[0], np.uint32)
        vals = np.zeros(1, np.uint8) if pred is None else np.ascontiguousarray(pred[1], np.uint8)
        npred = 0 if pred is None else len(pred[0])
        secs = C.c_double()
        hits = C.c_uint64()
        self.ref._ck(self.ref.lib.ref_bench_xoshiro(self._h, seed, n_threads, steps_per_thread,
                                                    _u32p(bits), _u8p(vals), npred, method,
                                                    self.model._h, C.byref(secs), C.byref(hits)))
        return secs.value, hits.value

    def bench_ensemble(self, seed, n_threads, n_traj, steps, pred=None, method=0):
        """CPU baseline on an ensemble: n_traj trajectories x steps, dealt to
        n_threads threads (reference stepper + xoshiro256 seeded seed + id)."""
        bits = np.zeros(1, np.uint32) if pred is None else np.ascontiguousarray(pred[0], np.uint32)
        vals = np.zeros(1, np.uint8) if pred is None else np.ascontiguousarray(pred[1], np.uint8)
        npred = 0 if pred is None else len(pred[0])
        secs = C.c_double()
        hits = C.c_uint64()
        self.ref._ck(self.ref.lib.ref_bench_ensemble(self._h, seed, n_threads, n_traj, steps,
                                                     _u32p(bits), _u8p(vals), npred, method,
                                                     self.model._h, C.byref(secs),
                                                     C.byref(hits)))
        return secs.value, hits.value

    def grouped_row(self, e):
        out = np.zeros(1 << self.n_kept, np.float64)
        self.ref._ck(self.ref.lib.ref_grouped_row(self._h, e, _dp(out)))
        return out

    def estimate(self, terms, precision, confidence=0.95, pilot=10000, seed=1, stream=-1, traj=0):
        nodes = np.array([t[0] for t in terms], np.uint32)
        vals = np.array([t[1] for t in terms], np.uint8)
        est, burn = C.c_double(), C.c_uint64()
        n = C.c_uint64()
        deg = C.c_int()
        self.ref._ck(self.ref.lib.ref_estimate(self._h, _u32p(nodes), _u8p(vals), len(terms),
                                               precision, confidence, pilot, seed, stream, traj,
                                               C.byref(est), C.byref(n), C.byref(burn),
                                               C.byref(deg)))
        return {"estimate": est.value, "sample_size": n.value, "burn_in": burn.value,
                "degenerate": bool(deg.value), "steps": int(self.ref.lib.ref_last_estimate_steps())}


def available():
    return os.path.exists(ORACLE_SO), os.path.exists(REF_SO)
