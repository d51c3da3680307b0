#!/usr/bin/env python3
"""Throughput benchmark of the PBN trajectory hot path (BASELINE.json metric:
node-updates/s and trajectory-steps/s; % of the shared-memory lookup roofline).

One bench "step" = one pass of the hot path over the workload: every trajectory
of the ensemble advanced by the config's step count (c2: 4096 trajectories x
1e5 steps per GPU), continuing from the previous step's states.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--stream u53|u32]
  python bench.py --impl reference ...   # the reference's own CPU stepper, all host cores

Multi-GPU (torchrun, one rank per GPU): each rank owns a contiguous range of
global trajectory ids (weak scaling); the per-trajectory counts are combined
with ONE NCCL all-reduce at the end; time = max over ranks of device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gzip  # noqa: E402

import numpy as np  # noqa: E402

# The workload table and model texts are plain files (workloads/): the
# reference arm reads them without importing the engine package, so its
# process never maps libpbn_b200.so.
WORKLOADS_DIR = os.path.join(ROOT, "workloads")
with open(os.path.join(WORKLOADS_DIR, "workloads.json")) as _f:
    WORKLOADS = json.load(_f)


def workload_text(name, p=None):
    """Committed model text of a workload (workloads/<name>.pbn.gz), with the
    perturbation rate replaced when `p` is given (the c5 sweep): the generator
    draws the network independently of p and the serialiser prints p with
    %.12g (io.hpp:199-203), so this equals the generator's text at that p
    (tests/test_workloads.py)."""
    with gzip.open(os.path.join(WORKLOADS_DIR, f"{name}.pbn.gz"), "rt") as f:
        text = f.read()
    if p is not None:
        lines = text.split("\n")
        assert lines[1].startswith("perturbation ")
        lines[1] = f"perturbation {p:.12g}"
        text = "\n".join(lines)
    return text


# Philox4x32-10 blocks/s of a Philox-only kernel of this engine on one B200
# (tools/ceilings.cu, 416 blocks per step, 4144 warps; profiles/r02_ceilings.jsonl):
# the 32x32->64 multiplies (IMAD.WIDE, 17 per block) bound it, not issue
PHILOX_BLOCKS_PER_S = 4.797e11

METRIC = "node-updates/sec"
BACKEND = os.environ.get("PBN_BENCH_BACKEND", "nccl")
UNIT = "node-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--stream", default="u53", choices=["u53", "u32"])
    ap.add_argument("--p", type=float, default=None, help="override perturbation rate (c5 sweep)")
    ap.add_argument("--traj", type=int, default=None, help="trajectories per GPU")
    ap.add_argument("--sim-steps", type=int, default=None, help="simulation steps per bench step")
    ap.add_argument("--lpt", type=int, default=0)
    ap.add_argument("--k", type=int, default=None, help="override the plan's k_max")
    ap.add_argument("--mgp", type=int, default=None, help="override max_group_parents")
    ap.add_argument("--placement", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--method", default="grouped", choices=["grouped", "reduction", "old"],
                    help="stepper: the structure-based grouped stepper (the hot path) or the "
                         "reference's node-by-node Method_reduction / Method_old")
    ap.add_argument("--mode", default="auto", choices=["auto", "simulate", "estimate"],
                    help="c3 defaults to the steady-state estimate workload")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_workload(cfg, p_override, method="grouped", k=None, mgp=None):
    """Model text is the interchange format: both arms parse the same committed
    text (workloads/<cfg>.pbn.gz), so their plans are bitwise identical."""
    import dataclasses

    import paper_1605_00854_b200 as pb
    from paper_1605_00854_b200.configs import CONFIGS

    w = CONFIGS[cfg]
    if k is not None:
        w = dataclasses.replace(w, k_max=k)
    if mgp is not None:
        w = dataclasses.replace(w, mgp=mgp)
    text = workload_text(cfg, p_override)
    terms = [tuple(t) for t in WORKLOADS[cfg]["terms"]]
    model = pb.parse_model(text)
    if method == "grouped":
        plan = pb.prepare(model, w.theta, w.k_max, w.mgp)
    else:
        plan = pb.prepare_nodewise(model, method == "reduction")
    return w, text, model, plan, terms


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


METHOD_CODE = {"grouped": 0, "old": 1, "reduction": 2}


def ref_ensemble_sample(rplan, pred, n_traj, seconds, threads, method_code):
    """Steps per trajectory so that the reference stepper (oracle/_ref) runs the
    ensemble's n_traj trajectories in about `seconds` on `threads` threads."""
    cal = min(n_traj, 4 * threads)
    rplan.bench_ensemble(41, threads, cal, 200, pred, method_code)  # cold: threads, pages
    t, _ = rplan.bench_ensemble(42, threads, cal, 1000, pred, method_code)
    per_traj_step = max(t / 1000 * threads / cal, 1e-10)  # thread-seconds
    return max(500, int(seconds * threads / (per_traj_step * n_traj)))


def cpu_reference_rate(text, w, terms, seconds, n_traj, threads=None, method="grouped"):
    """The unmodified reference stepper (oracle/_ref, xoshiro256) — grouped,
    Method_old or Method_reduction — on the GPU arm's ensemble: all n_traj
    trajectories, a bounded number of steps each, over every host thread.
    Returns (traj-steps/s, threads, steps per trajectory, seconds, state bits)."""
    import oracle

    ref = oracle.Reference()
    rm = ref.parse(text)
    rplan = rm.prepare(w.theta, w.k_max, w.mgp)
    pred = rplan.compile_predicate(terms)
    threads = threads or os.cpu_count() or 1
    code = METHOD_CODE[method]
    steps = ref_ensemble_sample(rplan, pred, n_traj, seconds, threads, code)
    t, _ = rplan.bench_ensemble(42, threads, n_traj, steps, pred, code)
    rate = n_traj * steps / t
    n_state = {"grouped": rplan.n_kept, "reduction": rplan.n_kept}.get(method, w.n)
    return rate, threads, steps, t, n_state


def reference_estimate_arm(a, w, rplan, terms, threads):
    """c3 reference arm: the reference's own estimate_steady_state (r = 1e-3,
    conf 0.95, xoshiro256), one independent estimate per host thread."""
    from concurrent.futures import ThreadPoolExecutor

    def one(seed):
        return rplan.estimate(terms, 1e-3, 0.95, 10000, seed, -1, 0)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(9000, 9000 + threads * max(1, a.warmup // 3))))
    total, steps, est = 0.0, 0, []
    for k in range(a.steps):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            rs = list(ex.map(one, range(100 * k, 100 * k + threads)))
        total += time.perf_counter() - t0
        steps += sum(r["steps"] for r in rs)
        est.append(rs[0]["estimate"])
    val = steps * rplan.n_kept / total
    print(json.dumps({
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1000 * total / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{a.config}: {w.note}", "n": w.n, "n_kept": rplan.n_kept,
                   "precision": 1e-3, "confidence": 0.95},
        "trajectory_steps_per_s": steps / total, "estimates": est,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{threads} concurrent reference estimate_steady_state runs "
                                   f"per step (xoshiro256)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_reference_arm(a):
    """The reference's own CPU implementation of the path: the unmodified
    grouped_simulator + xoshiro256 (oracle/_ref/libpbnref.so, built from
    /root/reference's headers) on every host thread, over the same workload
    text and plan as the GPU arm — all of the ensemble's trajectories, a
    bounded number of steps each. Imports `oracle` only: the engine library is
    never loaded in this process."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    import oracle

    wd = WORKLOADS[a.config]
    p = a.p if a.p is not None else wd["p"]
    text = workload_text(a.config, a.p)
    terms = [tuple(t) for t in wd["terms"]]
    theta = wd["theta"]
    k = a.k if a.k is not None else wd["k_max"]
    mgp = a.mgp if a.mgp is not None else wd["mgp"]
    ref = oracle.Reference()
    rmodel = ref.parse(text)
    rplan = rmodel.prepare(theta, k, mgp)
    pred = rplan.compile_predicate(terms)
    threads = os.cpu_count() or 1

    class _W:  # the fields reference_estimate_arm reads
        n = wd["n"]
        note = wd["note"]

    if wd["n_steps"] == 0:
        return reference_estimate_arm(a, _W, rplan, terms, threads)
    n_traj = a.traj or wd["n_traj"]
    steps = ref_ensemble_sample(rplan, pred, n_traj, 6.0, threads, 0)  # ~6 s per bench step
    for _ in range(a.warmup):
        rplan.bench_ensemble(7, threads, n_traj, max(20, steps // 10), pred)
    times = []
    for kk in range(a.steps):
        t, _ = rplan.bench_ensemble(42 + 1000 * kk, threads, n_traj, steps, pred)
        times.append(t)
    total = sum(times)
    tsteps = n_traj * steps * a.steps
    val = tsteps * rplan.n_kept / total
    # the same ensemble at the reference's default plan (engine.hpp:81-83:
    # theta 2^25, k 16, mgp 18), a shorter sample, reported beside it
    default_plan = {"plan": {"theta": 1 << 25, "k_max": 16, "mgp": 18}}
    try:
        dplan = rmodel.prepare(1 << 25, 16, 18)
        dpred = dplan.compile_predicate(terms)
        dsteps = ref_ensemble_sample(dplan, dpred, n_traj, 3.0, threads, 0)
        dt, _ = dplan.bench_ensemble(42, threads, n_traj, dsteps, dpred)
        default_plan.update({"value": n_traj * dsteps * dplan.n_kept / dt, "unit": UNIT,
                             "trajectory_steps_per_s": n_traj * dsteps / dt,
                             "sample": f"{n_traj} trajectories x {dsteps} steps"})
    except oracle.RefError as e:  # e.g. c4: the default mgp does not plan
        default_plan["error"] = str(e)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1000 * total / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{a.config}: {wd['note']}", "n": wd["n"], "n_kept": rplan.n_kept,
                   "method": "grouped", "trajectories_per_gpu": n_traj,
                   "sim_steps_sampled_per_trajectory": steps,
                   "p": p, "plan": {"theta": theta, "k_max": k, "mgp": mgp},
                   "model": f"workloads/{a.config}.pbn.gz"},
        "trajectory_steps_per_s": tsteps / total,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"all {n_traj} trajectories x {steps} steps per bench step "
                                   f"(the GPU arm runs {wd['n_steps']}), unmodified reference "
                                   f"grouped_simulator + xoshiro256, count_nodes=false, "
                                   f"predicate on, {threads} threads"},
        "reference_default_plan": default_plan,
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_estimate_mode(a, torch, dist, rank, world, local, dev):
    """c3: pooled two-state MC steady-state estimate (r = 1e-3, conf 0.95) over
    the config's trajectories, strong-scaled across ranks (shard_range); the
    C++ estimator drives per-rank device rounds with one all-reduce of the
    pooled counters per round. One bench step = one complete estimate."""
    import paper_1605_00854_b200 as pb
    from paper_1605_00854_b200.ensemble import DeviceShard, estimate_sharded, shard_range

    w, text, model, plan, terms = build_workload(a.config, a.p, "grouped", a.k, a.mgp)
    pred = plan.compile_predicate(terms)
    n_total = a.traj or w.n_traj
    stream = pb.STREAM_U53 if a.stream == "u53" else pb.STREAM_U32
    eng = pb.GpuEnsemble(plan, device=local, lanes_per_traj=a.lpt, placement=a.placement)
    b, c = shard_range(n_total, world, rank)
    pilot = 1000
    cap = pilot + 1

    def one(seed):
        shard = DeviceShard(eng, pred, seed, b, c, stream, cap)
        req = pb.make_request(precision=1e-3, confidence=0.95, pilot=pilot, seed=seed,
                              stream=stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = estimate_sharded(req, shard, n_total, cap, device=dev)
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0, res

    for k in range(max(a.warmup, 3)):
        one(1000 + k)
    times, results = [], []
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            dt, res = one(42 + k)
            times.append(dt)
            results.append(res)
    t = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s = float(t.item())
    traj_steps = sum(r["steps_per_traj"] for r in results) * n_total
    n_kept = plan.n_kept
    value = traj_steps * n_kept / total_s
    # end to end through the public C-ABI (pbn_estimate: host states in/out) at N=1
    e2e = None
    if world == 1:
        h_states = np.zeros((n_total, eng.words), np.uint64)
        pb.estimate(eng, pred, pb.make_request(  # untimed warm-up of the C-ABI path
            precision=1e-3, confidence=0.95, pilot=pilot, seed=999, n_traj=n_total,
            stream=stream), h_states.copy())
        t0 = time.perf_counter()
        e_steps = 0
        for k in range(a.steps):
            res, _ = pb.estimate(eng, pred, pb.make_request(
                precision=1e-3, confidence=0.95, pilot=pilot, seed=42 + k, n_traj=n_total,
                stream=stream), h_states)
            e_steps += res["steps_per_traj"] * n_total
        e2e = {"value": e_steps * n_kept / (time.perf_counter() - t0), "unit": UNIT,
               "h2d_bytes_per_step": n_total * eng.words * 8,
               "d2h_bytes_per_step": n_total * eng.words * 8 + 72}
    if rank != 0:
        return
    est = [r["estimate"] for r in results]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": max(a.warmup, 3), "ms_per_step": 1000 * total_s / a.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"{a.config}: {w.note}", "n": w.n, "n_kept": n_kept,
                   "trajectories_total": n_total, "precision": 1e-3, "confidence": 0.95,
                   "pilot_per_trajectory": pilot, "stream": a.stream,
                   "plan": {"theta": w.theta, "k_max": w.k_max, "mgp": w.mgp},
                   "engine": eng.info(), "parallelism": f"trajectory-sharded x{world}",
                   "l2": "inputs (plan + states) re-staged per launch; no flush"},
        "trajectory_steps_per_s": traj_steps / total_s,
        "estimates": est, "sample_size_used": [r["sample_size_used"] for r in results],
        "e2e": e2e, "gpu_launches": None, "clocks": clk.summary(),
    }
    if not a.no_cpu_baseline and world == 1:
        import oracle

        rplan = oracle.Reference().parse(text).prepare(w.theta, w.k_max, w.mgp)
        t0 = time.perf_counter()
        r = rplan.estimate(terms, 1e-3, 0.95, 10000, 42, -1, 0)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {
            "value": r["steps"] * n_kept / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"one reference estimate_steady_state at r=1e-3 ({r['steps']} steps, "
                      f"{dt:.2f} s, estimate {r['estimate']:.6f})"}
    print(json.dumps(line), flush=True)


def run_ours(a):
    import torch

    import paper_1605_00854_b200 as pb

    rank, world, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist

        # PBN_BENCH_BACKEND=gloo (tests only): host-side collectives over gloo and
        # every rank on the visible devices round-robin — exercises the N > 1
        # code path on a one-GPU box (the device group then falls back)
        if BACKEND != "nccl":
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rdev = dev if BACKEND == "nccl" else torch.device("cpu")  # collective tensors
    if a.mode == "estimate" or (a.mode == "auto" and WORKLOADS[a.config]["n_steps"] == 0):
        run_estimate_mode(a, torch, dist if world > 1 else None, rank, world, local, dev)
        if world > 1:
            dist.destroy_process_group()
        return

    w, text, model, plan, terms = build_workload(a.config, a.p, a.method, a.k, a.mgp)
    flat = plan.flat()
    pred = plan.compile_predicate(terms)
    n_traj = a.traj or w.n_traj
    sim_steps = a.sim_steps or (w.n_steps if w.n_steps else 100_000)
    stream = pb.STREAM_U53 if a.stream == "u53" else pb.STREAM_U32
    eng = pb.GpuEnsemble(plan, device=local, lanes_per_traj=a.lpt, placement=a.placement)
    words = eng.words
    from paper_1605_00854_b200.ensemble import allreduce_totals, pooled, shard_range

    traj_begin, _ = shard_range(n_traj * world, world, rank)  # weak scaling: n_traj per GPU

    states = torch.zeros((n_traj, words), dtype=torch.int64, device=dev)
    counts = torch.zeros((n_traj, 8), dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > L2 (126 MB)
    cs = torch.cuda.current_stream(dev)
    step_pos = 0

    def one(n_steps):
        nonlocal step_pos
        eng.simulate_device(42, n_traj, n_steps, states.data_ptr(), counts.data_ptr(),
                            traj_begin=traj_begin, step_begin=step_pos, pred=pred, stream=stream,
                            cuda_stream=cs.cuda_stream)
        step_pos += n_steps

    for _ in range(max(a.warmup, 3)):
        one(max(1, sim_steps // 10))
    torch.cuda.synchronize(dev)

    fn_steps = 0
    launches = 0
    ev_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            flush.fill_(k)  # L2 flush between timed iterations (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            one(sim_steps)
            e1.record(cs)
            launches += eng.last_launches()
            e1.synchronize()
            ev_ms.append(e0.elapsed_time(e1))
            fn_steps += int(counts[:, 6].sum().item())
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    my_ms = sum(ev_ms)
    t_ms = torch.tensor([my_ms], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)  # measurement: max over ranks
    total_ms = float(t_ms.item())
    # the single collective of the path: one all-reduce of the pooled counts
    mine = pooled(counts.cpu().numpy().view(np.uint64))
    mine[6] = fn_steps  # function-phase steps over all timed launches
    totals = allreduce_totals(mine, device=rdev)
    fn_total = int(totals[6])
    traj_steps = n_traj * world * sim_steps * a.steps
    value = traj_steps * flat.n_kept / (total_ms / 1e3)

    # ---- end to end through the public C-ABI with HOST buffers (pinned),
    # host<->device copies inside the timed region (pbn_gpu_run is synchronous)
    host_states = torch.zeros((n_traj, words), dtype=torch.int64).pin_memory()
    host_counts = torch.zeros((n_traj, 8), dtype=torch.int64).pin_memory()
    import ctypes as C

    def e2e_one(n_steps, s0):
        args = eng._args(42, traj_begin, n_traj, n_steps, s0, pred, stream)
        pb._check(pb.lib.pbn_gpu_run(eng._h, C.byref(args),
                                     C.cast(host_states.data_ptr(), C.POINTER(C.c_uint64)),
                                     C.cast(host_counts.data_ptr(), C.POINTER(C.c_uint64)), None))

    grp, e2e_path = None, "pbn_gpu_run (C-ABI, host buffers)"
    if world > 1:
        # N > 1: end to end through the C-ABI device group (pbn_group_run):
        # host rows in, this rank's launch, pooling kernels, ONE ncclAllReduce
        # of the pooled counts, host rows + job totals out. If the group cannot
        # be built on every rank, every rank falls back to pbn_gpu_run (the
        # reason goes into the line) rather than failing the run.
        ok, why = 1, ""
        try:
            ids = [pb.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
            grp = pb.GpuGroup(plan, device=local, nranks=world, rank=rank, nccl_id=ids[0])
        except Exception as e:  # noqa: BLE001
            ok, why = 0, f"{type(e).__name__}: {e}"
        flag = torch.tensor([ok], dtype=torch.int32, device=rdev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            e2e_path = ("pbn_group_run (C-ABI device group: one ncclAllReduce of the pooled "
                        "counts)")
            g_states = np.zeros((n_traj, words), np.uint64)

            def e2e_one(n_steps, s0):  # noqa: F811
                nonlocal g_states
                g_states, _, _, _ = grp.simulate(42, n_traj * world, n_steps, step_begin=s0,
                                                 states=g_states, pred=pred, stream=stream)
        else:
            e2e_path += f" (device group unavailable: {why or 'on another rank'})"

    e2e_one(max(1, sim_steps // 10), 0)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(a.steps):
        e2e_one(sim_steps, k * sim_steps)
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_val = traj_steps * flat.n_kept / float(e2e_t.item())
    info = eng.info()  # the timed kernel (before the alternate-stream run below)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # the other stream kind, one timed bench step (reported beside the headline)
    alt_kind = pb.STREAM_U32 if stream == pb.STREAM_U53 else pb.STREAM_U53
    alt = None
    if world == 1:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.simulate_device(42, n_traj, max(1, sim_steps // 10), states.data_ptr(),
                            counts.data_ptr(), traj_begin=traj_begin, step_begin=0, pred=pred,
                            stream=alt_kind, cuda_stream=cs.cuda_stream)
        flush.fill_(7)
        e0.record(cs)
        eng.simulate_device(42, n_traj, sim_steps, states.data_ptr(), counts.data_ptr(),
                            traj_begin=traj_begin, step_begin=0, pred=pred, stream=alt_kind,
                            cuda_stream=cs.cuda_stream)
        e1.record(cs)
        e1.synchronize()
        alt = {"stream": "u32" if alt_kind == pb.STREAM_U32 else "u53",
               "value": n_traj * sim_steps * flat.n_kept / (e0.elapsed_time(e1) / 1e3),
               "unit": UNIT}

    peaks = measured_peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(a.config, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    props = torch.cuda.get_device_properties(dev)
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak_lookups = props.multi_processor_count * 32 * sm_mhz * 1e6
    lookups = flat.expected_lookups(fn_total, traj_steps)
    achieved = lookups / (total_ms / 1e3) / world
    # Ceiling the injected stream imposes: a kernel doing
    # nothing but generating the workload's Philox4x32-10 blocks, at the
    # measured Philox-only rate of a B200.
    dpb = 4  # both streams: 4 high words per Philox block (U53 low words only on ties)
    n_alias = int(np.count_nonzero(flat.grp_alias_size))
    has_leaf = 1 if a.method != "old" else 0
    blocks = (-(-(flat.pert_groups + has_leaf) // dpb)) * traj_steps + (-(-n_alias // dpb)) * fn_total
    # measured: the engine's own Philox4x32-10 issues at most this many blocks
    # per second on a B200 (tools/ceilings.cu, profiles/r02_ceilings.jsonl)
    philox_peak_blocks = PHILOX_BLOCKS_PER_S
    rng_ceiling_steps = philox_peak_blocks / (blocks / traj_steps)
    rng_ceiling = rng_ceiling_steps * lookups / traj_steps
    spill = None
    if info["placement"] == "global":
        # spill case: the plan is read through L1/L2. The lookup
        # roofline stays the headline; the memory view is reported beside it
        # (if every probe were a 32-B sector from HBM) — L1 serves ~92% of them
        # (profiles/r01_c4_u53.txt), so this is an upper bound on memory demand.
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        spill = {"bound": "hbm", "algorithmic_gbs_if_every_probe_were_a_sector":
                 achieved * 32 / 1e9, "peak_gbs": hbm,
                 "measured": "ncu: L1 hit 92%, L2 hit 99.9%, 459 GB/s L2->SM (profiles/r01_c4_u53.txt)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": max(a.warmup, 3), "ms_per_step": total_ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{a.config}: {w.note}", "n": w.n, "n_kept": flat.n_kept,
                   "method": a.method,
                   "trajectories_per_gpu": n_traj, "sim_steps_per_bench_step": sim_steps,
                   "p": a.p if a.p is not None else w.p,
                   "plan": {"theta": w.theta, "k_max": w.k_max, "mgp": w.mgp},
                   "stream": a.stream, "engine": info,
                   "l2": "flushed between timed iterations (256 MiB write)",
                   "parallelism": f"trajectory-sharded x{world}"},
        "trajectory_steps_per_s": traj_steps / (total_ms / 1e3),
        "node_updates_per_s_original_n": traj_steps * w.n / (total_ms / 1e3),
        "fn_phase_fraction": fn_total / traj_steps,
        "e2e": {"value": e2e_val, "unit": UNIT,
                "path": e2e_path,
                "h2d_bytes_per_step": n_traj * words * 8,
                "d2h_bytes_per_step": n_traj * words * 8 + n_traj * 8 * 8},
        "gpu_launches": launches,
        "alt_stream": alt,
        "spill_view": spill,
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak_lookups,
                     "unit": "lookups/s", "frac": achieved / peak_lookups, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu, profiles/traffic.json)",
                     "issue_bound_evidence": "profiles/r02_c2_u53.txt: issue slots ~72% "
                                             "busy, ALU pipe ~71%, smem wavefronts ~57% of peak",
                     "note": "lookup roofline = SMs x 32 probes/clk x sm_max_mhz "
                             "(MEASURED_PEAKS.json); algorithmic lookups = g per step + "
                             "(A+G) per function-phase step (SURVEY 8d), per GPU",
                     "lookups_per_step": lookups / traj_steps,
                     "rng_ceiling_frac": rng_ceiling / peak_lookups,
                     "frac_of_rng_ceiling": achieved / rng_ceiling,
                     "rng_ceiling_note": "lookup rate of a kernel generating only the workload's "
                                         "Philox4x32-10 blocks at the measured Philox-only rate "
                                         "of a B200 (profiles/r02_ceilings.jsonl); DESIGN.md §7"},
        "clocks": clk.summary(),
    }
    if not a.no_cpu_baseline and world == 1:
        try:
            rate, threads, steps, secs, nk = cpu_reference_rate(text, w, terms, a.cpu_seconds,
                                                                n_traj, method=a.method)
            line["cpu_baseline"] = {
                "value": rate * nk, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"all {n_traj} trajectories x {steps} steps ({secs:.1f} s) on {threads} "
                          f"threads, unmodified reference {a.method} stepper + xoshiro256 "
                          f"(oracle/_ref)",
                "trajectory_steps_per_s": rate}
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def launch_ranks(a):
    """`--gpus N` without a torchrun environment: re-launch this command as N
    ranks (one process per GPU) through torch.distributed.run, the way the
    driver launches it. Under torchrun, WORLD_SIZE must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != a.gpus:
            sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {a.gpus}")
        return False
    if a.gpus <= 1:
        return False
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)  # rank 0 alone (other ranks exit without work)
    else:
        launch_ranks(a)
        run_ours(a)


if __name__ == "__main__":
    main()
