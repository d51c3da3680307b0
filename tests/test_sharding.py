"""N>1 host path on CPU: world_size-2 gloo ranks shard the global trajectory
ids, each rank steps its range (the oracle stands in for the device here),
and one all-reduce of the pooled counts gives exactly the single-process
totals (trajectory-keyed stream => results independent of the rank count)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1605_00854_b200.ensemble import pooled, run_sharded, run_sharded_nodes, shard_range


def test_shard_ranges_partition_ids():
    for n in [0, 1, 7, 4096, 65537]:
        for world in [1, 2, 3, 8]:
            ranges = [shard_range(n, world, r) for r in range(world)]
            assert sum(c for _, c in ranges) == n
            pos = 0
            for b, c in ranges:
                assert b == pos
                pos += c


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    import oracle
    import paper_1605_00854_b200 as pb

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, terms = pb.generate_model(96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607)
    plan = pb.prepare(model, 1 << 25, 12, 8)
    pred = plan.compile_predicate(terms)
    orc = oracle.Oracle()
    tot = run_sharded(lambda b, c: orc.simulate(plan.view, 42, b, c, 300, pred=pred)[1],
                      37, world, rank)
    out_q.put((rank, tot.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_totals_equal_single_process():
    import oracle
    import paper_1605_00854_b200 as pb

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    model, terms = pb.generate_model(96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607)
    plan = pb.prepare(model, 1 << 25, 12, 8)
    pred = plan.compile_predicate(terms)
    _, cnt = oracle.Oracle().simulate(plan.view, 42, 0, 37, 300, pred=pred)
    want = pooled(cnt).tolist()
    assert res[0] == want and res[1] == want


def _est_worker(rank, world, port, out_q):
    import sys

    import torch.distributed as dist

    import oracle
    import paper_1605_00854_b200 as pb
    from paper_1605_00854_b200.ensemble import estimate_sharded

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from estimator_support import OracleEnsemble

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, terms = pb.generate_model(96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607)
    plan = pb.prepare(model, 1 << 25, 12, 8)
    pred = plan.compile_predicate(terms)
    b, c = shard_range(40, world, rank)
    shard = OracleEnsemble(oracle.Oracle(), plan.view, pred, 3, c, traj_begin=b, cap=4096)

    class Local:
        def run(self, *a):
            return shard.run(*a).astype(np.int64)

        def stats(self, kappa, length):
            return shard.stats(kappa, length)

    res = estimate_sharded(pb.make_request(precision=0.02, pilot=300, seed=3), Local(), 40, 4096)
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_estimate_equals_single_process():
    import oracle
    import paper_1605_00854_b200 as pb
    from estimator_support import OracleEnsemble

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_est_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    model, terms = pb.generate_model(96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607)
    plan = pb.prepare(model, 1 << 25, 12, 8)
    pred = plan.compile_predicate(terms)
    single = OracleEnsemble(oracle.Oracle(), plan.view, pred, 3, 40, cap=4096).estimate(
        pb.make_request(precision=0.02, pilot=300, seed=3, n_traj=40))
    for k in ("estimate", "sample_size_used", "burn_in_used", "kappa", "steps_per_traj"):
        assert res[0][k] == res[1][k] == single[k], k


def _nodes_worker(rank, world, port, out_q):
    import torch.distributed as dist

    import oracle
    import paper_1605_00854_b200 as pb

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, terms = pb.generate_model(96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607)
    plan = pb.prepare(model, 1 << 25, 16, 8)
    pred = plan.compile_predicate(terms)
    orc = oracle.Oracle()

    def sim(b, c):
        _, cnt, nc = orc.simulate(plan.view, 42, b, c, 250, pred=pred, node_counts=True)
        return cnt, nc

    tot, nodes = run_sharded_nodes(sim, 29, plan.n_kept, world, rank)
    out_q.put((rank, (tot.tolist(), nodes.tolist())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_node_counts_equal_single_process():
    """Per-node one-counts (engine.hpp:378-379) pooled over ranks with the
    same single all-reduce as the counts (concatenated vector)."""
    import oracle
    import paper_1605_00854_b200 as pb

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nodes_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    model, terms = pb.generate_model(96, (1, 2), (2, 5), 0.001, 0.3, 2, False, 1607)
    plan = pb.prepare(model, 1 << 25, 16, 8)
    pred = plan.compile_predicate(terms)
    _, cnt, nc = oracle.Oracle().simulate(plan.view, 42, 0, 29, 250, pred=pred, node_counts=True)
    want = (pooled(cnt).tolist(), nc.sum(axis=0, dtype=np.uint64).astype(np.int64).tolist())
    assert res[0] == want and res[1] == want
    assert sum(want[1]) > 0
