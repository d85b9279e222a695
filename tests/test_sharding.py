"""Multi-rank path on CPU: instance partitioning and the (f, A, B) gather with
torch.distributed over gloo (world_size 2), the same code NCCL runs on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_07747_b200.sharding import all_partitions, gather_blocks, partition_instances


def test_partition_covers_every_instance_once():
    for inst, world in ((65536, 1), (65536, 2), (65536, 8), (7, 3), (3, 4)):
        parts = all_partitions(inst, 50, world)
        assert sum(p.num_instances for p in parts) == inst
        nxt = 0
        for p in parts:
            assert p.first_instance == nxt
            nxt += p.num_instances
            assert p.num_nodes == p.num_instances * 50
        sizes = [p.num_instances for p in parts]
        assert max(sizes) - min(sizes) <= 1


def test_partition_rejects_bad_args():
    with pytest.raises(ValueError):
        partition_instances(10, 50, 2, 2)
    with pytest.raises(ValueError):
        partition_instances(10, 0, 0, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, instances, horizon, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    part = partition_instances(instances, horizon, rank, world)
    z_all = oracle.quad_nodes(2203, instances * horizon)
    om = oracle.OracleModel.random_net([17, 16, 16, 6], "silu", 3, True)
    z = z_all[part.first_node:part.first_node + part.num_nodes]
    f, j, _ = om.batched_eval(z, 1, threads=1)
    ft = gather_blocks(torch.from_numpy(f))
    jt = gather_blocks(torch.from_numpy(j))
    if rank == 0:
        fr, jr, _ = om.batched_eval(z_all, 1, threads=1)
        out.put((bool(torch.equal(ft, torch.from_numpy(fr))), bool(torch.equal(jt, torch.from_numpy(jr)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("instances", [6, 7])
def test_gloo_gather_reassembles_rank_blocks(instances, oracle_lib):
    """Ragged (7 instances over 2 ranks) and even partitions: the gathered
    blocks equal the single-process evaluation of all nodes, in order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, instances, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    ok_f, ok_j = q.get(timeout=10)
    assert ok_f and ok_j


def _step_worker(rank, world, port, instances, horizon, chunks, out):
    """bench.py's multi-rank step on CPU: the rank's node rows are computed in
    row chunks straight into the Gatherers' send buffers and each chunk's gather
    is issued asynchronously before the next chunk is computed
    (sharding.partitioned_step, the code bench.run_ours times under torchrun)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2203_07747_b200.sharding import Gatherer, all_partitions, partitioned_step
    parts = all_partitions(instances, horizon, world)
    part = parts[rank]
    counts = [p.num_nodes for p in parts]
    z_all = oracle.quad_nodes(2203, instances * horizon)
    om = oracle.OracleModel.random_net([17, 16, 16, 6], "silu", 3, True)
    z = z_all[part.first_node:part.first_node + part.num_nodes]
    gf = Gatherer(counts, (6,), torch.float64, "cpu")
    gj = Gatherer(counts, (6, 17), torch.float64, "cpu")
    calls = []

    def compute(lo, hi):
        calls.append((lo, hi))
        f, j, _ = om.batched_eval(z[lo:hi], 1, threads=1)
        gf.send[lo:hi] = torch.from_numpy(f)
        gj.send[lo:hi] = torch.from_numpy(j)

    for _ in range(2):  # a second step reuses the persistent buffers
        partitioned_step(compute, [gf, gj], part.num_nodes, chunks)
    pad_zero = bool((gf.send[part.num_nodes:] == 0).all()) and bool((gj.send[part.num_nodes:] == 0).all())
    covered = sorted(calls[: len(calls) // 2]) == [c for c in sorted(calls[: len(calls) // 2])]
    if rank == 0:
        ft = torch.cat(gf.result())
        jt = torch.cat(gj.result())
        fr, jr, _ = om.batched_eval(z_all, 1, threads=1)
        out.put((bool(torch.equal(ft, torch.from_numpy(fr))), bool(torch.equal(jt, torch.from_numpy(jr))), pad_zero,
                 covered, [tuple(c) for c in calls[: len(calls) // 2]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("instances,chunks", [(7, 3), (6, 1), (9, 8)])
def test_gloo_chunked_partitioned_step(instances, chunks, oracle_lib):
    """Ragged partitions (7 or 9 instances over 2 ranks), chunked gathers
    overlapping compute: rank 0 reassembles exactly the single-process result;
    each rank computes only its own rows, in chunk order; padding rows stay zero."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port, instances, 5, chunks, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    ok_f, ok_j, pad_zero, covered, calls = q.get(timeout=10)
    assert ok_f and ok_j and pad_zero and covered
    n0 = partition_instances(instances, 5, 0, 2).num_nodes
    assert calls[0][0] == 0 and calls[-1][1] == n0  # rank 0 computed exactly its rows, in order
    assert all(a[1] == b[0] for a, b in zip(calls, calls[1:]))


def test_chunk_bounds_cover_rows():
    from paper_2203_07747_b200.sharding import chunk_bounds
    for rows, chunks in ((10, 3), (10, 1), (3, 8), (0, 4), (16384, 8)):
        b = chunk_bounds(rows, chunks)
        assert sum(h - l for l, h in b) == rows
        assert all(a[1] == c[0] for a, c in zip(b, b[1:]))
