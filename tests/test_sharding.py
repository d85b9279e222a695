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
