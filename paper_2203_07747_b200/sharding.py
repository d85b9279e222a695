"""Instance partitioning across ranks (one process per GPU) and the one
exchange step of the path: the gather of the per-node (f, A, B) blocks to
the consumer rank.

MPC instances are independent (no cross-row coupling in the MLP), so rank g
takes the contiguous instance block [g·B/G, (g+1)·B/G) with the weights
replicated; the only collective is the final gather. The
reference has no multi-process backend at all (threads only,
proj/include/resmpc/threadpool.hpp); this module is new.

`torch.distributed` is the plumbing: NCCL on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Partition:
    rank: int
    world: int
    instances: int          # total MPC instances
    horizon: int            # shooting nodes per instance
    first_instance: int
    num_instances: int

    @property
    def first_node(self) -> int:
        return self.first_instance * self.horizon

    @property
    def num_nodes(self) -> int:
        return self.num_instances * self.horizon


def partition_instances(instances: int, horizon: int, rank: int, world: int) -> Partition:
    """Contiguous, balanced instance blocks; the first `instances % world`
    ranks take one extra instance. Node rows of an instance never straddle
    ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if instances < 0 or horizon < 1:
        raise ValueError("bad instances/horizon")
    base, extra = divmod(instances, world)
    first = rank * base + min(rank, extra)
    n = base + (1 if rank < extra else 0)
    return Partition(rank, world, instances, horizon, first, n)


def all_partitions(instances: int, horizon: int, world: int) -> list[Partition]:
    return [partition_instances(instances, horizon, r, world) for r in range(world)]


def gather_blocks(local, dst: int = 0, group=None):
    """Gathers every rank's per-node result block (a tensor whose leading dim
    is the rank's node count) to `dst`, concatenated in rank (= instance)
    order. Blocks may be ragged across ranks; they are padded to the largest
    block for the collective and trimmed afterwards. Returns the full tensor
    on `dst` and None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_local = torch.tensor([local.shape[0]], device=local.device, dtype=torch.int64)
    counts = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(counts, n_local, group=group)
    counts = [int(c.item()) for c in counts]
    n_max = max(counts)
    if local.shape[0] < n_max:
        pad = torch.zeros((n_max - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        send = torch.cat([local, pad])
    else:
        send = local.contiguous()
    if rank == dst:
        recv = [torch.empty_like(send) for _ in range(world)]
        dist.gather(send, recv, dst=dst, group=group)
        return torch.cat([r[:c] for r, c in zip(recv, counts)])
    dist.gather(send, None, dst=dst, group=group)
    return None


class Gatherer:
    """Preallocated fixed-shape gather used in the timed loop: every rank
    sends the same-sized block (balanced partitions, padded), rank `dst`
    receives into persistent buffers, so the step issues exactly one NCCL
    gather per output tensor and no allocations."""

    def __init__(self, shape_per_rank, dtype, device, dst: int = 0, group=None):
        import torch
        import torch.distributed as dist
        self.dst = dst
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.send = torch.zeros(shape_per_rank, dtype=dtype, device=device)
        self.recv = ([torch.empty(shape_per_rank, dtype=dtype, device=device) for _ in range(self.world)]
                     if self.rank == dst else None)

    def __call__(self, local):
        import torch.distributed as dist
        n = local.shape[0]
        self.send[:n].copy_(local)
        dist.gather(self.send, self.recv, dst=self.dst, group=self.group)
        return self.recv
