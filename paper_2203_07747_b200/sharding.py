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
    """Preallocated fixed-shape gather of one per-node output tensor, used in the
    timed loop: every rank sends the same `rows_max` rows (balanced partitions
    differ by at most one instance; the tail is zero padding), rank `dst`
    receives into persistent per-rank buffers. The kernel writes its rows
    straight into `send` (no copy in the step), and the gather can be issued
    in row chunks [lo, hi) so chunk i's transfer overlaps chunk i+1's compute
    (SURVEY §8e). `counts[r]` are the valid rows of rank r; `result()` trims."""

    def __init__(self, counts, row_shape, dtype, device, dst: int = 0, group=None):
        import torch
        import torch.distributed as dist
        self.dst = dst
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if len(counts) != self.world:
            raise ValueError("one row count per rank")
        self.counts = [int(c) for c in counts]
        self.rows_max = max(self.counts)
        shape = (self.rows_max,) + tuple(row_shape)
        self.send = torch.zeros(shape, dtype=dtype, device=device)  # tail rows stay zero
        self.recv = ([torch.empty(shape, dtype=dtype, device=device) for _ in range(self.world)]
                     if self.rank == dst else None)

    @property
    def local(self):
        """This rank's valid rows of the send buffer (the kernel's output)."""
        return self.send[:self.counts[self.rank]]

    def start(self, lo: int, hi: int):
        """Asynchronous gather of rows [lo, hi) of every rank's block."""
        import torch.distributed as dist
        recv = [r[lo:hi] for r in self.recv] if self.recv is not None else None
        return dist.gather(self.send[lo:hi], recv, dst=self.dst, group=self.group, async_op=True)

    def __call__(self, local=None):
        """Whole-block gather (optionally copying `local` into the send rows
        first); returns the trimmed per-rank blocks on dst, None elsewhere."""
        if local is not None:
            n = local.shape[0]
            self.send[:n].copy_(local)
            self.send[n:].zero_()
        self.start(0, self.rows_max).wait()
        return self.result()

    def result(self):
        if self.recv is None:
            return None
        return [r[:c] for r, c in zip(self.recv, self.counts)]


def chunk_bounds(rows: int, chunks: int) -> list[tuple[int, int]]:
    """[lo, hi) row ranges of `chunks` near-equal pieces of `rows` (empty pieces dropped)."""
    if rows <= 0:
        return []
    chunks = max(1, min(int(chunks), rows))
    per = -(-rows // chunks)
    return [(lo, min(rows, lo + per)) for lo in range(0, rows, per)]


def partitioned_step(compute, gatherers, n_local: int, chunks: int = 1):
    """One instance-partitioned step (the body bench.py times under torchrun):
    for every row chunk [lo, hi) of the common padded block, `compute(lo, hi)`
    enqueues this rank's rows [lo, min(hi, n_local)) into the gatherers' send
    buffers, then the chunk's gathers are issued asynchronously so they overlap
    the next chunk's compute. Every rank issues the same gathers (same padded
    shapes), including chunks past its own rows. Waits on all gathers (on GPUs:
    the current stream waits for NCCL; the host does not block)."""
    rows_max = gatherers[0].rows_max
    works = []
    for lo, hi in chunk_bounds(rows_max, chunks):  # identical on every rank (common rows_max)
        if lo < n_local:
            compute(lo, min(hi, n_local))
        for g in gatherers:
            works.append(g.start(lo, hi))
    for w in works:
        w.wait()
