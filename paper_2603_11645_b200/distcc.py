"""Edge-partitioned connectivity across GPUs (config 5, Kron-28).

Rank r of k owns the edges whose smaller endpoint lies in
[r*n/k, (r+1)*n/k). Because the normalized edge list is sorted by that
endpoint, the rank's edges are ONE contiguous range of the global list:
global edge id = e_base + local index, with e_base = the edge counts of the
lower ranks (one all-gather). The hook keys (winner << 32 | global edge id)
are therefore the single-GPU keys, and the result is bit-identical to the
1-GPU run (cc_spanning_forest, cc_forest.cpp:73-102).

Per round (mode alternates min/max, starting with min):
  hook      local edge pass into the replicated slot[n] (int64, INT64_MAX empty)
  exchange  all_reduce(slot, MIN) over NCCL -- exactly combine_min
            (cc_forest.cpp:34) across ranks; the only data-path collective
  apply     replicated on every rank: rep[v] = winner, count applied hooks
  compress  replicated two-level pointer jumping
  stop      when a round applied nothing (identical on every rank)

`kernels` supplies init/hook/apply/compress on this rank's tensors: the CUDA
kernels of the C ABI (GpuKernels) in production; the CPU gloo tests plug in
a numpy restatement to check the partitioning and exchange logic.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def part_range(n: int, rank: int, world: int):
    return n * rank // world, n * (rank + 1) // world


def edge_base(local_m: int, rank: int, world: int, device) -> int:
    """Global id of this rank's first edge: exclusive prefix of edge counts."""
    if world == 1:
        return 0
    t = torch.tensor([local_m], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return int(sum(int(x.item()) for x in out[:rank]))


class GpuKernels:
    """The C-ABI CUDA kernels on a DeviceGraph holding this rank's edges."""

    def __init__(self, dg):
        self.dg = dg
        # Launch on torch's current stream so the NCCL all-reduce (ordered on
        # that stream) is complete before apply reads the slots.
        dg.set_stream(torch.cuda.current_stream().cuda_stream)

    def init(self, rep, slot):
        self.dg.cc_init(rep.data_ptr(), slot.data_ptr())

    def hook(self, mode, rep, slot):
        self.dg.cc_hook(mode, rep.data_ptr(), slot.data_ptr())

    def apply(self, rep, slot):
        return self.dg.cc_apply(rep.data_ptr(), slot.data_ptr())

    def compress(self, rep):
        self.dg.cc_compress(rep.data_ptr())


def distributed_cc(kernels, n: int, device, world: int = 1, max_rounds: int | None = None):
    """Runs the exact edge-partitioned connectivity; returns (rep, rounds, hooks).

    rep: int32 tensor of converged representatives (identical on all ranks).
    """
    rep = torch.empty(n, dtype=torch.int32, device=device)
    slot = torch.empty(n, dtype=torch.int64, device=device)
    kernels.init(rep, slot)
    mode, rounds, hooks = 0, 0, 0
    limit = max_rounds if max_rounds is not None else n + 1  # cc_forest.cpp:88
    while True:
        if rounds > limit:
            raise RuntimeError("hooking failed to converge")
        kernels.hook(mode, rep, slot)
        if world > 1:
            dist.all_reduce(slot, op=dist.ReduceOp.MIN)
        applied = kernels.apply(rep, slot)
        rounds += 1
        if applied == 0:
            break
        hooks += applied
        kernels.compress(rep)
        mode ^= 1
    return rep, rounds, hooks
