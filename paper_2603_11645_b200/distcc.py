"""Edge-partitioned connectivity across GPUs (config 5, Kron-28).

Rank r of k owns the edges whose smaller endpoint lies in
[r*n/k, (r+1)*n/k). Because the normalized edge list is sorted by that
endpoint, the rank's edges are ONE contiguous range of the global list:
global edge id = e_base + local index, with e_base = the edge counts of the
lower ranks (one all-gather). The hook keys (winner << 32 | global edge id)
are therefore the single-GPU keys, and the labels are bit-identical to the
1-GPU run (cc_spanning_forest, cc_forest.cpp:73-102).

The rounds are the single-GPU ones (csrc/cc.cu cc_exact, rstg_cc_labels):
round 0 from hook keys, lazy rounds that find roots, apply over the current
roots list only. Everything but the proposals is replicated on every rank:
the roots list, apply, the roots-list pointer jump and the stop decision.
The exchange before each apply is the only data-path collective:

  round 0   all_reduce(MIN) of the dense int64 slot array (8n bytes): every
            vertex may receive a key when all reps are singletons
  later     all_reduce(MIN) of the current roots' slots, gathered in roots-
            list order (8 bytes per root): road 24M has ~3.9K roots after
            round 0, RMAT-24 a few hundred thousand -- the exchange shrinks
            with the roots instead of costing 8n every round

That is exactly combine_min (cc_forest.cpp:34) across ranks. With the
NCCL backend the all-reduce runs on the device buffers on the handle's
stream; with gloo (CPU tests, several ranks sharing one GPU) it is staged
through host memory.
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


class SlotExchange:
    """The reduce_min callback of rstg_cc_labels: MIN-combines the hook
    slots (which 0: slot[:count], dense) or the roots' gathered slots
    (which 1: xbuf[:count]) across the ranks. Records (which, count) per
    call so callers can report the exchanged bytes."""

    def __init__(self, n: int, device, world: int, staged: bool | None = None):
        self.slot = torch.empty(max(n, 1), dtype=torch.int64, device=device)
        self.xbuf = torch.empty(max(n, 1), dtype=torch.int64, device=device)
        self.world = world
        if staged is None:
            staged = world > 1 and (torch.device(device).type == "cuda"
                                    and dist.get_backend() != "nccl")
        self.staged = staged
        self.calls: list[tuple[int, int]] = []
        self.error: BaseException | None = None

    def __call__(self, which: int, count: int) -> int:
        try:
            t = (self.slot if which == 0 else self.xbuf)[:count]
            self.calls.append((which, int(count)))
            if self.world > 1:
                if self.staged:
                    h = t.cpu()  # (ordered after the proposals: same stream)
                    dist.all_reduce(h, op=dist.ReduceOp.MIN)
                    t.copy_(h)
                else:
                    dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return 0
        except BaseException as e:  # reported by distributed_cc
            self.error = e
            return 1

    def bytes_per_rank(self) -> int:
        return 8 * sum(c for _, c in self.calls)


def distributed_cc(dg, n: int, world: int, tflag: torch.Tensor | None = None,
                   exchange: SlotExchange | None = None):
    """Exact connectivity labels of the edge-partitioned graph (this rank's
    DeviceGraph `dg`, edge base already set). Returns (rep int32 tensor,
    stats dict); rep is identical on all ranks and equal to the 1-GPU
    labels. world == 1: the optimised single-GPU rounds, no exchange."""
    # the collective runs on torch's current stream: launch there too
    dg.set_stream(torch.cuda.current_stream().cuda_stream)
    rep = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    if world > 1 and exchange is None:
        exchange = SlotExchange(n, "cuda", world)
    tp = tflag.data_ptr() if tflag is not None else 0
    try:
        if world > 1:
            st = dg.cc_labels(rep.data_ptr(), tp, exchange.slot.data_ptr(),
                              exchange.xbuf.data_ptr(), exchange)
        else:
            st = dg.cc_labels(rep.data_ptr(), tp)
    except Exception:
        if exchange is not None and exchange.error is not None:
            raise exchange.error
        raise
    return rep[:n], st
