"""CPU (gloo, world_size 2 and 3) test of the edge-partitioned connectivity
driver (paper_2603_11645_b200/distcc.py): partitioning by smaller endpoint,
global edge ids via the all-gathered prefix, MIN all-reduce of the hook
slots, replicated apply/compress. The per-rank kernels are a numpy
restatement of cc_forest.cpp's hook/apply/jump (the CUDA kernels are
covered by tests/test_gpu_parity.py); the labels must equal the
single-process reference labels bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

INF = np.iinfo(np.int64).max


class NumpyKernels:
    def __init__(self, eu, ev, e_base):
        self.eu, self.ev, self.e_base = eu, ev, e_base

    def init(self, rep, slot):
        rep.copy_(torch.arange(len(rep), dtype=torch.int32))
        slot.fill_(INF)

    def hook(self, mode, rep, slot):  # cc_forest.cpp:18-35 on the local edges
        r = rep.numpy()
        s = slot.numpy()
        ru, rv = r[self.eu], r[self.ev]
        keep = ru != rv
        lo, hi = np.minimum(ru, rv)[keep], np.maximum(ru, rv)[keep]
        win, los = (lo, hi) if mode == 0 else (hi, lo)
        ids = (np.nonzero(keep)[0] + self.e_base).astype(np.int64)
        keys = (win.astype(np.int64) << 32) | ids
        np.minimum.at(s, los, keys)

    def apply(self, rep, slot):  # cc_forest.cpp:39-46
        r, s = rep.numpy(), slot.numpy()
        hit = s != INF
        r[hit] = (s[hit] >> 32).astype(np.int32)
        s[hit] = INF
        return int(hit.sum())

    def compress(self, rep):  # fixed point of jump_to_convergence
        r = rep.numpy()
        while True:
            nr = r[r]
            if np.array_equal(nr, r):
                break
            r[:] = nr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, eu, ev, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_11645_b200.distcc import distributed_cc, edge_base, part_range

    lo, hi = part_range(n, rank, world)
    sel = (eu >= lo) & (eu < hi)  # eu = smaller endpoint (normalized list)
    idx = np.nonzero(sel)[0]
    assert len(idx) == 0 or np.all(np.diff(idx) == 1), "partition must be contiguous"
    base = edge_base(len(idx), rank, world, "cpu")
    assert len(idx) == 0 or base == idx[0]
    rep, rounds, hooks = distributed_cc(NumpyKernels(eu[sel], ev[sel], base), n, "cpu", world)
    out[rank] = (rep.numpy().astype(np.int64).copy(), rounds, hooks)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,spec", [(2, ("kron", 10)), (2, ("random", 300, 0.01)),
                                        (2, ("road", 30)), (3, ("kron", 11)), (3, ("path", 200))])
def test_distributed_cc_matches_single(O, world, spec):
    g = O.gen(*spec, seed=5) if spec[0] == "random" else O.gen(*spec)
    labels, te = O.cc_spanning_forest(g)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, g.n, g.eu, g.ev, out), nprocs=world, join=True)
    for r in range(world):
        rep, rounds, hooks = out[r]
        assert np.array_equal(rep, labels), f"rank {r} labels differ"
        assert hooks == len(te)
