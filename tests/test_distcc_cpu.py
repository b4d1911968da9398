"""CPU (gloo, world_size 2 and 3) test of the edge-partitioned connectivity
protocol (paper_2603_11645_b200/distcc.py, csrc/cc.cu cc_exact with a
CcExchange): partitioning by smaller endpoint, global edge ids via the
all-gathered prefix, the dense round-0 slot exchange, then per round the
MIN all-reduce of the CURRENT ROOTS' slots only (gathered in roots-list
order, the list replicated on every rank), replicated apply over the roots
list, and the global stop decision.

The per-rank kernels are a numpy restatement of that round structure (the
CUDA kernels run the same protocol in tests/test_gpu_parity.py::
test_distcc_multiprocess_cuda); the exchange is distcc.SlotExchange
itself, over gloo. Labels and tree-edge totals must equal the single-
process reference labels bit for bit, and the exchanged volume after round
0 must be the roots' slots, not 8n per round."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

INF = np.iinfo(np.int64).max
SENT = INF - 1  # kKeyEdge (common.cuh)


def protocol_cc(n, eu, ev, e_base, exchange):
    """cc_exact's edge-partitioned rounds (cc.cu) in numpy on this rank's
    edges; exchange = distcc.SlotExchange (CPU tensors)."""
    slot = exchange.slot.numpy()
    xbuf = exchange.xbuf.numpy()
    rep = np.arange(n, dtype=np.int64)
    ids = np.arange(len(eu), dtype=np.int64) + e_base
    # round 0 (min mode, singleton reps): slot[v] = min over edges (u, v),
    # u < v; the smaller endpoint gets the "has an edge" sentinel, so after
    # the exchange an empty slot marks an isolated vertex (kept off the list)
    slot[:n] = INF
    lo, hi = np.minimum(eu, ev), np.maximum(eu, ev)
    np.minimum.at(slot, hi, (lo << 32) | ids)
    np.minimum.at(slot, lo, SENT)
    exchange(0, n)
    hit = slot[:n] < SENT
    rep[hit] = slot[:n][hit] >> 32
    roots = np.nonzero(slot[:n] == SENT)[0]  # replicated on every rank, in id order
    slot[:n] = INF
    hooks = int(hit.sum())
    while True:  # jump to convergence (compressed reps for the next hook)
        nr = rep[rep]
        if np.array_equal(nr, rep):
            break
        rep = nr
    mode, rounds = 1, 1
    while True:
        rounds += 1
        ru, rv = rep[eu], rep[ev]
        keep = ru != rv
        a, b = np.minimum(ru, rv)[keep], np.maximum(ru, rv)[keep]
        win, los = (a, b) if mode == 0 else (b, a)
        np.minimum.at(slot, los, (win << 32) | ids[keep])
        R = len(roots)
        xbuf[:R] = slot[roots]  # gather in roots-list order
        exchange(1, R)
        slot[roots] = xbuf[:R]
        got = slot[roots] != INF
        if not got.any():  # global: the same on every rank
            break
        hooked = roots[got]
        rep[hooked] = slot[hooked] >> 32
        slot[hooked] = INF
        hooks += len(hooked)
        roots = roots[~got]
        while True:
            nr = rep[rep]
            if np.array_equal(nr, rep):
                break
            rep = nr
        mode ^= 1
    return rep, rounds, hooks


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
    from paper_2603_11645_b200.distcc import SlotExchange, edge_base, part_range

    lo, hi = part_range(n, rank, world)
    sel = (eu >= lo) & (eu < hi)  # eu = smaller endpoint (normalized list)
    idx = np.nonzero(sel)[0]
    assert len(idx) == 0 or np.all(np.diff(idx) == 1), "partition must be contiguous"
    base = edge_base(len(idx), rank, world, "cpu")
    assert len(idx) == 0 or base == idx[0]
    ex = SlotExchange(n, "cpu", world)
    rep, rounds, hooks = protocol_cc(n, eu[sel], ev[sel], base, ex)
    out[rank] = (rep.copy(), rounds, hooks, list(ex.calls))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,spec", [(2, ("kron", 10)), (2, ("random", 300, 0.01)),
                                        (2, ("road", 30)), (3, ("kron", 11)), (3, ("path", 200)),
                                        (3, ("random", 400, 0.002))])
def test_distributed_cc_matches_single(O, world, spec):
    g = O.gen(*spec, seed=5) if spec[0] == "random" else O.gen(*spec)
    labels, te = O.cc_spanning_forest(g)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, g.n, g.eu, g.ev, out), nprocs=world, join=True)
    calls0 = out[0][3]
    for r in range(world):
        rep, rounds, hooks, calls = out[r]
        assert np.array_equal(rep, labels), f"rank {r} labels differ"
        assert hooks == len(te)
        assert calls == calls0  # every rank joins the same collectives
    # one dense round-0 exchange, then only the shrinking roots lists
    assert calls0[0] == (0, g.n)
    counts = [c for w, c in calls0[1:]]
    assert all(w == 1 for w, _ in calls0[1:])
    assert counts == sorted(counts, reverse=True) and counts[0] < g.n


def test_slot_exchange_single_rank_is_identity():
    from paper_2603_11645_b200.distcc import SlotExchange

    ex = SlotExchange(5, "cpu", 1)
    ex.slot[:] = torch.tensor([5, 4, 3, 2, 1])
    assert ex(0, 5) == 0 and ex.slot.tolist() == [5, 4, 3, 2, 1]
    assert ex.calls == [(0, 5)] and ex.bytes_per_rank() == 40
