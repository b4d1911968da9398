"""Verifies BASELINE config 5 (Kronecker-28 connectivity, ~4.2e9 edges) on one
B200 against independent host checks (the reference's host
Graph would need ~200 GB, so it cannot run this size).

  1. GPU: rstg_cc_labels on the device-generated graph (the bench's path,
     edge-partitioned code with one partition) -> labels + tree-edge flags;
     the flagged edges are copied out as (u, v) pairs.
  2. Host (oracle/kron_uf.c, test infrastructure): every one of the 2^32
     Kronecker tuples is regenerated on the host cores and unioned into an
     int32 union-find (1 GiB) -- validate.cpp:46-53 oracle_components,
     streamed. Then:
       * the GPU labels describe the same partition as the union-find;
       * tree edges = n - components;
       * a second union-find over the GPU's tree edges alone has exactly
         n - T classes (every tree edge merges two classes: no cycle) and the
         same classes as the graph (the forest spans every component).
  3. Optionally (--ranks K): K processes sharing the GPU run the
     edge-partitioned rounds with the host-staged exchange; each rank's
     labels must equal the 1-partition labels bit for bit.

    python scripts/verify_kron28.py --scale 28 --out gpurun_out/kron28_verify.json [--ranks 2]
"""
import argparse
import json
import os
import socket
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gpu_labels(spec):
    import torch

    import paper_2603_11645_b200 as P
    from paper_2603_11645_b200.distcc import distributed_cc

    t0 = time.perf_counter()
    dg = P.DeviceGraph.generate_part(spec, 0, 1)
    gen_s = time.perf_counter() - t0
    n, m = dg.n, dg.m
    tflag = torch.zeros(max(m, 1), dtype=torch.uint8, device="cuda")
    distributed_cc(dg, n, 1, tflag)  # warm-up
    tflag.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep, st = distributed_cc(dg, n, 1, tflag)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    labels = rep.cpu().numpy()
    te = dg.edges_flagged(tflag.data_ptr(), n).astype(np.int32)
    dg.close()
    del tflag, rep
    torch.cuda.empty_cache()
    return labels, te, {"n": n, "m": m, "gpu_ms": ms, "rounds": st["rounds"],
                        "tree_edges": st["tree_edges"], "generation_s": round(gen_s, 2)}


def _rank_worker(rank, world, port, spec, outdir):
    import torch
    import torch.distributed as dist

    import paper_2603_11645_b200 as P
    from paper_2603_11645_b200.distcc import SlotExchange, distributed_cc, edge_base

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dg = P.DeviceGraph.generate_part(spec, rank, world)
    dg.set_edge_base(edge_base(dg.m, rank, world, "cpu"))
    ex = SlotExchange(dg.n, "cuda", world, staged=True)
    t0 = time.perf_counter()
    rep, st = distributed_cc(dg, dg.n, world, None, ex)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"rank{rank}.npy"), rep.cpu().numpy())
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump({"m_local": dg.m, "wall_s": time.perf_counter() - t0, "rounds": st["rounds"],
                   "tree_edges": st["tree_edges"], "exchange_calls": ex.calls}, f)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--ranks", type=int, default=0)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import oracle as O

    spec = f"kron:{args.scale}:{args.ef}"
    rec = {"spec": spec, "host_threads": args.threads}
    labels, te, g = gpu_labels(spec)
    rec.update(g)
    n, T = g["n"], len(te)
    print(f"gpu: n={n} m={g['m']} {g['gpu_ms']:.1f} ms, rounds {g['rounds']}, T={T}", flush=True)

    t0 = time.perf_counter()
    root, comps = O.kron_uf(args.scale, args.ef, args.threads)
    rec["host_uf_s"] = round(time.perf_counter() - t0, 1)
    rec["components"] = comps
    rec["labels_partition_equal"] = bool(O.same_partition(labels, root))
    rec["tree_edges_eq_n_minus_c"] = bool(T == n - comps and g["tree_edges"] == T)
    t0 = time.perf_counter()
    troot, tcomps = O.uf_edges(n, te, args.threads)
    rec["tree_uf_s"] = round(time.perf_counter() - t0, 1)
    rec["tree_acyclic"] = bool(tcomps == n - T)
    rec["tree_spans_components"] = bool(np.array_equal(troot, root))
    rec["tree_edges_oriented"] = bool(T == 0 or (te[:, 0] < te[:, 1]).all())
    print(json.dumps(rec), flush=True)

    if args.ranks > 1:
        import tempfile

        import torch.multiprocessing as mp
        with tempfile.TemporaryDirectory() as d:
            s = socket.socket()
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
            s.close()
            t0 = time.perf_counter()
            mp.spawn(_rank_worker, args=(args.ranks, port, spec, d), nprocs=args.ranks, join=True)
            ranks = []
            for r in range(args.ranks):
                lab_r = np.load(os.path.join(d, f"rank{r}.npy"))
                info = json.load(open(os.path.join(d, f"rank{r}.json")))
                info["labels_equal_1gpu"] = bool(np.array_equal(lab_r, labels))
                info["exchange_bytes"] = 8 * sum(c for _, c in info.pop("exchange_calls"))
                ranks.append(info)
            rec["partitioned"] = {"ranks": args.ranks, "exchange": "gloo, host-staged (one GPU)",
                                  "wall_s": round(time.perf_counter() - t0, 1), "per_rank": ranks}
    rec["verified"] = bool(rec["labels_partition_equal"] and rec["tree_edges_eq_n_minus_c"] and
                           rec["tree_acyclic"] and rec["tree_spans_components"] and
                           all(r["labels_equal_1gpu"] for r in rec.get("partitioned", {}).get("per_rank", [])))
    print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rec, f, indent=1)
    return 0 if rec["verified"] else 1


if __name__ == "__main__":
    sys.exit(main())
