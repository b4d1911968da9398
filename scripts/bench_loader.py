#!/usr/bin/env python
"""Loader throughput: a road_usa-sized edge-list
text -- road:4899 (24.0M vertices), every edge written in BOTH directions
with shuffled line order and a MatrixMarket header, 57.7M lines as in the
road_usa .mtx -- loaded by rstg_edge_list_load (multi-threaded parse, device
id remap + normalize) and turned into a device graph. The reference's
load_edge_list (oracle/_ref, single-threaded parse + std::sort) is timed on
the same text when --ref is given, and the two EdgeLists are compared.

    python scripts/bench_loader.py [--ref] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_text(R=4899, seed=1):
    import oracle as O
    g = O.gen("road", R)
    u = np.concatenate([g.eu, g.ev]) + 1  # MatrixMarket ids are 1-based
    v = np.concatenate([g.ev, g.eu]) + 1
    perm = np.random.RandomState(seed).permutation(len(u))
    u, v = u[perm], v[perm]
    body = np.char.add(np.char.add(u.astype("S10"), b" "), np.char.add(v.astype("S10"), b"\n"))
    head = f"%%MatrixMarket matrix coordinate pattern symmetric\n{g.n} {g.n} {len(u)}\n".encode()
    return g, head + b"".join(body.tolist())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--R", type=int, default=4899)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    t0 = time.perf_counter()
    g, text = make_text(a.R)
    gen_s = time.perf_counter() - t0
    import paper_2603_11645_b200 as P
    threads = os.cpu_count() or 1
    P.load_edge_list(b"1 2\n")  # (library + CUDA context warm-up)
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        dg = P.DeviceGraph.from_edge_list_text(text, threads)
        times.append(time.perf_counter() - t0)
        n, m = dg.n, dg.m
        dg.close()
    t0 = time.perf_counter()
    n2, e, ids = P.load_edge_list(text, threads)
    el_s = time.perf_counter() - t0
    out = {"text_bytes": len(text), "lines": int(text.count(b"\n")), "n": n, "m": m,
           "host_threads": threads, "generate_text_s": round(gen_s, 1),
           "edge_list_to_device_graph_s": [round(t, 3) for t in times],
           "load_edge_list_with_copy_out_s": round(el_s, 3),
           "matches_generator": bool(m == g.m and np.array_equal(e[:, 0], g.eu - 0)
                                     and np.array_equal(e[:, 1], g.ev))}
    if a.ref:
        import oracle as O
        t0 = time.perf_counter()
        rn, ru, rv, rids = O.ref_load_edge_list(text)
        out["reference_load_edge_list_s"] = round(time.perf_counter() - t0, 3)
        out["equal_to_reference"] = bool(rn == n2 and np.array_equal(ru, e[:, 0])
                                         and np.array_equal(rv, e[:, 1])
                                         and np.array_equal(rids, ids))
    print(json.dumps(out))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
