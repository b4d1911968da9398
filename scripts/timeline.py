#!/usr/bin/env python
"""Kernel timeline of warm builds (CUPTI via torch.profiler, no replay):
per kernel its start offset, duration and the idle gap before it, so the
time a build spends between kernels (host syncs, launch latency) is visible
next to the kernels themselves. Not a bench number: the profiler adds a
little overhead per launch.

    python scripts/timeline.py --workload road --algo cc-euler [--builds 3] [--json out.json]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2603_11645_b200 as P  # noqa: E402

SPECS = {"road": "road:4899", "grid": "grid:1024:1024", "path": "path:16777216",
         "rmat24": "kron:24:16"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="road", choices=sorted(SPECS))
    ap.add_argument("--algo", default="cc-euler", choices=sorted(P.ALGOS))
    ap.add_argument("--builds", type=int, default=3)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    g = P.DeviceGraph.generate(SPECS[a.workload])
    root = 0
    if a.workload == "rmat24":
        e = g.edges()
        root = int(np.argmax(np.bincount(e.ravel(), minlength=g.n)))
        del e
    algo = P.ALGOS[a.algo]
    par = torch.empty(g.n, dtype=torch.int32, device="cuda")
    lv = torch.empty(g.n, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    g.set_stream(s.cuda_stream)
    for _ in range(3):
        g.run_device(algo, root, par.data_ptr(), lv.data_ptr())
    torch.cuda.synchronize()
    builds = []
    for _ in range(a.builds):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            g.run_device(algo, root, par.data_ptr(), lv.data_ptr())
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if str(getattr(e, "device_type", "")).endswith("CUDA")]
        ev = sorted(ev, key=lambda e: e.time_range.start)
        rows, prev_end, t0 = [], None, ev[0].time_range.start if ev else 0
        for e in ev:
            st, en = e.time_range.start, e.time_range.end
            nm = e.name.replace("(anonymous namespace)::", "").split("(")[0][:60]
            rows.append({"name": nm, "start_us": st - t0, "dur_us": en - st,
                         "gap_us": 0 if prev_end is None else max(0, st - prev_end)})
            prev_end = en if prev_end is None else max(prev_end, en)
        builds.append(rows)
    last = builds[-1]
    span = [b[-1]["start_us"] + b[-1]["dur_us"] for b in builds]
    busy = [sum(r["dur_us"] for r in b) for b in builds]
    print(f"{a.workload} {a.algo}: span {statistics.median(span):.1f} us, kernels "
          f"{statistics.median(busy):.1f} us, idle {statistics.median(span) - statistics.median(busy):.1f} us, "
          f"{len(last)} device activities")
    agg = {}
    for r in last:
        acc = agg.setdefault(r["name"], [0.0, 0, 0.0])
        acc[0] += r["dur_us"]
        acc[1] += 1
        acc[2] += r["gap_us"]
    print("per kernel (us, launches, idle before):")
    for k, (d, c, gp) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"  {d:10.1f} {c:5d} {gp:8.1f}  {k}")
    for r in last:
        print(f"{r['start_us']:9.1f} {r['dur_us']:8.1f} gap {r['gap_us']:7.1f}  {r['name']}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"span_us": span, "busy_us": busy, "last": last}, f, indent=1)


if __name__ == "__main__":
    main()
