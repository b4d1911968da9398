#!/usr/bin/env python
"""One RST build (or a few) bracketed by cudaProfilerStart/Stop, for ncu:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --builds 2
    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -k regex:k_walk -c 2 -o gpurun_out/prof python scripts/profile_step.py

The graph is generated and the build warmed up (3 builds) outside the
profiled range, so the launch list holds exactly the timed builds' kernels.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_11645_b200 as P  # noqa: E402

SPECS = {"road": "road:4899", "grid": "grid:1024:1024", "path": "path:16777216",
         "rmat24": "kron:24:16"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="road", choices=sorted(SPECS))
    ap.add_argument("--algo", default="cc-euler", choices=sorted(P.ALGOS))
    ap.add_argument("--builds", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    g = P.DeviceGraph.generate(SPECS[a.workload])
    root = 0
    if a.workload == "rmat24":
        e = g.edges()
        root = int(np.argmax(np.bincount(e.ravel(), minlength=g.n)))
    algo = P.ALGOS[a.algo]
    par = torch.empty(g.n, dtype=torch.int32, device="cuda")
    lv = torch.empty(g.n, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    g.set_stream(s.cuda_stream)
    for _ in range(a.warmup):
        g.run_device(algo, root, par.data_ptr(), lv.data_ptr())
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.builds):
        st = g.run_device(algo, root, par.data_ptr(), lv.data_ptr())
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({"workload": a.workload, "algo": a.algo, "launches_per_build": st["launches"]})


if __name__ == "__main__":
    main()
