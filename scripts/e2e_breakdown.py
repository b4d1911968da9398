#!/usr/bin/env python
"""Breakdown of the end-to-end path (bench.py e2e) on the road mesh:
upload (pinned int64 edges -> device + device CSR build), device build,
and the parent readback, each timed on its own."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_11645_b200 as P  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "road:4899"
g = P.DeviceGraph.generate(spec)
n, m = g.n, g.m
e = g.edges()
eh = torch.from_numpy(np.ascontiguousarray(e.ravel())).pin_memory()
ph = torch.empty(n, dtype=torch.int64).pin_memory()
ge = P.DeviceGraph.generate("path:2")
ge.upload(n, eh.numpy())
ge.run(1, 0)
d_par = torch.empty(n, dtype=torch.int32, device="cuda")


def t(f, k=5):
    xs = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        xs.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(xs)


up = t(lambda: ge.upload(n, eh.numpy()))
dev = t(lambda: ge.run_device(1, 0, d_par.data_ptr()))
full = t(lambda: ge.run(1, 0, out=ph.numpy(), want_roots=False, want_levels=False))
rd = t(lambda: ph.copy_(d_par.to(torch.int64), non_blocking=True))
both = t(lambda: (ge.upload(n, eh.numpy()), ge.run(1, 0, out=ph.numpy(), want_roots=False,
                                                      want_levels=False)))
print({"upload_ms": up, "device_build_ms": dev, "run_with_readback_ms": full,
       "torch_readback_ms": rd, "e2e_ms": both, "h2d_GBps": eh.numel() * 8 / up / 1e6})
