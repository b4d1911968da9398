#!/usr/bin/env python
"""Collect per-phase DRAM traffic from ncu launch lists into
profiles/phase_traffic.json (read by bench.py for roofline.traffic):

    python scripts/make_phase_traffic.py gpurun_out profiles/phase_traffic.json TAG

Inputs: gpurun_out/phases_<workload>.json written by scripts/ncu_top.py from
`ncu --nvtx --print-nvtx-rename kernel --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum` over scripts/profile_step.py
(cc-euler, 2 builds; values per build).
"""
import glob
import json
import os
import sys


def main(src, dst, tag):
    out = {}
    if os.path.exists(dst):
        with open(dst) as f:
            out = json.load(f)
    for f in sorted(glob.glob(os.path.join(src, "phases_*.json"))):
        wl = os.path.basename(f)[len("phases_"):-len(".json")]
        algo = "cc-euler"
        if "__" in wl:  # phases_<workload>__<algo>.json
            wl, algo = wl.split("__", 1)
        with open(f) as fh:
            ph = json.load(fh)
        out.setdefault(wl, {})[algo] = {
            "source": f"ncu --nvtx --print-nvtx-rename kernel, dram__bytes_read.sum + dram__bytes_write.sum, "
                      f"per build, capture {tag} (profiles/{tag}/)",
            "phases": ph,
        }
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", dst, {k: list(v) for k, v in out.items()})


if __name__ == "__main__":
    main(*sys.argv[1:4])
