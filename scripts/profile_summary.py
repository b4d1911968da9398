#!/usr/bin/env python
"""Condense one gpurun_out/ of scripts/gpu_round.sh into profiles/<tag>/:

    python scripts/profile_summary.py gpurun_out profiles/<tag>

Copies the bench lines, launch-list summaries (per kernel and per phase,
with DRAM bytes) and the --page details CSVs of the full captures, and
writes full_captures.md: one row of key metrics per captured kernel (time,
DRAM bytes read/write, DRAM throughput, L1/L2 hit rates, occupancy).
"""
import csv
import glob
import json
import os
import shutil
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit %"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    for pat in ("bench_*.json", "*_summary.txt", "kernels_*.json", "phases_*.json", "pytest_gpu.log",
                "smoke.log", "smi.txt", "prof_*_details.csv"):
        for f in glob.glob(os.path.join(src, pat)):
            shutil.copy(f, dst)
    rows = []
    for f in sorted(glob.glob(os.path.join(src, "prof_*_raw.csv"))):
        data = list(csv.reader(open(f)))
        if len(data) < 3:
            continue
        hdr, units = data[0], data[1]
        for r in data[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0]
            vals = []
            for k, _ in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    vals.append(f"{r[i]} {units[i]}".strip())
                else:
                    vals.append("")
            rows.append((name, vals))
    if rows:
        with open(os.path.join(dst, "full_captures.md"), "w") as out:
            out.write("| kernel | " + " | ".join(lbl for _, lbl in KEYS) + " |\n")
            out.write("|---" * (len(KEYS) + 1) + "|\n")
            for name, vals in rows:
                out.write(f"| {name} | " + " | ".join(vals) + " |\n")
    print("wrote", dst, sorted(os.listdir(dst)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
