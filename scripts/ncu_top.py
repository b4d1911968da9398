#!/usr/bin/env python
"""Summarise an ncu launch list (--csv, one row per kernel launch and metric).

    python scripts/ncu_top.py launches.csv [--builds B] [--top K] [--names] [--json OUT]

Per kernel name (or per NVTX phase when the list was captured with
--nvtx --print-nvtx-rename kernel): launches, total device time, share, and
DRAM bytes read+written when those metrics were collected -- all divided by
--builds (the number of RST builds inside the profiled range). --names
prints the top-K kernel base names joined by '|' (for ncu -k regex:...).
--json writes {name: {"us": .., "launches": .., "dram_bytes": ..}} per build.
"""
import argparse
import collections
import csv
import json
import re
import sys

SCALE_T = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
           "second": 1e6, "s": 1e6}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    per = collections.OrderedDict()
    for r in csv.DictReader(lines):
        key = r.get("ID") or str(len(per))
        d = per.setdefault(key, {"name": r["Kernel Name"]})
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", "") or 0)
        mn = r["Metric Name"]
        if mn == "gpu__time_duration.sum":
            d["us"] = v * SCALE_T.get(unit, 1e-3)
        elif mn in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            d["dram"] = d.get("dram", 0.0) + v * SCALE_B.get(unit, 1)
        elif mn == "lts__t_sector_hit_rate.pct":
            d["l2hit"] = v
        elif mn in ("lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum"):
            d["atom"] = d.get("atom", 0.0) + v
    return list(per.values())


def base(name):
    head = name.split("(")[0]
    if "/" in head:  # NVTX-renamed: "<phase>/<kernel>(...)" -> phase
        return head.split("/")[0]
    name = re.sub(r"^void ", "", name)
    name = name.split("(")[0]
    return re.sub(r"<.*", "", name).split("::")[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--builds", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--names", action="store_true")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    data = launches(a.csv)
    tot = collections.defaultdict(float)
    dram = collections.defaultdict(float)
    cnt = collections.Counter()
    l2w = collections.defaultdict(float)  # time-weighted L2 hit rate
    atom = collections.defaultdict(float)
    have_dram = any("dram" in d for d in data)
    have_l2 = any("l2hit" in d for d in data)
    for d in data:
        k = base(d["name"])
        tot[k] += d.get("us", 0.0)
        dram[k] += d.get("dram", 0.0)
        l2w[k] += d.get("l2hit", 0.0) * d.get("us", 0.0)
        atom[k] += d.get("atom", 0.0)
        cnt[k] += 1
    total = sum(tot.values()) or 1.0
    order = sorted(tot, key=lambda k: -tot[k])
    if a.names:
        print("|".join(order[: a.top]))
        return
    B = a.builds
    if a.json:
        with open(a.json, "w") as f:
            json.dump({k: {"us": tot[k] / B, "launches": cnt[k] / B,
                           "dram_bytes": dram[k] / B if have_dram else None,
                           **({"l2_hit_pct": l2w[k] / tot[k] if tot[k] else None,
                               "l2_atom_red_sectors": atom[k] / B} if have_l2 else {})}
                       for k in order}, f, indent=1)
    hdr = f"{'name':34s} {'launches':>8s} {'us/build':>10s} {'share':>7s}"
    if have_dram:
        hdr += f" {'DRAM MB/build':>14s} {'GB/s':>8s}"
    if have_l2:
        hdr += f" {'L2 hit%':>8s} {'atom+red sect':>14s} {'Gsect/s':>8s}"
    print(hdr)
    for k in order[: a.top]:
        line = f"{k:34s} {cnt[k] / B:8.1f} {tot[k] / B:10.1f} {tot[k] / total:7.1%}"
        if have_dram:
            line += f" {dram[k] / B / 1e6:14.1f} {dram[k] / (tot[k] * 1e3) if tot[k] else 0:8.0f}"
        if have_l2:
            line += (f" {l2w[k] / tot[k] if tot[k] else 0:8.1f} {atom[k] / B:14.0f}"
                     f" {atom[k] / (tot[k] * 1e3) if tot[k] else 0:8.2f}")
        print(line)
    print(f"{'TOTAL':34s} {sum(cnt.values()) / B:8.1f} {total / B:10.1f}")


if __name__ == "__main__":
    sys.exit(main())
