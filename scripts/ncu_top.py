#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python scripts/ncu_top.py launches.csv [--skip-before REGEX] [--top K] [--names]

Prints per-kernel totals (count, total us, share) over the launches after the
first launch matching --skip-before (e.g. the first timed-step kernel), or
with --names only the top-K kernel base names (for ncu -k regex:...).
"""
import argparse
import collections
import csv
import re
import sys


def rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "nsecond")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        yield r["Kernel Name"], v * scale


def base(name):
    name = re.sub(r"^void ", "", name)
    name = name.split("(")[0]
    return re.sub(r"<.*", "", name).split("::")[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--skip-before", default=None)
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--names", action="store_true")
    a = ap.parse_args()
    data = list(rows(a.csv))
    if a.skip_before:
        for i, (k, _) in enumerate(data):
            if re.search(a.skip_before, k):
                data = data[i:]
                break
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, us in data:
        tot[base(k)] += us
        cnt[base(k)] += 1
    total = sum(tot.values())
    order = sorted(tot, key=lambda k: -tot[k])
    if a.names:
        print("|".join(order[: a.top]))
        return
    print(f"{'kernel':32s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
    for k in order[: a.top]:
        print(f"{k:32s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k] / total:7.1%}")
    print(f"{'TOTAL':32s} {sum(cnt.values()):8d} {total:10.1f}")


if __name__ == "__main__":
    sys.exit(main())
