#!/usr/bin/env python
"""Per-source-line stall summary of an ncu --set full capture (imported
source, -lineinfo): the lines with the most warp-stall samples and their
dominant stall reasons.

    python scripts/ncu_lines.py prof.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import subprocess
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows, hdr, fname = [], None, ""
    for line in out.splitlines():
        if line.startswith('"File Path"'):
            fname = line.split(",")[1].strip('"').split("/")[-1]
            continue
        if line.startswith('"Line No"'):
            hdr = next(csv.reader([line]))
            hdr[1] = "Source"
            hdr[3] = "SASS"
            continue
        if hdr is None or line.startswith('""'):
            continue  # (per-instruction rows; the line rows carry the sums)
        r = next(csv.reader([line]))
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        d["file"] = fname
        rows.append(d)
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r.get(key) or 0) for r in rows) or 1.0
    stall_cols = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
    rows.sort(key=lambda r: -float(r.get(key) or 0))
    print(f"total samples {tot:.0f}")
    for r in rows[: a.top]:
        s = float(r.get(key) or 0)
        if s == 0:
            break
        st = sorted(((float(r.get(c) or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        reasons = " ".join(f"{n}:{v / s:.0%}" for v, n in st if v > 0)
        print(f"{s / tot:6.1%} {r['file']}:{r['Line No']:>5s}  {r['Source'].strip()[:70]:70s} {reasons}")


if __name__ == "__main__":
    sys.exit(main())
