"""Generates the golden fixtures in this directory from the REFERENCE itself.

Runs the unmodified reference core (oracle/_ref/librst_ref.so, compiled by
oracle/Makefile from /root/reference/proj/core) through its public API --
run_algorithm (bench.cpp:38-54), cc_spanning_forest (cc_forest.hpp:42),
build_euler/compute_successor/break_cycles/list_rank (euler_rooting.hpp) --
and stores inputs and outputs as compressed .npz. The fixtures travel with
the repo, so the oracle and the CUDA path are pinned to the reference even
where /root/reference is absent (the GPU box).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

CASES = [
    ("path:10", 0), ("path:100", 42), ("path:256", 7), ("star:10", 0), ("star:64", 5),
    ("grid:5:7", 0), ("grid:9:11", 13), ("grid:12:9", 5), ("grid:100:100", 0),
    ("complete:12", 3), ("random:200:0.02", 0), ("random:500:0.004", 0),
    ("random:2000:0.002", 17), ("random:1000:0.01", 3),
]
SEEDS = {"random:200:0.02": [1, 2, 3], "random:500:0.004": [1, 2, 3, 4, 5],
         "random:2000:0.002": [11], "random:1000:0.01": [3]}
EXTRA = {  # hand-built graphs of tests/oracles.hpp and test_bfs.cpp
    "two-triangles": (6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)], [0, 4]),
    "tiebreak": (4, [(0, 1), (0, 2), (1, 3), (2, 3)], [0]),
    "isolated": (8, [(1, 2), (5, 6), (6, 7)], [0, 2, 6]),
}


def run_case(name, g, roots):
    out = {"n": g.n, "eu": g.eu, "ev": g.ev}
    labels, te = O.ref_cc_spanning_forest(g)
    out["cc_labels"], out["cc_tree_edges"] = labels, te
    for root in roots:
        for algo, tag in ((0, "bfs"), (1, "cc_euler"), (2, "pr_rst")):
            p, r, lv = O.ref_run(g, algo, root)
            out[f"{tag}_r{root}_parent"] = p
            out[f"{tag}_r{root}_roots"] = r
            if lv is not None:
                out[f"{tag}_r{root}_levels"] = lv
    out["roots"] = np.array(roots, np.int64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def euler_fixture():
    # random attachment trees: reference ranks (list_rank) per arc
    rs = np.random.RandomState(424242)
    out = {}
    for t in range(20):
        n = int(rs.randint(2, 200))
        te = np.array([(int(rs.randint(0, v)), v) for v in range(1, n)], np.int64)
        succ, rank = O.ref_euler_ranks(n, te, [0])
        out[f"t{t}_n"] = np.array([n])
        out[f"t{t}_edges"] = te
        out[f"t{t}_succ"] = succ
        out[f"t{t}_rank"] = rank
    np.savez_compressed(os.path.join(HERE, "euler_ranks.npz"), **out)


def main():
    if not O.have_ref():
        O.build()
    for spec, root in CASES:
        for seed in SEEDS.get(spec, [0]):
            g = O.ref_generate(spec, seed)
            roots = sorted({root, 0, g.n - 1})
            name = spec.replace(":", "_") + (f"_s{seed}" if spec.startswith("random") else "")
            run_case(name, g, roots)
    for name, (n, edges, roots) in EXTRA.items():
        run_case(name, O.from_edges(n, edges), roots)
    euler_fixture()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
