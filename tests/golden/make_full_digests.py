"""Full-size parity digests, generated from the REFERENCE itself.

For every BASELINE.json configuration that fits one host (grid 1024^2, path
16M, road 24M, RMAT/Kronecker-24), this runs the unmodified reference core
(oracle/_ref/librst_ref.so, compiled by oracle/Makefile from
/root/reference/proj/core) through its public API -- run_algorithm
(bench.cpp:38-54) for cc-euler and pr-rst, cc_spanning_forest
(cc_forest.hpp:42) for labels and tree-edge ids -- and stores sha256
digests of the outputs (little-endian int64, the reference's own layout) in
full_digests.json. The GPU test (tests/test_gpu_parity.py::
test_full_size_reference_digests) recomputes the digests from the CUDA path
on the device-generated graph, so the 24M-vertex headline is pinned to the
reference's own outputs, not only to the C restatement.

BFS on path/road/RMAT is infeasible for the reference (n x
levels scans); its digests come from the oracle's O(n+m) restatement
(og_bfs_rst_fast, pinned to the reference on every fixture) and are marked
"source": "restatement". Grid BFS comes from the reference.

The edge list of each graph is digested too: the device generators must
produce exactly the list the reference was given.

    python tests/golden/make_full_digests.py [name ...]   # ~10 min on 8 cores
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

# name -> (generator spec for O.gen / the device, root rule)
CASES = {
    "grid:1024:1024": (("grid", 1024, 1024), 0),
    "path:16777216": (("path", 16777216), 0),
    "road:4899": (("road", 4899), 0),
    "kron:24:16": (("kron", 24, 16), "maxdeg"),
}
OUT = os.path.join(HERE, "full_digests.json")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def edge_digest(eu, ev) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(eu, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(ev, dtype="<i8").tobytes())
    return h.hexdigest()


def max_degree_root(n, eu, ev) -> int:
    deg = np.bincount(eu, minlength=n) + np.bincount(ev, minlength=n)
    return int(np.argmax(deg))  # smallest id on ties


def main(names):
    workers = os.cpu_count() or 1
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        spec, root = CASES[name]
        t0 = time.time()
        g = O.gen(*spec)
        if root == "maxdeg":
            root = max_degree_root(g.n, g.eu, g.ev)
        rec = {"spec": list(spec), "n": int(g.n), "m": int(g.m), "root": int(root),
               "edges": edge_digest(g.eu, g.ev), "workers": workers}
        print(f"{name}: n={g.n} m={g.m} root={root} ({time.time() - t0:.1f} s gen)", flush=True)
        labels, te = O.ref_cc_spanning_forest(g, workers)
        rec["cc_labels"], rec["cc_tree_edges"] = digest(labels), digest(te)
        rec["components"] = int(g.n - len(te))
        for algo, tag in ((1, "cc_euler"), (2, "pr_rst")):
            t1 = time.time()
            p, r, _ = O.ref_run(g, algo, root, workers)
            rec[tag] = {"parent": digest(p), "roots": digest(r), "num_roots": int(len(r)),
                        "source": "reference", "ref_s": round(time.time() - t1, 2)}
            print(f"  {tag}: {rec[tag]['ref_s']} s", flush=True)
        if name.startswith("grid"):
            p, r, lv = O.ref_run(g, 0, root, workers)
            src = "reference"
        else:
            p, r, lv = O.run(g, 0, root)
            src = "restatement"
        rec["bfs"] = {"parent": digest(p), "roots": digest(r), "levels": digest(lv),
                      "num_roots": int(len(r)), "depth": int(lv.max()), "source": src}
        out[name] = rec
        json.dump(out, open(OUT, "w"), indent=1, sort_keys=True)
        print(f"  done in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
