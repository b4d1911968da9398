#!/usr/bin/env python
"""Small runs of every strategy for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): the smoke graph plus road:40, kron:10 and path:1000,
each through the C ABI, checked against the oracle so a sanitizer-perturbed
run is still verified. No torch import (faster under the sanitizer).

    compute-sanitizer --tool memcheck --error-exitcode 99 python scripts/sanitize.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2603_11645_b200 as P  # noqa: E402

CASES = [(("grid", 64, 48), 5), (("road", 40), 0), (("kron", 10), None), (("path", 1000), 999)]


def main():
    quick = "--quick" in sys.argv
    for spec, root in CASES[:2] if quick else CASES:
        g = O.gen(*spec)
        if root is None:
            root = int(np.argmax(np.diff(g.offsets)))
        dg = P.DeviceGraph.from_host(g.n, np.stack([g.eu, g.ev], 1), g.offsets, g.nbrs, g.origin)
        for algo in (P.BFS, P.CC_EULER, P.PR_RST):
            p, r, lv, _ = dg.run(algo, root, 5)
            ep, er, _ = O.run(g, algo, root, 5)
            assert np.array_equal(p, ep) and np.array_equal(r, er), (spec, algo)
        # the edge-list upload path (device CSR build, keyed round 0) too
        de = P.DeviceGraph.from_host(g.n, np.stack([g.eu, g.ev], 1))
        for algo in (P.CC_EULER, P.PR_RST, P.BFS):
            assert np.array_equal(de.run(algo, root, 5)[0], O.run(g, algo, root, 5)[0])
        labels, te = dg.cc_spanning_forest()
        assert np.array_equal(te, O.cc_spanning_forest(g)[1])
        assert dg.validate(O.run(g, 1, root)[0], root)[0]
        dg.close()
        de.close()
        print("ok", spec, flush=True)
    print("sanitize run complete")


if __name__ == "__main__":
    main()
