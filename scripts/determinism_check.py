import sys, numpy as np
sys.path.insert(0, '.')
import oracle as O, paper_2603_11645_b200 as P
gs = {"path4096": O.gen("path", 4096), "grid50": O.gen("grid", 50, 50), "rand": O.gen("random", 1000, 0.01, seed=3),
      "tt": O.from_edges(6, [(0,1),(1,2),(0,2),(3,4),(4,5),(3,5)])}
for name, g in gs.items():
    for csr in (True, False):
        dg = P.DeviceGraph.from_host(g.n, np.stack([g.eu, g.ev], 1), *( (g.offsets, g.nbrs, g.origin) if csr else ()))
        for algo in (0, 1, 2):
            res = []
            for _ in range(4):
                p, r, lv, st = dg.run(algo, 0)
                res.append((p.tobytes(), st["steps"], st["work"]))
            same = all(x == res[0] for x in res)
            if not same:
                print(name, "csr" if csr else "nocsr", algo, [(x[1], x[2]) for x in res], [x[0] == res[0][0] for x in res])
        dg.close()
print("done")
