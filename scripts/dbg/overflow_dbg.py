import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_11645_b200 as P

def run(g, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return g.run(1, 7)[0]
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v

spec = sys.argv[1] if len(sys.argv) > 1 else "road:3000"
g = P.DeviceGraph.generate(spec)
walk = run(g, {"RSTG_LR_TILES": "0"})
for tag, env in [("tiles", {"RSTG_LR_TILES": "1"}), ("tiles2", {"RSTG_LR_TILES": "1"}),
                 ("overflow_deferred", {"RSTG_LR_TILES": "1", "RSTG_LR_TILECONTRACT": "1000000"}),
                 ("shortbound", {"RSTG_LR_TILES": "1", "RSTG_LR_SEGBOUND": "20000"})]:
    p = run(g, env)
    print(tag, "mismatches", int((p != walk).sum()), flush=True)
g2 = P.DeviceGraph.generate(spec)
p = run(g2, {"RSTG_LR_TILES": "1", "RSTG_LR_TILECONTRACT": "1000000"})
print("overflow_fresh", "mismatches", int((p != walk).sum()), flush=True)
p = run(g2, {"RSTG_LR_TILES": "1", "RSTG_LR_TILELEVELS": "0"})
print("levels0", "mismatches", int((p != walk).sum()), flush=True)
