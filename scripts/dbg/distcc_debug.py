"""Debug: edge-partitioned cc_exact (a) 1 rank with an identity exchange,
(b) k ranks emulated by threads in one process (barrier + torch.minimum)."""
import os, sys, threading
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle as O
import paper_2603_11645_b200 as P
from paper_2603_11645_b200.distcc import SlotExchange

spec = sys.argv[1] if len(sys.argv) > 1 else "kron:13"
s = int(spec.split(":")[1])
g = O.gen("kron", s)
labels, te = O.cc_spanning_forest(g)
# (a) identity exchange, 1 rank
dg = P.DeviceGraph.generate_part(spec, 0, 1)
ex = SlotExchange(dg.n, "cuda", 1)
rep = torch.empty(dg.n, dtype=torch.int32, device="cuda")
dg.set_stream(torch.cuda.current_stream().cuda_stream)
st = dg.cc_labels(rep.data_ptr(), 0, ex.slot.data_ptr(), ex.xbuf.data_ptr(), ex)
print("identity-exchange 1 rank:", np.array_equal(rep.cpu().numpy(), labels), st["tree_edges"], len(te), ex.calls[:6])
# (b) k ranks by threads
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
parts = [P.DeviceGraph.generate_part(spec, r, k) for r in range(k)]
base = 0
for p in parts:
    p.set_edge_base(base); base += p.m
n = parts[0].n
streams = [torch.cuda.Stream() for _ in range(k)]
exs = [SlotExchange(n, "cuda", 1) for _ in range(k)]
bar = threading.Barrier(k)
reps = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(k)]
out = [None] * k
def make_cb(r):
    def cb(which, count):
        torch.cuda.synchronize()
        bar.wait()
        if r == 0 and which == 1 and len(exs[0].calls) == 1:
            INF = np.iinfo(np.int64).max
            rp = [x.cpu().numpy().astype(np.int64) for x in reps]
            print("rep equal across ranks:", np.array_equal(rp[0], rp[1]), "rep compressed:", np.array_equal(rp[0][rp[0]], rp[0]))
            ru, rv = rp[0][g.eu], rp[0][g.ev]
            keep = ru != rv
            lo, hi = np.minimum(ru, rv)[keep], np.maximum(ru, rv)[keep]
            exp = np.full(n, INF, np.int64)
            np.minimum.at(exp, lo, (hi << 32) | np.nonzero(keep)[0])
            got = np.minimum(*[e.slot.cpu().numpy()[:n] for e in exs])
            print("round-1 proposals: expected", int((exp != INF).sum()), "got", int((got != INF).sum()),
                  "equal", np.array_equal(exp, got))
            bad = np.nonzero(exp != got)[0][:8]
            print("  diffs at", bad, exp[bad], got[bad], [ (e.slot.cpu().numpy()[bad]) for e in exs])
            isroot = rp[0] == np.arange(n)
            print("  got at non-roots:", int(((got != INF) & ~isroot).sum()))
        if r == 0 and which == 1 and len(exs[0].calls) <= 3:
            INF = np.iinfo(np.int64).max
            for q, e in enumerate(exs):
                sl = e.slot.cpu().numpy()[:n]; xb = e.xbuf.cpu().numpy()[:count]
                print(f"  call {len(exs[0].calls)} rank {q}: slot non-INF {(sl != INF).sum()}, xbuf non-INF {(xb != INF).sum()} of {count}, xbuf sorted-unique-nonINF {len(np.unique(xb[xb != INF]))}")
        if r == 0:
            bufs = [(e.slot if which == 0 else e.xbuf)[:count] for e in exs]
            m = bufs[0].clone()
            for b in bufs[1:]:
                m = torch.minimum(m, b)
            for b in bufs:
                b.copy_(m)
            torch.cuda.synchronize()
        bar.wait()
        exs[r].calls.append((which, int(count)))
        return 0
    return cb
def run(r):
    with torch.cuda.stream(streams[r]):
        parts[r].set_stream(streams[r].cuda_stream)
        out[r] = parts[r].cc_labels(reps[r].data_ptr(), 0, exs[r].slot.data_ptr(), exs[r].xbuf.data_ptr(), make_cb(r))
ths = [threading.Thread(target=run, args=(r,)) for r in range(k)]
[t.start() for t in ths]; [t.join() for t in ths]
for r in range(k):
    rr = reps[r].cpu().numpy()
    print(f"rank {r}: labels equal {np.array_equal(rr, labels)}, tree {out[r]['tree_edges']} vs {len(te)}, rounds {out[r]['rounds']}, calls {exs[r].calls[:8]}")
    if not np.array_equal(rr, labels):
        bad = np.nonzero(rr != labels)[0]
        print("   first diffs", bad[:10], rr[bad[:10]], labels[bad[:10]])
