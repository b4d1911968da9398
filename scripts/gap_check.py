"""Per-step device time inside the pipeline (stats device_ms) vs the event
delta between consecutive steps: the difference is host time between steps."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_11645_b200 as P
spec = sys.argv[1] if len(sys.argv) > 1 else "road:4899"
timing = len(sys.argv) > 2 and sys.argv[2] == "timing"
g = P.DeviceGraph.generate(spec)
s = torch.cuda.Stream()
g.set_stream(s.cuda_stream)
d = torch.empty(g.n, dtype=torch.int32, device="cuda")
for _ in range(3):
    g.run_device(1, 0, d.data_ptr())
torch.cuda.synchronize()
g.set_timing(timing)
K = 20
evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
dev = []
evs[0].record(s)
for i in range(K):
    st = g.run_device(1, 0, d.data_ptr())
    if timing:
        g.phase_times()
    dev.append(st["device_ms"])
    evs[i + 1].record(s)
torch.cuda.synchronize()
step = [evs[i].elapsed_time(evs[i + 1]) for i in range(K)]
print(spec, "timing" if timing else "", "step ms median %.3f  device_ms median %.3f  launches %d"
      % (statistics.median(step), statistics.median(dev), st["launches"]))
