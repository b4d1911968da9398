#!/usr/bin/env python
"""Benchmark driver: RST build throughput on B200 (arXiv 2603.11645 strategies).

A *step* is one full rooted-spanning-tree build (every component) of one
synthetic graph from a root: device-resident CSR + edge list in, parent
array P (P[r] = r) out. Default workload (BASELINE.json configs[2], the
north-star target): GConn-style CC + Euler-tour rooting (cc-euler) on the
road_usa-shaped mesh R=4899 (n = 24,000,201, m = 28,858,008), root 0.

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload road|grid|path|rmat24] [--algo cc-euler|pr-rst|bfs]
                    [--impl ours|reference]

Prints ONE JSON line (rank 0). `value` = edges/s over the device-resident
timed region (max over ranks; N>1 runs N independent replicas -- the Euler
tour is one linked list and does not shard). `e2e` = the same
metric through the C ABI from pinned host int64 buffers (edge list in,
parent array out, copies inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (device generator spec, root rule, BASELINE config index)
    "road": ("road:4899", 0, 2),
    "grid": ("grid:1024:1024", 0, 0),
    "path": ("path:16777216", 0, 1),
    "rmat24": ("kron:24:16", "maxdeg", 3),
    # edge-partitioned CC labels only (config 5); shards over ranks with an
    # NCCL MIN all-reduce per hook round
    "kron28cc": ("kron:28:16", None, 4),
    "kron26cc": ("kron:26:16", None, 4),
    "kron24cc": ("kron:24:16", None, 4),
}
REF_SAMPLE = {  # the reference arm times the SAME graph as the GPU arm
    "road": ("road", 4899),
    "grid": ("grid", 1024, 1024),
    "path": ("path", 1 << 24),
    "rmat24": ("kron", 24, 16),
}
# bench_row protocol of the reference (bench.cpp:56-92): 1 warm-up + 5 timed
# runs, median. The reference arm caps K and W at these (a road build is
# ~15 s on 16 cores), and says so in its line.
REF_MAX_TIMED, REF_MAX_WARMUP = 5, 1
ALGO_ID = {"bfs": 0, "cc-euler": 1, "pr-rst": 2}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="road", choices=sorted(WORKLOADS))
    ap.add_argument("--algo", default="cc-euler", choices=sorted(ALGO_ID))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bfs-ratio", action="store_true")
    ap.add_argument("--ref-workers", type=int, default=0,
                    help="reference arm: run_algorithm workers (default: every host core)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region (B200_PROFILING.md). NVML directly, every 2 ms: a whole timed
    region of a few-ms build is only tens of ms long, shorter than the
    nvidia-smi -lms floor. Falls back to nvidia-smi when NVML is absent."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index, period_s=0.002):
        self.index = index
        self.period = period_s
        self.samples = []  # (sm_mhz, reason bitmask)
        self.max_mhz = None
        self.stop = threading.Event()
        self.nv = None
        self.smi = []

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.nv = nv
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _sample(self):
        nv = self.nv
        self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))

    def _loop(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join(timeout=1)
            try:
                self._sample()  # at least one sample at the end of the region
            except Exception:
                pass
        else:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      "--query-gpu=clocks.sm,clocks.max.sm",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=10).stdout
                sm, mx = [float(x) for x in out.strip().split(",")[:2]]
                self.samples.append((sm, 0))
                self.max_mhz = mx
            except Exception:
                pass

    def summary(self):
        reasons = set()
        if self.nv:
            for name, attr in self.REASONS:
                bit = getattr(self.nv, attr, 0)
                if any(r & bit for _, r in self.samples):
                    reasons.add(name)
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nv else "nvidia-smi"}


# --------------------------------------------------------- roofline model
def phase_bytes(phase, n, m, E):
    """Algorithmic (compulsory) bytes of one build's worth of a phase:
    each array element the phase must touch, once."""
    T = E // 2
    R = E // 32 + 1
    return {
        "cc.init": 16 * n,                  # rep 4 + slot 8 + tree-edge slot 4 per vertex
        "cc.round0": 4 * (n + 1) + 16 * n,  # offsets + first neighbour/edge id 8 + rep 4 + tree edge 4
        "cc.hook_min": 16 * m,              # edge 8 + two rep gathers 4+4 (first visit; upper bound)
        "cc.hook_max": 16 * m,
        "cc.apply_compress": 16 * n,        # slot 8 + rep read/write 8 per vertex
        "euler.roots": 12 * n,              # labels 4 + min-vertex table 4 + parent 4
        "euler.arcs": 30 * T,               # tree list 4 + edge 8 per tree edge; arc 8 + succ 4 per arc
        "lr.rulers": 8 * R,                 # ruler position + word
        "lr.walk": 8 * E,                   # succ read 4 + (ruler, offset) word write 4 per arc
        "lr.rulers_rank": 16 * R,           # ruler list prefix (one pass)
        "euler.orient": 14 * E,             # arc pair 16 + words 8 + parent write 4 per tree edge
    }.get(phase)


def profiled_traffic(workload, algo, phase):
    """DRAM bytes (read + write) per build of `phase`, from the committed ncu
    capture of the same workload (profiles/phase_traffic.json, written by
    scripts/ncu_top.py from an `ncu --nvtx --print-nvtx-rename kernel` launch
    list with dram__bytes_{read,write}.sum). None when not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "phase_traffic.json")) as f:
            t = json.load(f)
        return t[workload][algo]["phases"][phase]["dram_bytes"], t[workload][algo]["source"]
    except Exception:
        return None, None


def count_kernels(step):
    """Kernels of this library (namespace rstg) launched by one step, from
    CUPTI activity records (torch.profiler); None if profiling is unavailable."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events()
                 if str(getattr(e, "device_type", "")).endswith("CUDA")]
        return sum(1 for nm in names if "rstg::" in nm or nm.startswith("k_"))
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


# ------------------------------------------------------------- cpu side
def cpu_reference(workload, algo, steps, warmup, cores=None):
    """The reference's own CPU implementation (oracle/_ref, compiled from
    /root/reference) on the same graph as the GPU arm; edges/s. Times
    exactly what bench_row times (bench.cpp:73-76): run_algorithm including
    its StepEngine construction, `cores` workers (default: every host core)."""
    import numpy as np
    import oracle as O

    cores = cores or os.cpu_count() or 1
    spec = REF_SAMPLE[workload]
    t0 = time.perf_counter()
    g = O.gen(*spec)
    root = 0
    if WORKLOADS[workload][1] == "maxdeg":
        root = int(np.argmax(np.diff(g.offsets)))
    kind = "reference" if O.have_ref() else "port"
    times = []
    if kind == "reference":
        rg = O.RefGraph(g)
        setup_s = time.perf_counter() - t0
        for i in range(warmup + steps):
            ms = rg.run_ms(ALGO_ID[algo], root, cores, 5)
            if i >= warmup:
                times.append(ms)
        del rg
    else:
        setup_s = time.perf_counter() - t0
        cores = 1
        for i in range(warmup + steps):
            t1 = time.perf_counter()
            O.run(g, ALGO_ID[algo], root)
            if i >= warmup:
                times.append((time.perf_counter() - t1) * 1e3)
    med = statistics.median(times)
    return {
        "value": g.m / (med / 1e3), "unit": "edges/s", "cores": cores, "kind": kind,
        "sample": f"{':'.join(map(str, spec))} (n={g.n}, m={g.m}, the GPU arm's graph), root {root}, "
                  f"{algo}, median of {len(times)} timed runs after {warmup} warm-up of run_algorithm "
                  f"with {cores} workers",
        "ms": med, "runs_ms": [round(t, 1) for t in times], "graph_setup_s": round(setup_s, 2),
    }


# ------------------------------------------------------- kron CC (multi-GPU)
def bench_kron_cc(args, rank, world, dev, metric, config):
    """Config 5: exact connectivity of a Kronecker graph, edges partitioned
    over the ranks (paper_2603_11645_b200/distcc.py): the single-GPU rounds
    of rstg_cc_labels with a MIN all-reduce of the hook slots before each
    apply (dense in round 0, the current roots' slots after). Strong
    scaling: the graph is fixed, each rank holds 1/N of the edges."""
    import torch

    import paper_2603_11645_b200 as P
    from paper_2603_11645_b200.distcc import SlotExchange, distributed_cc, edge_base

    spec = WORKLOADS[args.workload][0]
    t0 = time.perf_counter()
    dg = P.DeviceGraph.generate_part(spec, rank, world, device=dev)
    base = edge_base(dg.m, rank, world, "cuda")
    dg.set_edge_base(base)
    m_local = torch.tensor([dg.m], dtype=torch.int64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(m_local)
    m_total, n = int(m_local.item()), dg.n
    gen_s = time.perf_counter() - t0
    ex = SlotExchange(n, "cuda", world) if world > 1 else None

    def step():
        if ex is not None:
            ex.calls.clear()
        return distributed_cc(dg, n, world, None, ex)

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = None
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            rep, st = step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    comps = int((rep == torch.arange(n, device="cuda", dtype=torch.int32)).sum().item())
    peaks, peak_kind = measured_peaks()
    b_cc = 8 * m_total + 4 * n  # read edges once + write labels
    # phase breakdown of one instrumented (untimed) step
    dg.set_timing(True)
    step()
    phases = dg.phase_times()
    dg.set_timing(False)
    if rank == 0:
        config.update({"n": n, "m": m_total, "edges_per_rank": "1/N by smaller endpoint",
                       "rounds": st["rounds"], "tree_edges": st["tree_edges"], "components": comps,
                       "generation_s": round(gen_s, 2),
                       "exchange": ("NCCL all_reduce(int64 MIN): dense 8n bytes in round 0, "
                                    "then 8 B per current root") if world > 1 else "none (1 GPU)",
                       "exchange_bytes_per_rank": ex.bytes_per_rank() if ex else 0})
        line = {"metric": f"CC edges/sec ({args.workload}, edge-partitioned)",
                "value": m_total / (ms_per_step / 1e3), "unit": "edges/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "int32", "data": "synthetic", "config": config,
                "step_roofline": {"b_alg": b_cc,
                                  "frac_of_measured": b_cc / (ms_per_step / 1e3) / 1e9 / peaks["hbm_gbs"]},
                "phases_ms_per_step": {k: [round(v[0], 4), v[1], v[2]] for k, v in phases.items()},
                "clocks": clk.summary(), "cpu_baseline": None, "e2e": None}
    per_step = count_kernels(step)
    if rank == 0:
        line["gpu_launches"] = per_step * args.steps if per_step is not None else None
        line["gpu_launches_source"] = "CUPTI kernel records of one untimed step x steps"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    spec, root_rule, cfg_idx = WORKLOADS[args.workload]
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        baseline = json.load(f)
    metric = f"RST build edges/sec ({args.algo}, {args.workload})"
    config = {"workload": f"{spec} ({baseline['configs'][cfg_idx][:60]})", "algo": args.algo,
              "root": root_rule, "l2": "inputs larger than L2 (graph >> 126 MB)"
              if args.workload != "grid" else "grid CSR (25 MB) fits in L2: L2-resident",
              "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}

    if args.impl == "reference":
        # The reference arm: rank 0 only, the box's host cores.
        if rank != 0:
            return
        k, w = min(args.steps, REF_MAX_TIMED), min(args.warmup, REF_MAX_WARMUP)
        cb = cpu_reference(args.workload, args.algo, k, w, cores=args.ref_workers or None)
        line = {"impl": "reference", "metric": metric, "value": cb["value"], "unit": "edges/s",
                "n_gpus": args.gpus, "steps": k, "warmup": w,
                "requested": {"steps": args.steps, "warmup": args.warmup},
                "protocol": "bench_row (bench.cpp:56-92): median of the timed runs; K and W capped "
                            f"at {REF_MAX_TIMED} and {REF_MAX_WARMUP}",
                "runs_ms": cb["runs_ms"], "graph_setup_s": cb["graph_setup_s"],
                "ms_per_step": cb["ms"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int64", "data": "synthetic", "config": config,
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": "edges/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch

    import paper_2603_11645_b200 as P

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    if args.workload.startswith("kron") and args.workload.endswith("cc"):
        return bench_kron_cc(args, rank, world, dev, metric, config)
    stream = torch.cuda.Stream()
    g = P.DeviceGraph.generate(spec, device=dev)
    n, m = g.n, g.m
    root = 0
    e_host = None
    if root_rule == "maxdeg" or not args.no_e2e:
        e_host = g.edges()
    if root_rule == "maxdeg":
        deg = np.bincount(e_host.ravel(), minlength=n)
        root = int(np.argmax(deg))
        config["root"] = root
    g.set_stream(stream.cuda_stream)
    algo = ALGO_ID[args.algo]
    d_parent = torch.empty(n, dtype=torch.int32, device="cuda")
    d_levels = torch.empty(n, dtype=torch.int32, device="cuda") if algo == 0 else None
    lp = d_levels.data_ptr() if d_levels is not None else 0

    def step():
        return g.run_device(algo, root, d_parent.data_ptr(), lp)

    # the first build on a fresh handle pays the workspace allocation and the
    # one-time fills (slot array all-INF, Euler min table all-ones) that later
    # builds keep as invariants: reported beside the steady state, untimed
    # (the library's kernels are loaded first, on a tiny graph: module
    # loading is a per-process cost, not a per-handle one)
    tiny = P.DeviceGraph.generate("path:1000", device=dev)
    tiny.run_device(algo, 0, d_parent.data_ptr(), lp)
    tiny.close()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    c0.record(stream)
    step()
    c1.record(stream)
    torch.cuda.synchronize()
    cold_ms = c0.elapsed_time(c1)
    for _ in range(max(0, args.warmup - 1)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: device-resident, CUDA events on the launch stream
    # (uninstrumented: the phase timer's events cost ~0.1 ms a build, so the
    # phase breakdown comes from separate instrumented steps below)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]

    # ---- phase breakdown: instrumented steps (CUDA events per phase), untimed
    g.set_timing(True)
    phases = {}
    for _ in range(min(args.steps, 5)):
        step()
        for k, v in g.phase_times().items():
            phases.setdefault(k, []).append(v)
    g.set_timing(False)
    # ---- kernel launches per step, counted by CUPTI (torch.profiler) on one
    # extra untimed step: every kernel of the library's .so (namespace rstg)
    per_step_kernels = count_kernels(step)
    launches = per_step_kernels * args.steps if per_step_kernels is not None else None
    total_ms = evs[0].elapsed_time(evs[-1])
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * m / (ms_per_step / 1e3)

    # parity spot-check of the timed output against the device validator
    parent_host = d_parent.cpu().numpy().astype(np.int64)
    valid = g.validate(parent_host, root)[0]

    # ---- roofline of the dominant kernel (phase) ----
    E = 2 * (n - int((parent_host == np.arange(n)).sum()))
    peaks, peak_kind = measured_peaks()
    # per phase: mean over steps of (ms in the step, records in the step,
    # algorithmic bytes the library attributes to the phase -- DESIGN.md §3)
    agg = {k: (statistics.mean(x[0] for x in v), statistics.mean(x[1] for x in v),
               statistics.mean((x[2] if len(x) > 2 else 0) for x in v))
           for k, v in phases.items()}
    dominant = max(agg, key=lambda k: agg[k][0]) if agg else None
    roofline = None
    if dominant:
        per_step_ms, per_step_launches, lib_bytes = agg[dominant]
        # algorithmic bytes of the phase per step (library figure, else the model)
        b = lib_bytes or phase_bytes(dominant, n, m, E)
        achieved = (b / (per_step_ms / 1e3) / 1e9) if b else None
        traffic, traffic_src = profiled_traffic(args.workload, args.algo, dominant)
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": achieved,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": (achieved / peaks["hbm_gbs"]) if achieved else None,
                    "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
                    "algorithmic_bytes_per_step": b, "kernel_ms_per_step": per_step_ms,
                    "phase_records_per_step": per_step_launches,
                    "unit_of_launch": "one build's worth of the phase (all its kernel launches)",
                    "share_of_step": per_step_ms / ms_per_step}
    b_alg = 4 * (n + 1) + 8 * m + 4 * n
    step_roofline = {"b_alg": b_alg, "achieved_gbs": b_alg / (ms_per_step / 1e3) / 1e9,
                     "frac_of_measured": b_alg / (ms_per_step / 1e3) / 1e9 / peaks["hbm_gbs"],
                     "frac_of_8tbs": b_alg / (ms_per_step / 1e3) / 8e12}

    # ---- e2e through the C ABI with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        eh = torch.from_numpy(np.ascontiguousarray(e_host.ravel())).pin_memory()
        ph = torch.empty(n, dtype=torch.int64).pin_memory()
        ge = P.DeviceGraph.generate("path:2", device=dev)
        ge.upload(n, eh.numpy())  # allocate once (workspace reuse)
        out_np = ph.numpy()
        ge.run(algo, root)  # warm the handle's workspace
        times = []
        for _ in range(max(3, min(args.steps, 5))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ge.upload(n, eh.numpy())
            ge.run(algo, root, out=out_np, want_roots=False, want_levels=False)
            times.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = statistics.median(times)
        if world > 1:  # the slowest rank (replicas run concurrently)
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": world * m / (e2e_ms / 1e3), "unit": "edges/s", "ms": e2e_ms,
               "h2d_bytes_per_step": int(eh.numel() * 8), "d2h_bytes_per_step": int(n * 8)}
        ge.close()

    # ---- in-run GPU BFS baseline on the same graph (north-star ratio) ----
    bfs = None
    if not args.no_bfs_ratio and algo != 0 and rank == 0:
        lv = torch.empty(n, dtype=torch.int32, device="cuda")
        g.run_device(0, root, d_parent.data_ptr(), lv.data_ptr())  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        stb = g.run_device(0, root, d_parent.data_ptr(), lv.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        bms = e0.elapsed_time(e1)
        bfs = {"bfs_ms": bms, "bfs_levels": stb["levels"],
               "us_per_level": 1e3 * bms / max(1, stb["levels"]),
               "speedup_vs_gpu_bfs": bms / ms_per_step}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference(args.workload, args.algo, 1, 1)  # ~30 s of host work on road
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # the checker is optional on the box
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ms_per_step_median": statistics.median(step_ms),
            "cold_first_build_ms": cold_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config, "n": n, "m": m, "valid": bool(valid),
            "roofline": roofline, "step_roofline": step_roofline, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": launches,
            "gpu_launches_source": "CUPTI kernel records of one untimed step x steps",
            "phases_source": "separate instrumented steps (not the timed ones)",
            "clocks": clk.summary(), "phases_ms_per_step": {k: [round(v[0], 4), v[1], v[2]] for k, v in agg.items()},
            "bfs_baseline": bfs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
