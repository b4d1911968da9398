# round-2 re-entry call i: full GPU suite + default bench + per-strategy benches + smoke
O=gpurun_out; mkdir -p $O
nproc > $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 2400 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 3000 $O/bench_default.json
for W in road grid rmat24 path; do for A in bfs pr-rst; do [ "$W$A" = "pathbfs" ] && continue; timeout 300 python bench.py --workload $W --algo $A --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_$A.json; python -c "import json;d=json.load(open('$O/bench_${W}_$A.json'));print('$W $A', round(d['ms_per_step'],3), d.get('roofline',{}).get('frac'), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"; done; done
