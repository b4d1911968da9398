# round-2 call p: full GPU suite after the PR-RST buffer sizing fix + PR bench
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu_p.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_p.log; tail -2 $O/pytest_gpu_p.log
timeout 300 python bench.py --algo pr-rst --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_road_pr_p.json; python -c "import json;d=json.load(open('$O/bench_road_pr_p.json'));print('road pr', round(d['ms_per_step'],3), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
