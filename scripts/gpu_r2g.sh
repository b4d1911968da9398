O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "bfs or golden or small or random or full_size_configs or two_tri or isolated or tiebreak or handle or determinism" > $O/pytest_g.log 2>&1; echo "pytest rc=$?" >> $O/pytest_g.log; tail -3 $O/pytest_g.log
for W in road grid rmat24; do timeout 300 python bench.py --workload $W --algo bfs --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_bfs.json; python -c "import json;d=json.load(open('$O/bench_${W}_bfs.json'));print('$W bfs', round(d['ms_per_step'],3), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"; done
timeout 300 python scripts/timeline.py --workload road --algo bfs --builds 1 2>/dev/null | head -12
