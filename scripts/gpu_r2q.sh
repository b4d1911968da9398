# round-2 call q: round-0 exit-target dedup after compaction; parity + benches
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "full_size or golden or random or small or handle or medium or distcc or two_tri or isolated" > $O/pytest_q.log 2>&1; echo "pytest rc=$?" >> $O/pytest_q.log; tail -2 $O/pytest_q.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-bfs-ratio > $O/bench_road_q.json 2> $O/bench_road_q.err; python -c "
import json;d=json.load(open('$O/bench_road_q.json'));print('road', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
for W in rmat24 path grid; do timeout 300 python bench.py --workload $W --steps 5 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_q.json; python -c "import json;d=json.load(open('$O/bench_${W}_q.json'));print('$W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"; done
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 > $O/timeline_road_cc_q.txt 2>&1; sed -n 4,12p $O/timeline_road_cc_q.txt
