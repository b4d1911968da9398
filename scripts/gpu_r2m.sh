# round-2 call m: batched loads in k_euler_fix / k_tile_resolve, tail exits
# resolved by the level-2 kernel; parity + road bench + timeline
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "overflow or full_size or golden or random or small or handle or knobs or determinism or step_counts or euler or validator or two_tri or isolated or medium" > $O/pytest_m.log 2>&1; echo "pytest rc=$?" >> $O/pytest_m.log; tail -2 $O/pytest_m.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_road_m.json 2> $O/bench_road_m.err; python -c "
import json;d=json.load(open('$O/bench_road_m.json'));print('road', round(d['ms_per_step'],4), d['bfs_baseline'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
for W in rmat24 grid path; do timeout 300 python bench.py --workload $W --steps 5 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_m.json; python -c "import json;d=json.load(open('$O/bench_${W}_m.json'));print('$W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"; done
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 > $O/timeline_road_cc_m.txt 2>&1; head -24 $O/timeline_road_cc_m.txt | tail -21
