# round-2 call o: fewer launches around the Euler pass and round 0 (xbits kept
# zero between passes, counters zeroed by kernels, async flag copy after the
# orientation); parity + benches + timeline; loader throughput vs the reference
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_loader.py -x -q -m gpu -p no:cacheprovider -k "overflow or full_size or golden or random or small or handle or knobs or determinism or step_counts or euler or validator or two_tri or isolated or medium or distcc or load" > $O/pytest_o.log 2>&1; echo "pytest rc=$?" >> $O/pytest_o.log; tail -2 $O/pytest_o.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_road_o.json 2> $O/bench_road_o.err; python -c "
import json;d=json.load(open('$O/bench_road_o.json'));print('road', round(d['ms_per_step'],4), d['bfs_baseline'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 > $O/timeline_road_cc_o.txt 2>&1; sed -n 4,24p $O/timeline_road_cc_o.txt
timeout 1200 python scripts/bench_loader.py --ref --json $O/loader_road.json > $O/loader_road.log 2>&1; tail -2 $O/loader_road.log
