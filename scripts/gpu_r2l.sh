# round-2 call l: parity of the sync/memset removal, road bench + timeline,
# ncu --set full with source for the top cc-euler kernels (source pages as CSV)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "full_size or golden or random or small or handle or overflow or knobs or determinism or step_counts or distcc or euler" > $O/pytest_l.log 2>&1; echo "pytest rc=$?" >> $O/pytest_l.log; tail -2 $O/pytest_l.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_road_l.json 2> $O/bench_road_l.err; python -c "
import json;d=json.load(open('$O/bench_road_l.json'));print('road', round(d['ms_per_step'],4), d['cold_first_build_ms'], d['bfs_baseline'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 > $O/timeline_road_cc_l.txt 2>&1; head -24 $O/timeline_road_cc_l.txt | tail -21
for K in k_tile_rank k_tile_resolve k_euler_fix k_jump_x; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:^${K}" -c 1 -o $O/prof_r2l_${K} python scripts/profile_step.py --workload road > $O/ncu_full_${K}.log 2>&1
  ncu -i $O/prof_r2l_${K}.ncu-rep --page source --csv > $O/prof_r2l_${K}_source.csv 2>/dev/null
  ncu -i $O/prof_r2l_${K}.ncu-rep --page details --csv > $O/prof_r2l_${K}_details.csv 2>/dev/null
  ls -la $O/prof_r2l_${K}*
done
bash scripts/sanitize.sh
