# quick tests + default bench + launch list + full captures of named kernels
#   KERNELS="k_walk0 k_tile_resolve" bash scripts/exp_full.sh TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" -p no:cacheprovider > $O/pytest_quick.log 2>&1; tail -2 $O/pytest_quick.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_quick.json 2>&1
python -c "import json;d=json.load(open('$O/bench_quick.json'));print(round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})" || tail -3 $O/bench_quick.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/launches_road.csv python scripts/profile_step.py --workload road --builds 2 > $O/ncu_launch_road.log 2>&1
python scripts/ncu_top.py $O/launches_road.csv --builds 2 --json $O/kernels_road.json | tee $O/launches_road_summary.txt
for K in ${KERNELS:-k_walk0}; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:^${K}" -c 1 -o $O/prof_${TAG}_${K} python scripts/profile_step.py --workload road > $O/ncu_full_${K}.log 2>&1
  ncu -i $O/prof_${TAG}_${K}.ncu-rep --page raw --csv > $O/prof_${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i $O/prof_${TAG}_${K}.ncu-rep --page details --csv > $O/prof_${TAG}_${K}_details.csv 2>/dev/null
  ncu -i $O/prof_${TAG}_${K}.ncu-rep --page source --csv > $O/prof_${TAG}_${K}_source.csv 2>/dev/null
  rm -f $O/prof_${TAG}_${K}.ncu-rep
done
du -sh $O
