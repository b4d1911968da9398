# List-ranking parameter sweep on the road mesh (bench.py, device-timed).
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" -p no:cacheprovider > $O/pytest_quick.log 2>&1; tail -2 $O/pytest_quick.log
for cfg in "2 4 3" "1 4 3" "4 4 3" "1 5 3" "2 5 3" "2 3 3"; do
  set -- $cfg
  RSTG_LR_CHAINS=$1 RSTG_LR_LOGK0=$2 RSTG_LR_LOGK1=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/exp_$1_$2_$3.json 2>&1
  python -c "import json,sys;d=json.load(open('$O/exp_$1_$2_$3.json'));print('chains=$1 logk0=$2 logk1=$3', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})" || tail -3 $O/exp_$1_$2_$3.json
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/launches_road.csv python scripts/profile_step.py --workload road --builds 2 > $O/ncu_launch_road.log 2>&1
python scripts/ncu_top.py $O/launches_road.csv --builds 2 --json $O/kernels_road.json | tee $O/launches_road_summary.txt
