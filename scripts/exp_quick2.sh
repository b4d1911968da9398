# road/path/grid bench lines + tile-rank kernel times from an ncu launch list
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" -p no:cacheprovider > $O/pytest_quick.log 2>&1; tail -1 $O/pytest_quick.log
for W in ${WORKLOADS:-road path grid}; do
  timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/q_$W.json 2> $O/q_$W.err
  python -c "import json;d=json.load(open('$O/q_$W.json'));print('$W', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items() if k.startswith('lr') or k.startswith('euler')})" || tail -3 $O/q_$W.err
done
M=gpu__time_duration.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
  --log-file $O/q_launches.csv python scripts/profile_step.py --workload road --builds 2 > /dev/null 2>&1
python scripts/ncu_top.py $O/q_launches.csv --builds 2 > $O/q_launches.txt; head -12 $O/q_launches.txt
