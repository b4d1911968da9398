# Full GPU test suite + bench lines for every BASELINE config/strategy (no ncu).
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
for W in road grid path rmat24; do
  for A in cc-euler pr-rst bfs; do
    [ "$W$A" = "pathbfs" ] && continue
    timeout 300 python bench.py --workload $W --algo $A --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_${W}_${A}.json 2> $O/bench_${W}_${A}.err
    python -c "import json;d=json.load(open('$O/bench_${W}_${A}.json'));print('$W $A', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})" || tail -3 $O/bench_${W}_${A}.err
  done
done
