O=gpurun_out; mkdir -p $O
for V in default exp16k; do
  if [ $V = exp16k ]; then export RSTG_LIB_PATH=build/exp16k/librstg.so; fi
  for W in road path rmat24; do timeout 300 python bench.py --workload $W --steps 10 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_$V.json; python -c "import json;d=json.load(open('$O/bench_${W}_$V.json'));print('$V $W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items() if k.startswith('cc')})"; done
done
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 2>/dev/null | sed -n 4,10p
