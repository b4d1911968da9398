O=gpurun_out; mkdir -p $O
for V in default exphook_4_8 exphook_4_6; do
  if [ $V != default ]; then export RSTG_LIB_PATH=build/$V/librstg.so; fi
  for W in rmat24 road; do timeout 300 python bench.py --workload $W --steps 5 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_$V.json; python -c "import json;d=json.load(open('$O/bench_${W}_$V.json'));print('$V $W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items() if 'hook' in k})"; done
  timeout 300 python bench.py --workload rmat24 --algo pr-rst --steps 3 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_rmatpr_$V.json; python -c "import json;d=json.load(open('$O/bench_rmatpr_$V.json'));print('$V rmat pr', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items() if 'graft' in k})"
done
