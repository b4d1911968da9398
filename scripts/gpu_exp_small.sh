O=gpurun_out; mkdir -p $O
for V in 0 1; do
  export RSTG_LR_SMALLTILES=$V
  for W in road path grid; do timeout 300 python bench.py --workload $W --steps 10 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_s$V.json; python -c "import json;d=json.load(open('$O/bench_${W}_s$V.json'));print('small=$V $W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items() if k.startswith('lr')})"; done
done
RSTG_LR_SMALLTILES=1 RSTG_LR_DEBUG=1 timeout 300 python scripts/timeline.py --workload road --builds 1 2>&1 | grep -E "level|lr.tiles" | head
RSTG_LR_SMALLTILES=1 timeout 300 python scripts/timeline.py --workload road --builds 2 2>/dev/null | sed -n 4,40p | grep -E "rank_w|expand"
RSTG_LR_SMALLTILES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "full_size or knobs or overflow" 2>&1 | tail -2
