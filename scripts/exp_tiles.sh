# tile-contraction ranking vs the ruling-set walk (RSTG_LR_TILES, RSTG_LR_TILESLOTS)
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/ -x -q -m gpu -k "not full_size" -p no:cacheprovider > $O/pytest_full.log 2>&1; tail -3 $O/pytest_full.log
run() { # tag env...
  tag=$1; shift
  for W in ${WORKLOADS:-road rmat24 path grid}; do
    env "$@" timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/b_${W}_$tag.json 2> $O/b_${W}_$tag.err
    python -c "import json;d=json.load(open('$O/b_${W}_$tag.json'));print('$tag $W', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items() if k.startswith('lr') or k.startswith('euler')})" || tail -3 $O/b_${W}_$tag.err
  done
}
RSTG_LR_DEBUG=1 python bench.py --workload road --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>&1 >/dev/null | grep "tile0" | tail -7
run auto RSTG_NOTHING=1
