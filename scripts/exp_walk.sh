# level-0 walk parameter sweep (road, device-timed phases), 2 repeats each
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for cfg in "8 64 4 3" "4 64 4 3" "6 64 4 3" "3 64 4 3" "4 32 4 3" "4 128 4 3" "4 64 5 3" "6 64 5 3" "4 64 4 4" "4 64 4 2"; do
  set -- $cfg
  RSTG_LR_BLOCKS=$1 RSTG_LR_CHUNK=$2 RSTG_LR_LOGK0=$3 RSTG_LR_LOGK1=$4 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/w.json 2>&1
  python -c "import json;d=json.load(open('$O/w.json'));p=d['phases_ms_per_step'];print('blocks=$1 chunk=$2 logk0=$3 logk1=$4', round(d['ms_per_step'],3), d['valid'], 'walk', p['lr.walk'][0], 'rank', p['lr.rulers_rank'][0])" || tail -3 $O/w.json
done
done
