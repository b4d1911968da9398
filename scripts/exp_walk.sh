# level-0 walk parameter sweep (road, device-timed phases)
O=gpurun_out; mkdir -p $O
for cfg in "8 64 4" "4 64 4" "2 64 4" "8 16 4" "8 256 4" "8 1024 4" "8 64 5" "4 64 5"; do
  set -- $cfg
  RSTG_LR_BLOCKS=$1 RSTG_LR_CHUNK=$2 RSTG_LR_LOGK0=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/w_$1_$2_$3.json 2>&1
  python -c "import json;d=json.load(open('$O/w_$1_$2_$3.json'));p=d['phases_ms_per_step'];print('blocks=$1 chunk=$2 logk0=$3', round(d['ms_per_step'],3), d['valid'], 'walk', p['lr.walk'][0], 'rank', p['lr.rulers_rank'][0])" || tail -3 $O/w_$1_$2_$3.json
done
