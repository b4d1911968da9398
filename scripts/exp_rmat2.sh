O=gpurun_out; mkdir -p $O
for k in 4 5 3; do
RSTG_LR_DEBUG=1 RSTG_LR_LOGK0=$k timeout 300 python bench.py --workload rmat24 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/r_$k.json 2> $O/r_$k.err
python -c "import json;d=json.load(open('$O/r_$k.json'));print('logk0=$k', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
tail -4 $O/r_$k.err
done
