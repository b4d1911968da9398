# quick parity + a bench line per workload (device-timed phases)
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" -p no:cacheprovider > $O/pytest_quick.log 2>&1; tail -2 $O/pytest_quick.log
for W in ${WORKLOADS:-road rmat24 path grid}; do
timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/b_$W.json 2> $O/b_$W.err
python -c "import json;d=json.load(open('$O/b_$W.json'));print('$W', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})" || tail -3 $O/b_$W.err
done
