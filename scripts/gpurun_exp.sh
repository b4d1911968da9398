mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for W in road rmat24 path grid; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > gpurun_out/exp_$W.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/exp_$W.json'));print('$W', round(d['ms_per_step'],3), d['valid'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})" || tail -5 gpurun_out/exp_$W.json; done
