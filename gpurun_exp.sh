mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for W in road rmat24 path grid; do timeout 300 python bench.py --workload $W --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-bfs-ratio > gpurun_out/exp_$W.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/exp_$W.json'));print('$W', round(d['ms_per_step'],3), d['valid'], d['phases_ms_per_step'])" || tail -5 gpurun_out/exp_$W.json; done
timeout 600 python bench.py --workload kron28cc --steps 2 --warmup 1 > gpurun_out/exp_k28cc.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/exp_k28cc.json'));print('k28', round(d['ms_per_step'],3), d['value']/1e9)"
