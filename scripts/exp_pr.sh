O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" -p no:cacheprovider > $O/pytest_quick.log 2>&1; tail -1 $O/pytest_quick.log
for W in road path grid rmat24; do
  timeout 300 python bench.py --workload $W --algo pr-rst --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/pr_$W.json 2> $O/pr_$W.err
  python -c "import json;d=json.load(open('$O/pr_$W.json'));print('pr $W', round(d['ms_per_step'],3), d['valid'], {k:round(v[0],3) for k,v in d['phases_ms_per_step'].items()})" || tail -3 $O/pr_$W.err
done
