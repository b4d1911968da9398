# round-2 call k: road bench after the vtail restore, sanitizer logs, Kron-28
# verification record, reference arm with 1 worker (road:4899)
O=gpurun_out; mkdir -p $O
nproc > $O/nproc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_road_k.json 2> $O/bench_road_k.err; python -c "
import json;d=json.load(open('$O/bench_road_k.json'));print('road', round(d['ms_per_step'],4), d['cold_first_build_ms'], d['bfs_baseline'], {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "full_size or golden or random or small or handle or euler" > $O/pytest_k.log 2>&1; echo "pytest rc=$?" >> $O/pytest_k.log; tail -2 $O/pytest_k.log
bash scripts/sanitize.sh
timeout 1500 python scripts/verify_kron28.py --scale 28 --ranks 2 --out $O/kron28_verify.json > $O/kron28_verify.log 2>&1; echo "verify rc=$?"; tail -3 $O/kron28_verify.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 --ref-workers 1 > $O/bench_ref_1worker.json 2> $O/bench_ref_1worker.err; cat $O/bench_ref_1worker.json
