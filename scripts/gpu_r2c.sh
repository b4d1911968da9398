O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 1200 python scripts/verify_kron28.py --scale 28 --ranks 2 --out $O/kron28_verify.json > $O/kron28_verify.log 2>&1; echo "verify rc=$?"; tail -1 $O/kron28_verify.log
timeout 900 python bench.py --workload kron28cc --steps 3 --warmup 1 > $O/bench_kron28cc.json 2> $O/bench_kron28cc.err; cat $O/bench_kron28cc.json
for W in road rmat24; do timeout 300 python scripts/timeline.py --workload $W --json $O/timeline_$W.json > $O/timeline_$W.txt 2>&1; head -1 $O/timeline_$W.txt; done
