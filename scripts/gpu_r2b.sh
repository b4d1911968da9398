# round-2 call b: new GPU tests, Kron-28 verification, same-config reference arm, kron CC bench
O=gpurun_out; mkdir -p $O
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider -k "distcc or euler_structure or reference_acceptance or reference_digests or edge_upload or unconsumed or error_order or verification_script or handle_reuse or forest_depth or euler_root_forest" > $O/pytest_new.log 2>&1; echo "pytest rc=$?" >> $O/pytest_new.log; tail -5 $O/pytest_new.log
timeout 1200 python scripts/verify_kron28.py --scale 28 --ranks 2 --out $O/kron28_verify.json > $O/kron28_verify.log 2>&1; echo "verify rc=$?"; tail -2 $O/kron28_verify.log
timeout 900 python bench.py --workload kron28cc --steps 3 --warmup 1 > $O/bench_kron28cc.json 2> $O/bench_kron28cc.err; cat $O/bench_kron28cc.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; cat $O/bench_ref.json
