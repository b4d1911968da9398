# full GPU suite, smoke, the reference acceptance binary and the default bench line
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_final.log; tail -2 $O/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
[ -x build/ref_acceptance ] && timeout 600 ./build/ref_acceptance 2>&1 | tail -1
timeout 900 python bench.py > $O/bench_final.json 2> $O/bench_final.err; python -c "
import json;d=json.load(open('$O/bench_final.json'));print('road', round(d['ms_per_step'],4), round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,3), 'bfs x', round(d['bfs_baseline']['speedup_vs_gpu_bfs'],1), 'frac', round(d['roofline']['frac'],3), d['clocks']['reasons'])"
