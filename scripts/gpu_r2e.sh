O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_loader.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "load or smoke or small_generators or golden" > $O/pytest_e.log 2>&1; echo "pytest rc=$?" >> $O/pytest_e.log; tail -3 $O/pytest_e.log
python -c "
import paper_2603_11645_b200 as P, ctypes
" 
for A in pr-rst bfs; do timeout 600 python scripts/timeline.py --workload road --algo $A --builds 1 > $O/timeline_road_$A.txt 2>&1; head -1 $O/timeline_road_$A.txt; done
RSTG_BFS_SMALL=0 timeout 300 python bench.py --workload grid --algo bfs --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_grid_bfs_nosmall.json 2>&1; python -c "import json;print('grid bfs no-small', json.load(open('$O/bench_grid_bfs_nosmall.json'))['ms_per_step'])"
timeout 300 python bench.py --workload grid --algo bfs --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_grid_bfs_small.json 2>&1; python -c "import json;print('grid bfs small', json.load(open('$O/bench_grid_bfs_small.json'))['ms_per_step'])"
