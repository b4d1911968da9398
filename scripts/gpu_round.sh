# One gpurun session: GPU tests, bench lines, launch lists and one ncu full
# capture of the top kernels. Keeps gpurun_out/ small (< 64 MiB): the full
# capture is exported to CSV on the box and the .ncu-rep kept only if small.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh [TAG]'
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
lscpu | grep -E "^CPU\(s\)|Model name" >> $O/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -3 $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
  [ -x build/rst_acceptance ] && timeout 600 ./build/rst_acceptance > $O/acceptance.log 2>&1; tail -1 $O/acceptance.log
fi
timeout 900 python bench.py > $O/bench_road.json 2> $O/bench_road.err; cat $O/bench_road.json
if [ -z "$SKIP_EXTRA" ]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; cat $O/bench_ref.json
  for W in grid path rmat24; do
    for A in cc-euler pr-rst bfs; do
      [ "$W$A" = "pathbfs" ] && continue  # 16.7M levels: ~minutes per build
      timeout 300 python bench.py --workload $W --algo $A --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_${W}_${A}.json 2> $O/bench_${W}_${A}.err
    done
  done
  for A in pr-rst bfs; do
    timeout 300 python bench.py --algo $A --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_road_${A}.json 2> $O/bench_road_${A}.err
  done
fi
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for W in ${NCU_WORKLOADS:-road}; do
  # per kernel, then per phase (NVTX ranges of the phase timer), 2 builds each
  timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/launches_${W}.csv python scripts/profile_step.py --workload $W --builds 2 > $O/ncu_launch_${W}.log 2>&1
  python scripts/ncu_top.py $O/launches_${W}.csv --builds 2 --json $O/kernels_${W}.json > $O/launches_${W}_summary.txt
  timeout 600 ncu --profile-from-start off --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none --csv \
    --log-file $O/phases_${W}.csv python scripts/profile_step.py --workload $W --builds 2 > $O/ncu_phase_${W}.log 2>&1
  python scripts/ncu_top.py $O/phases_${W}.csv --builds 2 --json $O/phases_${W}.json > $O/phases_${W}_summary.txt
  cat $O/launches_${W}_summary.txt $O/phases_${W}_summary.txt
done
if [ -z "$SKIP_FULL" ]; then
  # one --set full capture per top kernel (first launch inside the profiled build)
  for K in $(python scripts/ncu_top.py $O/launches_road.csv --names --top ${NCU_TOP:-5} | tr '|' ' '); do
    timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:^${K}" -c 1 -o $O/prof_${TAG}_${K} python scripts/profile_step.py --workload road > $O/ncu_full_${K}.log 2>&1
    ncu -i $O/prof_${TAG}_${K}.ncu-rep --page raw --csv > $O/prof_${TAG}_${K}_raw.csv 2>/dev/null
    ncu -i $O/prof_${TAG}_${K}.ncu-rep --page details --csv > $O/prof_${TAG}_${K}_details.csv 2>/dev/null
    sz=$(stat -c %s $O/prof_${TAG}_${K}.ncu-rep 2>/dev/null || echo 0)
    if [ "$sz" -gt 12000000 ]; then rm -f $O/prof_${TAG}_${K}.ncu-rep; echo "ncu-rep $K too large ($sz), removed"; fi
  done
fi
du -sh $O
