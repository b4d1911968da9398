# Final-state evidence of a round: GPU suite, smoke, the reference acceptance
# binary, the default bench line (e2e + CPU baseline), the reference arm, every
# config x strategy bench line, ncu launch lists per kernel and per phase
# (NVTX) for road cc-euler / pr-rst / bfs, and --set full captures (stall
# summaries by source line) of the top cc-euler kernels.
#   gpurun --timeout 3600 -- 'bash scripts/gpu_profile_round.sh TAG'
TAG=${1:-r2}
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
lscpu | grep -E "^CPU\(s\)|Model name" >> $O/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 2400 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
  [ -x build/ref_acceptance ] && timeout 600 ./build/ref_acceptance > $O/ref_acceptance.log 2>&1; tail -2 $O/ref_acceptance.log
fi
timeout 900 python bench.py > $O/bench_road.json 2> $O/bench_road.err; tail -c 600 $O/bench_road.json; echo
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json; echo
for W in road grid path rmat24; do
  for A in cc-euler pr-rst bfs; do
    [ "$W$A" = "pathbfs" ] && continue  # 16.7M levels
    [ "$W$A" = "roadcc-euler" ] && continue
    timeout 300 python bench.py --workload $W --algo $A --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-bfs-ratio > $O/bench_${W}_${A}.json 2> $O/bench_${W}_${A}.err
    python -c "import json;d=json.load(open('$O/bench_${W}_${A}.json'));r=d['roofline'] or {};print('$W $A', round(d['ms_per_step'],3), r.get('kernel'), r.get('frac'))"
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum
for A in cc-euler pr-rst bfs; do
  B=2; [ $A = bfs ] && B=1
  timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/launches_road_$A.csv python scripts/profile_step.py --workload road --algo $A --builds $B > $O/ncu_launch_road_$A.log 2>&1
  python scripts/ncu_top.py $O/launches_road_$A.csv --builds $B --json $O/kernels_road_$A.json > $O/launches_road_${A}_summary.txt
  timeout 900 ncu --profile-from-start off --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none --csv \
    --log-file $O/phases_road_$A.csv python scripts/profile_step.py --workload road --algo $A --builds $B > $O/ncu_phase_road_$A.log 2>&1
  python scripts/ncu_top.py $O/phases_road_$A.csv --builds $B --json $O/phases_road__$A.json > $O/phases_road_${A}_summary.txt
  head -12 $O/launches_road_${A}_summary.txt
done
if [ -z "$SKIP_FULL" ]; then
  for K in $(python scripts/ncu_top.py $O/launches_road_cc-euler.csv --names --top ${NCU_TOP:-5} | tr '|' ' '); do
    timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:^${K}" -c 1 -o $O/prof_${TAG}_${K} python scripts/profile_step.py --workload road > $O/ncu_full_${K}.log 2>&1
    ncu -i $O/prof_${TAG}_${K}.ncu-rep --page details --csv > $O/prof_${TAG}_${K}_details.csv 2>/dev/null
    python scripts/ncu_lines.py $O/prof_${TAG}_${K}.ncu-rep --top 25 > $O/lines_${TAG}_${K}.txt 2>/dev/null
    rm -f $O/prof_${TAG}_${K}.ncu-rep
  done
fi
du -sh $O
