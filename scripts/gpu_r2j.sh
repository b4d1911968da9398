# round-2 call j: kernel timeline of road cc-euler at HEAD, ncu launch lists
# (time, DRAM, L2 hit rate, L2 atomic/reduction sectors) for road cc-euler, pr-rst, bfs
O=gpurun_out; mkdir -p $O
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 > $O/timeline_road_cc.txt 2>&1; head -30 $O/timeline_road_cc.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum
for A in cc-euler pr-rst bfs; do
  timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/launches_road_$A.csv python scripts/profile_step.py --workload road --algo $A --builds 1 > $O/ncu_launch_road_$A.log 2>&1
  echo "ncu $A rc=$?"
  python scripts/ncu_top.py $O/launches_road_$A.csv --builds 1 --json $O/kernels_road_$A.json > $O/launches_road_${A}_summary.txt 2>&1
  head -25 $O/launches_road_${A}_summary.txt
done
