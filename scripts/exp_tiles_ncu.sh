# launch list of one road build with tile ranking + one full capture of k_tile_rank
O=gpurun_out; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for W in ${WORKLOADS:-road path}; do
RSTG_LR_TILES=1 timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
  --log-file $O/tl_launches_${W}.csv python scripts/profile_step.py --workload $W --builds 2 > $O/tl_ncu_${W}.log 2>&1
python scripts/ncu_top.py $O/tl_launches_${W}.csv --builds 2 > $O/tl_launches_${W}_summary.txt; head -30 $O/tl_launches_${W}_summary.txt
done
RSTG_LR_TILES=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:k_tile_rank -c 1 -o $O/tl_prof python scripts/profile_step.py --workload road --builds 1 > $O/tl_prof.log 2>&1
ncu -i $O/tl_prof.ncu-rep --page details --csv > $O/tl_prof_details.csv 2>&1
ncu -i $O/tl_prof.ncu-rep --page source --csv > $O/tl_prof_source.csv 2>&1
ls -la $O/tl_prof*
