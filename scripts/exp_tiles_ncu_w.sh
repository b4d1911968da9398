O=gpurun_out; mkdir -p $O
RSTG_LR_TILES=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:k_tile_rank_w --launch-skip ${SKIP:-0} -c 1 -o $O/tlw_prof python scripts/profile_step.py --workload road --builds 1 > $O/tlw_prof.log 2>&1
ncu -i $O/tlw_prof.ncu-rep --page details --csv > $O/tlw_prof_details.csv 2>&1
ncu -i $O/tlw_prof.ncu-rep --page source --csv > $O/tlw_prof_source.csv 2>&1
rm -f $O/tlw_prof.ncu-rep
