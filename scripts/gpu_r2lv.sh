O=gpurun_out; mkdir -p $O
for S in 1 3; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:^k_tile_rank_w" -s $S -c 1 -o $O/prof_lv_s$S python scripts/profile_step.py --workload road > /dev/null 2>&1
python scripts/ncu_lines.py $O/prof_lv_s$S.ncu-rep --top 22 > $O/lines_lv_s$S.txt; head -24 $O/lines_lv_s$S.txt
ncu -i $O/prof_lv_s$S.ncu-rep --page details --csv > $O/prof_lv_s${S}_details.csv; rm -f $O/prof_lv_s$S.ncu-rep
done
