O=gpurun_out; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in 4 3; do
RSTG_LR_LOGK0=$k timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/l_$k.csv python scripts/profile_step.py --workload rmat24 --builds 1 > $O/l_$k.log 2>&1
python scripts/ncu_top.py $O/l_$k.csv --builds 1 | head -24
done
