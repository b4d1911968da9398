# round-2 call r: RMAT-24 hook rounds -- per-round stats and an ncu capture of the hooks
O=gpurun_out; mkdir -p $O
RSTG_CC_DEBUG=1 timeout 300 python scripts/profile_step.py --workload rmat24 --builds 1 --warmup 1 > $O/rmat_ccdebug.txt 2>&1; grep "cc round" $O/rmat_ccdebug.txt | tail -8
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_rmat24.csv python scripts/profile_step.py --workload rmat24 --builds 1 > /dev/null 2>&1
python scripts/ncu_top.py $O/launches_rmat24.csv --builds 1 > $O/launches_rmat24_summary.txt; head -16 $O/launches_rmat24_summary.txt
python - <<'PY'
import csv,collections
rows=[l for l in open('gpurun_out/launches_rmat24.csv') if l.startswith('"')]
per=collections.OrderedDict()
for r in csv.DictReader(rows):
    d=per.setdefault(r["ID"],{"name":r["Kernel Name"][:40]})
    d[r["Metric Name"]]=r["Metric Value"]
for k,d in per.items():
    if "k_hook" in d["name"]: print(d["name"], d.get("gpu__time_duration.sum"), d.get("dram__bytes_read.sum"), d.get("lts__t_sector_hit_rate.pct"), d.get("lts__t_sectors_op_atom.sum"))
PY
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:^k_hook" -c 1 -o $O/prof_r2r_k_hook_rmat python scripts/profile_step.py --workload rmat24 > /dev/null 2>&1
python scripts/ncu_lines.py $O/prof_r2r_k_hook_rmat.ncu-rep --top 20 > $O/lines_r2r_k_hook_rmat.txt; cat $O/lines_r2r_k_hook_rmat.txt
ncu -i $O/prof_r2r_k_hook_rmat.ncu-rep --page details --csv > $O/prof_r2r_k_hook_rmat_details.csv
