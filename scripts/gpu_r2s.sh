# round-2 call q: round-0 exit-target dedup after compaction; parity + benches
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "full_size or golden or random or small or handle or medium or distcc or two_tri or isolated" > $O/pytest_q.log 2>&1; echo "pytest rc=$?" >> $O/pytest_q.log; tail -2 $O/pytest_q.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-bfs-ratio > $O/bench_road_q.json 2> $O/bench_road_q.err; python -c "
import json;d=json.load(open('$O/bench_road_q.json'));print('road', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
for W in rmat24 path grid; do timeout 300 python bench.py --workload $W --steps 5 --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/bench_${W}_q.json; python -c "import json;d=json.load(open('$O/bench_${W}_q.json'));print('$W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"; done
timeout 300 python scripts/timeline.py --workload road --algo cc-euler --builds 3 > $O/timeline_road_cc_q.txt 2>&1; sed -n 4,12p $O/timeline_road_cc_q.txt
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
