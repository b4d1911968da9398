# compute-sanitizer evidence (race detection): memcheck,
# racecheck (shared memory), synccheck and initcheck over small runs of
# every strategy (scripts/sanitize.py). Logs -> gpurun_out/sanitize_<tool>.log
O=gpurun_out; mkdir -p $O
for T in memcheck racecheck synccheck initcheck; do
  EXTRA=""
  [ "$T" = "memcheck" ] && EXTRA="--leak-check full"
  # analysis: one report per racing source-line pair (not per thread)
  [ "$T" = "racecheck" ] && EXTRA="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $T $EXTRA --error-exitcode 99 --print-limit 400 \
    python scripts/sanitize.py > $O/sanitize_$T.log 2>&1
  echo "$T rc=$?" | tee -a $O/sanitize_$T.log
  tail -4 $O/sanitize_$T.log
done
# racecheck: the kernels and source lines reported
grep -E "^=========     (at|Write|Read)" $O/sanitize_racecheck.log | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -40 > $O/sanitize_racecheck_summary.txt
cat $O/sanitize_racecheck_summary.txt
