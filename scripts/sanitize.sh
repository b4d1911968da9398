# compute-sanitizer evidence (race detection): memcheck,
# racecheck (shared memory), synccheck and initcheck over small runs of
# every strategy (scripts/sanitize.py). Logs -> gpurun_out/sanitize_<tool>.log
O=gpurun_out; mkdir -p $O
for T in memcheck racecheck synccheck initcheck; do
  EXTRA=""
  [ "$T" = "memcheck" ] && EXTRA="--leak-check full"
  [ "$T" = "racecheck" ] && EXTRA="--racecheck-report all"
  [ "$T" = "initcheck" ] && EXTRA="--track-unused-memory no"
  timeout 1500 compute-sanitizer --tool $T $EXTRA --error-exitcode 99 --print-limit 50 \
    python scripts/sanitize.py > $O/sanitize_$T.log 2>&1
  echo "$T rc=$?" | tee -a $O/sanitize_$T.log
  tail -4 $O/sanitize_$T.log
done
