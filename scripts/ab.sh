# A/B experiment driver (under gpurun): bench lines for each variant, where a
# variant is a set of environment assignments -- knobs (RSTG_*), or an
# alternative build of the library (RSTG_LIB_PATH=build/<dir>/librstg.so,
# e.g. compiled with -DRSTG_JUMP_HOPS=8). Each variant runs every workload.
#   gpurun -- 'bash scripts/ab.sh "RSTG_CC_TAIL=1" "RSTG_CC_TAIL=0" -- road rmat24'
#   ALGO=pr-rst STEPS=5 bash scripts/ab.sh ...
O=gpurun_out; mkdir -p $O
variants=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do variants+=("$1"); shift; done
shift
workloads=("$@"); [ ${#workloads[@]} -eq 0 ] && workloads=(road)
i=0
for V in "${variants[@]}"; do
  for W in "${workloads[@]}"; do
    env $V timeout 300 python bench.py --workload $W --algo ${ALGO:-cc-euler} --steps ${STEPS:-10} \
      --no-e2e --no-cpu-baseline --no-bfs-ratio 2>/dev/null | tail -1 > $O/ab_${i}_$W.json
    python -c "import json;d=json.load(open('$O/ab_${i}_$W.json'));print('[$V] $W', round(d['ms_per_step'],4), {k:v[0] for k,v in d['phases_ms_per_step'].items()})"
  done
  i=$((i+1))
done
