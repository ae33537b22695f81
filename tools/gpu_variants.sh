# A/B of library builds under tools/_variants/<name>/ on the batched bench.
#   VARIANTS="mb1 mb16" TRACES="1184 2368" bash tools/gpu_variants.sh
cd $GRAFT_REPO_ROOT
for V in ${VARIANTS:-mb1}; do
  for T in ${TRACES:-2368}; do
    C=$(( (T + 147) / 148 ))
    echo "== $V T=$T conc=$C"
    MEMPLAN_LIB=tools/_variants/$V/libmemplan_b200.so MEMPLAN_CONC=$C timeout 900 \
      python bench.py --steps 2 --warmup 3 --no-cpu --no-check --no-replay --no-suite --traces $T 2>&1 \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'Mblocks/s', round(d['ms_per_step'],1), 'ms', 'single', round(d['single_trace']['latency_ms'],1), 'engine', d['plan_info']['engine'])"
  done
done
