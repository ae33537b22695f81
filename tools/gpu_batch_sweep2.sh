cd $GRAFT_REPO_ROOT
for T in 592 1184; do
for cfg in "MEMPLAN_NWARPS=1 MEMPLAN_TIER=0"; do
  echo "== T=$T $cfg"
  env $cfg timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-check --traces $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, 'Mblocks/s', d['ms_per_step'], 'ms', 'single', d['single_trace']['latency_ms'], 'engine', d['plan_info']['engine'])"
done
done
