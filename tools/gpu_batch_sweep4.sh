cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/lat_sweep.py 10000,100000 1 2>&1
for T in 1184; do
for cfg in "MEMPLAN_X=0" "MEMPLAN_TIER=0"; do
  echo "== T=$T $cfg"
  env $cfg timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-check --traces $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'Mblocks/s', round(d['ms_per_step'],1), 'ms', 'single', round(d['single_trace']['latency_ms'],1), 'engine', d['plan_info']['engine'])"
done
done
