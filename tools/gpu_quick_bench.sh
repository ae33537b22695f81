cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/lat_sweep.py ${LAT_SIZES:-10000,100000} 1 2>&1
for T in ${TRACES:-2368}; do
  echo "== T=$T $CFG"
  env $CFG timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-check --no-replay --no-suite --traces $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'Mblocks/s', round(d['ms_per_step'],1), 'ms', 'e2e', round(d['e2e']['value']/1e6,2), 'single', round(d['single_trace']['latency_ms'],1), 'engine', d['plan_info']['engine'])"
done
