cd $GRAFT_REPO_ROOT
for T in 2368 4144; do
  echo "== T=$T"
  timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-check --traces $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'Mblocks/s', round(d['ms_per_step'],1), 'ms', 'e2e', round(d['e2e']['value']/1e6,2), 'engine', d['plan_info']['engine'])"
done
