cd $GRAFT_REPO_ROOT
nproc
timeout 300 python bench.py --n 10000 --traces 148 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -3
