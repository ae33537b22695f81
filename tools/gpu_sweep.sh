cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/nw_sweep.py 100000 1,4,8,16
timeout 300 python tools/nw_sweep.py 10000 1,4
