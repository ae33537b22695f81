set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 600 python -m pytest tests/test_plan_gpu.py -x -q -s 2>&1 | tail -30
