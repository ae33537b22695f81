cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 600 python -m pytest tests/test_plan_gpu.py -x -q 2>&1 | tail -5
python tools/prof_plan.py cnn_1e4 3
python tools/prof_plan.py uniform_1e4 3
python tools/prof_plan.py walk_1e4 3
python tools/prof_plan.py cnn_1e4 2 4
python tools/prof_plan.py uniform_1e4 2 4
