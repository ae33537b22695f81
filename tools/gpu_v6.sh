cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-v6}
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -15 gpurun_out/pytest_${TAG}.log
timeout 600 python tools/lat_sweep.py 10000,100000 1,8 2>&1 | tee gpurun_out/lat_${TAG}.log
