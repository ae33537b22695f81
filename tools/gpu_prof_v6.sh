cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-v6}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan -c 1 -o gpurun_out/prof_${TAG}_u1e4 python tools/prof_big.py uniform 10000 1 > gpurun_out/ncu_${TAG}_u1e4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_plan -c 1 -o gpurun_out/prof_${TAG}_u1e5 python tools/prof_big.py uniform 100000 8 > gpurun_out/ncu_${TAG}_u1e5.log 2>&1
tail -2 gpurun_out/ncu_${TAG}_*.log
