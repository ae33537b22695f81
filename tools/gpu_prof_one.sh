# usage: TAG=.. FAM=uniform N=100000 NW=1 bash tools/gpu_prof_one.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_plan -c 1 -o gpurun_out/prof_${TAG}_${FAM}${N}_nw${NW} python tools/prof_big.py $FAM $N $NW > gpurun_out/ncu_${TAG}_${FAM}${N}_nw${NW}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}_${FAM}${N}_nw${NW}.log
