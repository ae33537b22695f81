cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-v2}
for tr in cnn_1e4 uniform_1e4; do
ncu --set full --clock-control none --import-source on -k regex:k_plan -c 1 -o gpurun_out/prof_${TAG}_$tr python tools/prof_plan.py $tr 1 > gpurun_out/ncu_log_$tr.txt 2>&1
done
tail -2 gpurun_out/ncu_log_*.txt
