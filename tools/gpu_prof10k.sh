cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tr in cnn uniform; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_plan -c 1 -o gpurun_out/prof_v4_${tr}1e4 python tools/prof_big.py $tr 10000 1 > gpurun_out/ncu_v4_$tr.log 2>&1
done
tail -1 gpurun_out/ncu_v4_*.log
