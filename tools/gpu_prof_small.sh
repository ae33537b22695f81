cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-v6}
for fam in ${FAMS:-cnn uniform}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan -c 1 -o gpurun_out/prof_${TAG}_${fam}1e4 python tools/prof_big.py $fam 10000 1 > gpurun_out/ncu_${TAG}_${fam}1e4.log 2>&1
done
ls gpurun_out
