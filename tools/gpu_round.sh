# One GPU call: tests, bench line, ncu launch list + one full capture of the
# planner kernel.  Outputs land in gpurun_out/ (scratch; summaries are copied
# into profiles/ by hand).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt
nproc >> gpurun_out/gpu_${TAG}.txt
lscpu | grep -i "model name" >> gpurun_out/gpu_${TAG}.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1
timeout 600 python bench.py --workload lstm --steps 20 --warmup 5 --no-suite --no-replay > gpurun_out/bench_lstm_${TAG}.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-check --no-replay --no-suite \
  ${BENCH_ARGS} > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_plan -s 2 -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu --no-check --no-replay --no-suite \
  ${BENCH_ARGS} > gpurun_out/prof_${TAG}.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_${TAG}.log gpurun_out/smoke_${TAG}.log gpurun_out/bench_${TAG}.log \
  gpurun_out/prof_${TAG}.log
