mkdir -p gpurun_out
python tools/small_lat.py > gpurun_out/sl_$TAG.log 2>&1
python -m pytest tests/test_fuzz_gpu.py -x -q > gpurun_out/t_$TAG.log 2>&1; tail -1 gpurun_out/t_$TAG.log
head -4 gpurun_out/sl_$TAG.log
