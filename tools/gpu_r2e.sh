#!/bin/bash
mkdir -p gpurun_out
PEARL_LIB_PATH=build/var_tl/libpearl_tl.so timeout 200 python tools/draft_timeline.py llama-68m 192 > gpurun_out/draft_timeline.log 2>&1
timeout 200 python tools/draft_times.py llama-68m > gpurun_out/draft_times.log 2>&1
for M in 1 16; do
  PEARL_LIB_PATH=build/var_tl/libpearl_tl.so timeout 200 python tools/timeline.py llama2-7b $M 192 > gpurun_out/timeline_M$M.log 2>&1
done
timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16 192 > gpurun_out/fwd_default.log 2>&1
PEARL_LIB_PATH=build/var_r90/libpearl_r90.so timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16 192 > gpurun_out/fwd_r90.log 2>&1
bash tools/ablate.sh > gpurun_out/ablate.log 2>&1
timeout 600 python -m pytest tests/test_llama_gpu.py tests/test_green_partition_gpu.py tests/test_long_decode_gpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log
