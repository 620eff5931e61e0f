#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16,20,32,64 192 > gpurun_out/fwd_default.log 2>&1
for M in 16 20; do PEARL_LIB_PATH=build/var_tl/libpearl_tl.so timeout 200 python tools/timeline.py llama2-7b $M 192 > gpurun_out/timeline_M$M.log 2>&1; done
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py tests/test_parity_shapes_gpu.py tests/test_batched_gpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log
