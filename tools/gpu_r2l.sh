#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/gemm_m_sweep.py > gpurun_out/gemm_m_sweep.log 2>&1
timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16,32,64,128 192 > gpurun_out/fwd_default.log 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py tests/test_parity_shapes_gpu.py tests/test_batched_gpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log
PEARL_LIB_PATH=build/var_tl/libpearl_tl.so timeout 200 python tools/timeline.py llama2-7b 128 192 > gpurun_out/timeline_M128.log 2>&1
