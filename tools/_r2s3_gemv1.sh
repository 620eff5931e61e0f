#!/bin/bash
mkdir -p gpurun_out
for v in 0 1; do PEARL_GEMV1=$v timeout 200 python tools/draft_fwd_ab.py >> gpurun_out/gemv1_ab.log 2>&1; done
for v in 0 1; do PEARL_DRAFT_SMS=40 PEARL_GEMV1=$v timeout 200 python tools/draft_fwd_ab.py >> gpurun_out/gemv1_ab.log 2>&1; done
timeout 900 python -m pytest tests/test_llama_gpu.py tests/test_parity_shapes_gpu.py tests/test_gemm_gpu.py tests/test_engines_plugin_gpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_gemv1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemv1.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/draft_launches_gemv1.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
timeout 300 python tools/step_times.py llama2-7b/68m 16,24 > gpurun_out/step_times_gemv1.log 2>&1
