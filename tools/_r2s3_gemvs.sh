#!/bin/bash
mkdir -p gpurun_out
for v in 0 1; do PEARL_GEMVS=$v timeout 200 python tools/draft_fwd_ab.py >> gpurun_out/gemvs_ab.log 2>&1; done
for v in 0 1; do PEARL_GEMVS=$v timeout 300 python tools/draft_partition_time.py >> gpurun_out/gemvs_partition.log 2>&1; done
PEARL_GEMVS=1 timeout 900 python -m pytest tests/test_llama_gpu.py tests/test_parity_shapes_gpu.py tests/test_gemm_gpu.py tests/test_engines_plugin_gpu.py tests/test_batched_gpu.py tests/test_long_decode_gpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_gemvs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemvs.log
PEARL_GEMVS=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/draft_launches_gemvs.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
PEARL_GEMVS=1 PEARL_DRAFT_SMS=40 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/draft_launches_gemvs_p40.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
PEARL_GEMVS=0 PEARL_DRAFT_SMS=40 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/draft_launches_gemv1_p40.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
