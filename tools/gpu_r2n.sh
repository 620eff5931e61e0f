#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16,32,64,128 192 > gpurun_out/fwd_default.log 2>&1
timeout 200 python tools/gemm_m_sweep.py > gpurun_out/gemm_m_sweep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --sd-gammas 4,8,16 --pearl-gammas 16 --greedy-leg 0 --no-cpu-baseline --batch-sweep 1,4,16,32 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
