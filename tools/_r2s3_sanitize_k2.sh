#!/bin/bash
# compute-sanitizer memcheck + racecheck over the K2 single-token GEMV (gemv1_kernel) paths:
# the GEMM batch-invariance test (CUDA-core engine) and the CUDA-core model forwards
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py -q -x -m gpu -k "test_batch_invariance and 0 or cudacore" \
    > gpurun_out/sanitize_k2_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_k2_$tool.log
done
