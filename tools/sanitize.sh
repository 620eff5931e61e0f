#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the kernel test files
# (K1 verify + pick, K3 GEMM, K2/K3/K4 forwards, engines).  Summaries -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_verify_gpu.py tests/test_gemm_gpu.py tests/test_llama_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest $T -q -x -m gpu ${SAN_K:+-k "$SAN_K"} > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
