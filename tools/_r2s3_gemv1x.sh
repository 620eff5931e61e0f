#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 0 1; do PEARL_GEMV1X=$v timeout 200 python tools/draft_fwd_ab.py >> gpurun_out/gemv1x_ab.log 2>&1; done
timeout 900 python -m pytest tests/test_llama_gpu.py tests/test_parity_shapes_gpu.py tests/test_gemm_gpu.py tests/test_engines_plugin_gpu.py tests/test_batched_gpu.py tests/test_long_decode_gpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_gemv1x.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemv1x.log
