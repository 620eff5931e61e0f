#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/gemm_layout_probe.py 1,4,16 > gpurun_out/gemm_layout_probe.log 2>&1
timeout 900 python -m pytest tests/test_long_decode_gpu.py tests/test_kv_rollback_gpu.py tests/test_runconfig.py tests/test_checkpoint_cpu.py -m gpu -q > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
SAN_TIMEOUT=300 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_verify_gpu.py -q -x -m gpu > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
