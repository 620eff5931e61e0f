#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_verify_gpu.py -q -x -m gpu > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
