#!/bin/bash
# session-3 final pass: GPU tests, smoke, default bench (committed calibrations)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final_s3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_final_s3.log
