#!/bin/bash
# final pass on the committed code: all GPU tests, smoke, default bench (20 prompts)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_close.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_close.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_close.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_close.log
timeout 1200 python bench.py > gpurun_out/bench_close.log 2>&1; echo "rc=$?" >> gpurun_out/bench_close.log
