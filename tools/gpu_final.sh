#!/bin/bash
# round-end pass: full GPU tests, smoke, refreshed planner calibrations (live, copied to gpurun_out/),
# then the default bench with them committed, reference arm, 33B line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --live-calibration > gpurun_out/bench_live.log 2>&1; echo "rc=$?" >> gpurun_out/bench_live.log
timeout 300 python bench.py --live-calibration --temperature 0 --batch-sweep "" --no-cpu-baseline --greedy-leg 0 --steps 1 --warmup 3 > /dev/null 2>&1
