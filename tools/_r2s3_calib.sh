#!/bin/bash
# refreshed planner calibrations (live) for 7B/68M at T=1 and T=0 with the session-3 kernels
mkdir -p gpurun_out
timeout 900 python bench.py --live-calibration > gpurun_out/bench_live_s3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_live_s3.log
timeout 400 python bench.py --live-calibration --temperature 0 --batch-sweep "" --no-cpu-baseline --greedy-leg 0 > gpurun_out/bench_live_T0_s3.log 2>&1
