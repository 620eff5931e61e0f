#!/bin/bash
# bench lines of the three BASELINE pairs with the current kernels (live planner calibrations -> gpurun_out/)
mkdir -p gpurun_out
timeout 900 python bench.py --live-calibration > gpurun_out/bench_7b.log 2>&1
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 2 --warmup 3 --live-calibration --batch-sweep "" --no-cpu-baseline > gpurun_out/bench_33b.log 2>&1
timeout 1800 python bench.py --pair llama3-70b/8b --steps 2 --warmup 3 --live-calibration --batch-sweep "" --no-cpu-baseline > gpurun_out/bench_70b.log 2>&1
