#!/bin/bash
# 33B / 70B bench lines at the driver's 20-prompt sample (live planner tables -> gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 20 --warmup 5 --live-calibration --batch-sweep "" \
  --no-cpu-baseline --sd-gammas 4,8,16 --pearl-gammas 8 > gpurun_out/bench_33b_s3.log 2>&1
timeout 2000 python bench.py --pair llama3-70b/8b --steps 20 --warmup 5 --live-calibration --batch-sweep "" \
  --no-cpu-baseline --sd-gammas 4,8,16 --pearl-gammas 8 > gpurun_out/bench_70b_s3.log 2>&1
