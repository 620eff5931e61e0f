#!/bin/bash
# 33B / 70B bench lines with the current kernels (live planner calibrations -> gpurun_out/), then racecheck on K1
mkdir -p gpurun_out
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 2 --warmup 3 --live-calibration --batch-sweep "" --no-cpu-baseline > gpurun_out/bench_33b.log 2>&1
timeout 1800 python bench.py --pair llama3-70b/8b --steps 2 --warmup 3 --live-calibration --batch-sweep "" --no-cpu-baseline > gpurun_out/bench_70b.log 2>&1
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_verify_gpu.py -q -x -m gpu -k "not large_vocab" > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
