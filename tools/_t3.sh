#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_committed.log 2>&1; echo "rc=$?" >> gpurun_out/bench_committed.log
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 2 --warmup 3 --live-calibration --batch-sweep "" --no-cpu-baseline > gpurun_out/bench_33b.log 2>&1
timeout 1800 python bench.py --pair llama3-70b/8b --steps 2 --warmup 3 --live-calibration --batch-sweep "" --no-cpu-baseline > gpurun_out/bench_70b.log 2>&1
