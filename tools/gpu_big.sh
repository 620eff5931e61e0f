#!/bin/bash
# Larger pairs on one B200 (co-resident): DSC-33B/1.3B (prompt 512) and Llama-3-70B/8B.
mkdir -p gpurun_out
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --new 128 --steps 3 --warmup 3 --no-cpu-baseline --batch-sweep 1,4,16 > gpurun_out/bench_dsc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dsc.log
timeout 1800 python bench.py --pair llama3-70b/8b --steps 3 --warmup 3 --no-cpu-baseline --batch-sweep 1,4,16 > gpurun_out/bench_70b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_70b.log
