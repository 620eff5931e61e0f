#!/bin/bash
# Round-end evidence: GPU tests, smoke, default bench (both arms), the larger pairs.
bash tools/gpu_check.sh
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dsc.log 2>&1
timeout 1800 python bench.py --pair llama3-70b/8b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_70b.log 2>&1
