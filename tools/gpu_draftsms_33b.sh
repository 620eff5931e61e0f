#!/bin/bash
# DSC-33B/1.3B: PEARL vs the draft's green-partition size (live planner calibration)
mkdir -p gpurun_out
for S in 32 64 80; do
  timeout 1200 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 2 --warmup 3 --draft-sms $S --live-calibration \
    --batch-sweep "" --no-cpu-baseline --greedy-leg 0 --sd-gammas 8 --pearl-gammas 8 > gpurun_out/draftsms33_$S.log 2>&1
done
