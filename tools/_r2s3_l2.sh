#!/bin/bash
# persisting-L2 window over the 68M draft's streamed weights, A/B with the session-3 GEMV
mkdir -p gpurun_out
PEARL_L2_DRAFT=1 timeout 120 python tools/l2_granted.py > gpurun_out/l2_s3.log 2>&1
for L in 0 1; do
  echo "L2_DRAFT=$L $(PEARL_L2_DRAFT=$L timeout 600 python bench.py --no-cpu-baseline --batch-sweep '' --greedy-leg 0 --sd-gammas 16,20,24 --pearl-gammas 16 2>&1 | tail -1)" >> gpurun_out/l2_s3.log
  PEARL_L2_DRAFT=$L timeout 300 python tools/step_times.py llama2-7b/68m 16,24 >> gpurun_out/l2_s3.log 2>&1
done
