#!/bin/bash
# draft partition sweep at the driver's 20-prompt sample (live planner tables per size)
mkdir -p gpurun_out
for S in 24 32 40 48; do
  timeout 600 python bench.py --draft-sms $S --live-calibration --batch-sweep "" --no-cpu-baseline --greedy-leg 0 \
    --sd-gammas 16 --pearl-gammas "" > gpurun_out/draftsms20_$S.log 2>&1
  mkdir -p gpurun_out/calib_$S; cp gpurun_out/planner_calib_llama2-7b_68m_T1.json gpurun_out/calib_$S/
done
