#!/bin/bash
# PEARL (adaptive + fixed 16/24) vs draft partition size, current kernels; live planner calibration
mkdir -p gpurun_out
for S in 16 24 32 40 48; do
  timeout 400 python bench.py --draft-sms $S --live-calibration --batch-sweep "" --no-cpu-baseline --greedy-leg 0 \
    --sd-gammas 16 --pearl-gammas 16,24 > gpurun_out/draftsms_$S.log 2>&1
done
