#!/bin/bash
# PEARL (adaptive) vs draft partition size with the single-token GEMV; live planner calibration
mkdir -p gpurun_out
for S in 24 32 40 48; do
  timeout 400 python bench.py --draft-sms $S --live-calibration --batch-sweep "" --no-cpu-baseline --greedy-leg 0 \
    --sd-gammas 20 --pearl-gammas 16 > gpurun_out/draftsms_s3_$S.log 2>&1
done
