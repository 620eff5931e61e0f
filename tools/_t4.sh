#!/bin/bash
mkdir -p gpurun_out
for S in 48 64; do
  timeout 1200 python bench.py --pair dsc-33b/1.3b --prompt 512 --steps 2 --warmup 3 --draft-sms $S --live-calibration \
    --batch-sweep "" --no-cpu-baseline --greedy-leg 0 --sd-gammas 8 --pearl-gammas 8 > gpurun_out/draftsms33b_$S.log 2>&1
done
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k tile_major > gpurun_out/pytest_tiled.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiled.log
