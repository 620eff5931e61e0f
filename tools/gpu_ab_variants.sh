#!/bin/bash
# A/B of diagnostic library variants against the default build (profiles/README.md, round 2):
#   python -m paper_2408_11850_b200.build --variant r90  -DPEARL_RING_KB=90 -DPEARL_GEMM_MINB=2     # 2 GEMM CTAs / SM
#   python -m paper_2408_11850_b200.build --variant deep -DPEARL_RING_KB=200 -DPEARL_MAX_STAGES=12  # 11-stage W ring
# then, on the GPU box: bash tools/gpu_ab_variants.sh r90 deep
mkdir -p gpurun_out
for V in default "$@"; do
  if [ "$V" = default ]; then unset PEARL_LIB_PATH; else export PEARL_LIB_PATH=build/var_$V/libpearl_$V.so; fi
  timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16 192 > gpurun_out/fwd_ab_$V.log 2>&1
  timeout 600 python bench.py --live-calibration --batch-sweep "" --no-cpu-baseline --greedy-leg 0 \
    --sd-gammas 16 --pearl-gammas 16 > gpurun_out/bench_ab_$V.log 2>&1
done
