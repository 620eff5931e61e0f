#!/bin/bash
# deeper weight ring (11 stages at NT=1) vs default, PEARL on the 108-SM target partition
mkdir -p gpurun_out
for V in default deep; do
  if [ $V = deep ]; then export PEARL_LIB_PATH=build/var_deep/libpearl_deep.so; else unset PEARL_LIB_PATH; fi
  timeout 600 python bench.py --live-calibration --batch-sweep "" --no-cpu-baseline --greedy-leg 0 --sd-gammas 16 --pearl-gammas 16 > gpurun_out/bench_ring_$V.log 2>&1
  timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,16 192 > gpurun_out/fwd_ring_$V.log 2>&1
done
