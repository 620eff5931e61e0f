#!/bin/bash
mkdir -p gpurun_out
for PF in 0 4 8 16 32 64; do
  for M in 1 4 16; do
    echo "L2PF=$PF $(PEARL_L2PF=$PF timeout 300 python tools/prof_forward.py llama2-7b $M tcgen05 3 2>&1 | grep cuda-graph)"
  done
done
