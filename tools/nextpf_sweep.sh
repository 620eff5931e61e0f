#!/bin/bash
mkdir -p gpurun_out
for PF in 0 2 4 8 16; do
  for M in 1 4 16; do
    echo "NEXTPF=$PF $(PEARL_NEXTPF=$PF timeout 300 python tools/prof_forward.py llama2-7b $M tcgen05 3 2>&1 | grep cuda-graph)"
  done
done
