#!/bin/bash
mkdir -p gpurun_out
for M in 4 16; do
  for T in 0 1 2 4; do
    echo "M=$M TPB=$T minb3 $(PEARL_ATTN_TPB=$T timeout 300 python tools/prof_forward.py llama2-7b $M tcgen05 3 2>&1 | grep cuda-graph)"
    echo "M=$M TPB=$T minb4 $(PEARL_LIB_PATH=build/var4/libpearl_var4.so PEARL_ATTN_TPB=$T timeout 300 python tools/prof_forward.py llama2-7b $M tcgen05 3 2>&1 | grep cuda-graph)"
  done
done
timeout 600 python -m pytest tests/test_llama_gpu.py -x -q 2>&1 | tail -2
