#!/bin/bash
# In-graph cost of each kernel class of a target forward (PEARL_ABLATE skips it; results wrong while set).
mkdir -p gpurun_out
for M in 4 16; do
for A in "" attn norm attn,norm gemm; do
  echo "== llama2-7b M=$M ablate=[$A]"
  PEARL_ABLATE=$A timeout 300 python tools/prof_forward.py llama2-7b $M tcgen05 3 2>&1 | grep -E "cuda-graph|per-op"
done; done
echo "== draft llama-68m M=1"
timeout 300 python tools/prof_forward.py llama-68m 1 cudacore 3 2>&1 | grep -E "graph|per-op"
