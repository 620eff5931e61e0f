#!/bin/bash
# In-graph cost of each kernel class of a target forward (PEARL_ABLATE skips
# it; results are wrong while set): tools/fwd_bench.py per ablation.
mkdir -p gpurun_out
for A in "" attn gemm; do
  echo "== llama2-7b ablate=[$A]"
  PEARL_ABLATE=$A timeout 300 python tools/fwd_bench.py llama2-7b tcgen05 1,16 192 2>&1 | grep llama2
done
