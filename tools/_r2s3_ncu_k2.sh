#!/bin/bash
# one --set full capture each of the 68M gate/up (gemv1n) and lm_head (gemv1) single-token GEMVs
mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemv1n_kernel -s 3 -c 1 \
  -o gpurun_out/k2_gemv1n_full python tools/draft_block_once.py 2 > gpurun_out/ncu_k2a.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"gemv1_kernel<4" -s 1 -c 1 \
  -o gpurun_out/k2_head_full python tools/draft_block_once.py 2 > gpurun_out/ncu_k2b.log 2>&1
ls -la gpurun_out/*.ncu-rep
