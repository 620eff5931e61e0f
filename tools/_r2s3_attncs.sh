#!/bin/bash
# attention cluster size (sequence mode) A/B: 68M draft token forward, 7B target windows
mkdir -p gpurun_out
for c in 1 2 4; do
  PEARL_ATTN_CLUSTER=$c timeout 200 python tools/draft_fwd_ab.py >> gpurun_out/attncs_draft.log 2>&1
  echo "cluster=$c" >> gpurun_out/attncs_target.log
  PEARL_ATTN_CLUSTER=$c timeout 300 python tools/fwd_bench.py llama2-7b tcgen05 1,16,20,24 192 >> gpurun_out/attncs_target.log 2>&1
  echo "cluster=$c" >> gpurun_out/attncs_draft_fwd.log
  PEARL_ATTN_CLUSTER=$c timeout 300 python tools/fwd_bench.py llama-68m cudacore 1 192,500 >> gpurun_out/attncs_draft_fwd.log 2>&1
done
