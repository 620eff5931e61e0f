#!/bin/bash
mkdir -p gpurun_out
for D in 16 24 32 48; do
  echo "== DRAFT_SMS=$D"; PEARL_DRAFT_SMS=$D timeout 600 python tools/step_times.py llama2-7b/68m 8,12,16,24 2>&1 | grep -v Warn
done
