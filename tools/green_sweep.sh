#!/bin/bash
mkdir -p gpurun_out
for D in 0 8 16 24 32; do
  echo "DRAFT_SMS=$D $(PEARL_DRAFT_SMS=$D timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1)"
done
