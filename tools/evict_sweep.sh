#!/bin/bash
mkdir -p gpurun_out
for E in 0 1; do
  echo "EF=$E $(PEARL_W_EVICT_FIRST=$E timeout 900 python bench.py --no-cpu-baseline --batch-sweep '' 2>&1 | tail -1)"
  echo "EF=$E steps: $(PEARL_W_EVICT_FIRST=$E PEARL_DRAFT_SMS=16 timeout 600 python tools/step_times.py llama2-7b/68m 12,16,24 2>&1 | grep -v Warn | tr '\n' ' ')"
done
