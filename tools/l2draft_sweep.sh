#!/bin/bash
mkdir -p gpurun_out
for L in 0 1; do for rep in 1 2; do
  echo "L2_DRAFT=$L $(PEARL_L2_DRAFT=$L timeout 600 python bench.py --no-cpu-baseline --batch-sweep '' 2>&1 | tail -1)"
done; done
