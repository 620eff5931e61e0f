#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/fwd_bench.py llama2-7b tcgen05 1,4,16,32 192 > gpurun_out/fwd_default.log 2>&1
for M in 1 16; do
  PEARL_LIB_PATH=build/var_tl/libpearl_tl.so timeout 200 python tools/timeline.py llama2-7b $M 192 > gpurun_out/timeline_M$M.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
