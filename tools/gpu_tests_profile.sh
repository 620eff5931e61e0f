#!/bin/bash
# GPU tests + smoke + default bench + reference arm + ncu evidence (launch list of one 7B M=16
# forward; one --set full capture of a tc_gemm_kernel inside it) -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_7b_m16.csv python tools/one_forward.py llama2-7b 16 192 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 40 -c 1 \
  -o gpurun_out/tc_gemm_full python tools/one_forward.py llama2-7b 16 192 1 > gpurun_out/ncu_full.log 2>&1
