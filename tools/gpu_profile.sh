#!/bin/bash
# ncu evidence for profiles/: launch list (time + DRAM bytes) of one 7B M=4 forward, and one
# --set full capture of a tc_gemm_kernel (layer 5 gate_up) inside it.
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "fwd/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/fwd7b_m4_launches.csv python tools/one_forward.py llama2-7b 4 > gpurun_out/prof1.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "fwd/" --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 22 -c 1 \
  -o gpurun_out/tc_gemm_full python tools/one_forward.py llama2-7b 4 > gpurun_out/prof2.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "fwd/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/fwd70b_m4_launches.csv python tools/one_forward.py llama3-70b 4 > gpurun_out/prof3.log 2>&1
