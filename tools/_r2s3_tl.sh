#!/bin/bash
mkdir -p gpurun_out
for M in 1 16 24; do PEARL_LIB_PATH=build/var_tl/libpearl_tl.so timeout 200 python tools/timeline.py llama2-7b $M 192 > gpurun_out/timeline_s3_M$M.log 2>&1; done
