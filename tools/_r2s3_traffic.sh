#!/bin/bash
# DRAM traffic of one target window forward at each bench line's dominant window (roofline.traffic)
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 400 ncu $M --log-file gpurun_out/traffic_7b_m20.csv python tools/one_forward.py llama2-7b 20 192 1 > /dev/null 2>&1
timeout 900 ncu $M --log-file gpurun_out/traffic_33b_m8.csv python tools/one_forward.py dsc-33b 8 576 1 > /dev/null 2>&1
timeout 1200 ncu $M --log-file gpurun_out/traffic_70b_m8.csv python tools/one_forward.py llama3-70b 8 192 1 > /dev/null 2>&1
ls -la gpurun_out/traffic_*
