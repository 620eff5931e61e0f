#!/bin/bash
# tests + draft launch list + step times
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/draft_launches3.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
timeout 300 python tools/step_times.py llama2-7b/68m 4,16 > gpurun_out/step_times3.log 2>&1
