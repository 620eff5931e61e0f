#!/bin/bash
# session-3 verification of HEAD: GPU tests, smoke, launch list of one eager 68M draft block
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/draft_launches_s3.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
timeout 300 python tools/step_times.py llama2-7b/68m 4,16 > gpurun_out/step_times_s3.log 2>&1
