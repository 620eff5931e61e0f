#!/bin/bash
# planner table A/B at the driver's sample size (20 prompts): A = the table measured with the
# 53-us draft, B = the one measured with the 49-us draft (tmp_calib/)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --batch-sweep "" > gpurun_out/calib_A.log 2>&1
cp tmp_calib/new_T1.json profiles/planner_calib_llama2-7b_68m_T1.json
cp tmp_calib/new_T0.json profiles/planner_calib_llama2-7b_68m_T0.json
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --batch-sweep "" > gpurun_out/calib_B.log 2>&1
