#!/bin/bash
# session-3 closing pass: GPU tests, smoke, live planner calibrations (T=1 and the greedy leg's
# T=0 table), then the default bench on those committed-to-be tables
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_final2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final2.log
timeout 900 python bench.py --live-calibration --no-cpu-baseline --batch-sweep "" > gpurun_out/bench_live_s3b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_live_s3b.log
cp gpurun_out/planner_calib_llama2-7b_68m_T1.json gpurun_out/planner_calib_llama2-7b_68m_T0.json profiles/
timeout 900 python bench.py > gpurun_out/bench_final_s3b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_final_s3b.log
