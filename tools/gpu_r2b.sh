#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_long_decode_gpu.py tests/test_runconfig.py tests/test_checkpoint_cpu.py -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_7b_m4_r02.csv python tools/one_forward.py llama2-7b 4 192 1 > /dev/null 2>&1
timeout 300 python tools/fwd_bench.py llama2-7b tcgen05 1,4,16,32 192,1000 > gpurun_out/fwd_bench.log 2>&1
SAN_TIMEOUT=600 bash tools/sanitize.sh
