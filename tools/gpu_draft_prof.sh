mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py -x -q > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/draft_launches2.csv python tools/draft_block_once.py 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sample_rows -s 1 -c 1 -o gpurun_out/sample_rows python tools/draft_block_once.py 2 > gpurun_out/ncu_sr.log 2>&1
timeout 300 python tools/step_times.py llama2-7b/68m 4,16 > gpurun_out/step_times2.log 2>&1
