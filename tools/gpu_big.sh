mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 1500 python bench.py --pair dsc-33b/1.3b --prompt 512 --new 128 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_dsc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dsc.log
timeout 1800 python bench.py --pair llama3-70b/8b --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_70b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_70b.log
nvidia-smi >> gpurun_out/free.txt
