#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bench_contract_gpu.py -m gpu -q -x > gpurun_out/pytest_bench_contract.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bench_contract.log
timeout 1200 python bench.py > gpurun_out/bench_default_s3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default_s3.log
