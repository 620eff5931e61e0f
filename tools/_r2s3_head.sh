#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 0 1; do PEARL_GEMV1N_HEAD=$v timeout 200 python tools/draft_fwd_ab.py >> gpurun_out/gemv1n_head_ab.log 2>&1; done
