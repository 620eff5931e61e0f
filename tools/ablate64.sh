mkdir -p gpurun_out
for M in 32 64; do for A in "" attn norm gemm; do
  echo "M=$M ablate=[$A] $(PEARL_ABLATE=$A timeout 300 python tools/prof_forward.py llama2-7b $M tcgen05 3 2>&1 | grep -E 'cuda-graph')"
done; done
