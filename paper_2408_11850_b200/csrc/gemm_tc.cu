// K3 placeholder: tcgen05 path not yet wired (returns an argument error).
#include "gemm_tc.cuh"

namespace pearl {
int tc_init(TcGemmCtx& ctx, const pearl_llama_config& cfg) {
  (void)ctx;
  (void)cfg;
  set_error("tcgen05 GEMM path not built yet");
  return PEARL_ERR_ARG;
}
void tc_free(TcGemmCtx& ctx) { (void)ctx; }
int tc_gemm(TcGemmCtx&, const __nv_bfloat16*, const __nv_bfloat16*, int, int, int, const EpiArgs&, cudaStream_t) {
  set_error("tcgen05 GEMM path not built yet");
  return PEARL_ERR_ARG;
}
}  // namespace pearl
