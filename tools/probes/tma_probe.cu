// Memory-system probe: stream a large bf16 matrix into shared memory with
// (a) 2D TMA boxes of R rows x 64 cols (SWIZZLE_128B), row stride K,
// (b) 1D cp.async.bulk copies of contiguous chunks,
// each from a persistent 148-CTA grid with an S-stage mbarrier ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}

template <int MODE>  // 0 = 2D TMA box, 1 = 1D bulk, 2 = 1D bulk contiguous per-CTA range
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm, const char* base, long long total_chunks,
                                                int chunk_bytes, int stages, int rows_per_box, int tiles_k, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ring = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(ring + stages * chunk_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // chunks c = blockIdx.x, +grid ... ; keep 'stages' in flight
  long long my = 0;
  long long lo = total_chunks * blockIdx.x / gridDim.x, hi = total_chunks * (blockIdx.x + 1) / gridDim.x;
  if (MODE == 2) my = hi - lo;
  else for (long long c = blockIdx.x; c < total_chunks; c += gridDim.x) ++my;
  unsigned long long acc = 0;
  long long issued = 0, done = 0;
  auto issue = [&](long long i) {
    long long c = (MODE == 2) ? lo + i : blockIdx.x + i * gridDim.x;
    int s = (int)(i % stages);
    unsigned char* dst = ring + s * chunk_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"(chunk_bytes) : "memory");
    if (MODE == 0) {
      int tile = (int)(c / tiles_k), kt = (int)(c % tiles_k);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(su(dst)), "l"((uint64_t)&tm), "r"(kt * 64), "r"(tile * rows_per_box), "r"(su(&full[s])) : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su(dst)), "l"(base + c * (long long)chunk_bytes), "r"(chunk_bytes), "r"(su(&full[s])) : "memory");
    }
  };
  for (; issued < my && issued < stages; ++issued) issue(issued);
  for (; done < my; ++done) {
    int s = (int)(done % stages);
    wait(&full[s], (uint32_t)((done / stages) & 1));
    acc += ring[s * chunk_bytes + (done & 63)];
    if (issued < my) { issue(issued); ++issued; }
  }
  atomicAdd(sink, acc);
}

int main() {
  const long long N = 131072, K = 4096;  // 1 GiB bf16
  const size_t bytes = N * K * 2;
  char* d; cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes);
  char* flush; cudaMalloc(&flush, 512 << 20);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](int mode, int rows, int chunk, int stages, int grid) {
    CUtensorMap tm{};
    if (mode == 0) {
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N}; cuuint64_t str[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)rows}; cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      chunk = rows * 128;
    }
    long long total = (long long)(bytes / chunk);
    int tiles_k = (int)(K / 64);
    size_t smem = 1024 + (size_t)stages * chunk + 512;
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(flush, it, 512 << 20);
      cudaEventRecord(a);
      if (mode == 0) probe<0><<<grid, 128, smem>>>(tm, d, total, chunk, stages, rows, tiles_k, sink);
      else if (mode == 1) probe<1><<<grid, 128, smem>>>(tm, d, total, chunk, stages, rows, tiles_k, sink);
      else probe<2><<<grid, 128, smem>>>(tm, d, total, chunk, stages, rows, tiles_k, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("mode=%d rows=%3d chunk=%6d stages=%2d grid=%4d : %7.1f GB/s %s\n", mode, rows, chunk, stages, grid,
           bytes / (best * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
  };
  for (int st : {8, 12}) run(0, 128, 0, st, sms);
  run(0, 128, 0, 6, 2 * sms);
  for (int st : {8, 12}) run(1, 0, 16384, st, sms);
  for (int st : {8, 12}) run(2, 0, 16384, st, sms);
  run(2, 0, 32768, 6, sms);
  run(2, 0, 16384, 6, 2 * sms);
  run(2, 0, 65536, 3, sms);
  return 0;
}
