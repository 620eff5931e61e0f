// K6 -- draft <-> target exchange over peer memory for a split pair (draft on
// one GPU, target on another, one process each).
//
// The reference's rendezvous is _PhaseRunner (engines.py:241-262): the draft
// closure's result (xs, qs) and the target closure's result (ps) meet in one
// host thread, which verifies.  Split across two GPUs, the meeting point is
// the target GPU: the draft rank pushes its gamma ids and q-logit rows
// straight into a mailbox in the target GPU's memory (NVLink stores through a
// CUDA-IPC mapping), the target verifies and pushes the 32-byte verdict back
// into the draft GPU's mailbox.  Each push is ONE kernel (payload stores,
// system-scope fence, last-arriving CTA releases a sequence flag); each
// receive is ONE single-thread kernel spinning on its local flag with an
// acquire load.  Both are stream-ordered device work, so a whole split step
// (forward -> push -> wait -> verify/commit) is still one CUDA graph per rank
// with no host round trip in between.
//
// Sequence numbers never reset: every step sends exactly one message in each
// direction, so the sender's and receiver's counters advance in lockstep for
// the life of the link, and a mailbox can never be overwritten before it was
// consumed (the draft pushes step t+1 only after the verdict of step t, which
// the target sends after consuming step t's payload).
#include <cuda_runtime.h>

#include <cstring>

#include "common.h"

namespace pearl {

constexpr int kXferThreads = 256;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kXferThreads) xfer_send_kernel(pearl_xfer_send_args a) {
  char* box = static_cast<char*>(a.peer_box);
  // ids (block 0)
  if (blockIdx.x == 0) {
    int32_t* dst = reinterpret_cast<int32_t*>(box + PEARL_MAILBOX_IDS_OFFSET);
    for (int i = threadIdx.x; i < a.n_ids; i += blockDim.x) dst[i] = a.ids[i];
  }
  // rows: one contiguous fp32 slab, 16-byte stores, grid-strided
  const size_t n = static_cast<size_t>(a.n_rows) * a.V;
  if (n) {
    const float* src = a.rows;
    float* dst = reinterpret_cast<float*>(box + PEARL_MAILBOX_ROWS_OFFSET);
    const size_t n4 = n / 4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // 4 independent 16-byte loads in flight per thread
    for (; i + 3 * stride < n4; i += 4 * stride) {
      const float4 v0 = __ldg(s4 + i), v1 = __ldg(s4 + i + stride), v2 = __ldg(s4 + i + 2 * stride),
                   v3 = __ldg(s4 + i + 3 * stride);
      d4[i] = v0;
      d4[i + stride] = v1;
      d4[i + 2 * stride] = v2;
      d4[i + 3 * stride] = v3;
    }
    for (; i < n4; i += stride) d4[i] = __ldg(s4 + i);
    if (blockIdx.x == 0)
      for (size_t j = n4 * 4 + threadIdx.x; j < n; j += blockDim.x) dst[j] = src[j];
  }
  // every CTA's stores are ordered before its arrival; the last arriver
  // publishes the new sequence number to the peer
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned prev = atomicAdd(a.arrive, 1u);
  if (prev + 1 != gridDim.x) return;
  *a.arrive = 0u;
  __threadfence_system();
  const unsigned long long seq = *a.send_seq + 1ull;
  *a.send_seq = seq;
  st_release_sys(reinterpret_cast<unsigned long long*>(box), seq);
}

__global__ void xfer_wait_kernel(const void* box, unsigned long long* recv_seq, int32_t* dst, int n_ids,
                                 int32_t* status, long long timeout_ns) {
  const unsigned long long want = *recv_seq + 1ull;
  const unsigned long long* flag = static_cast<const unsigned long long*>(box);
  const unsigned long long t0 = global_ns();
  unsigned ns = 32;
  while (ld_acquire_sys(flag) < want) {
    if (timeout_ns > 0 && static_cast<long long>(global_ns() - t0) > timeout_ns) {
      if (status) *status = PEARL_ERR_TIMEOUT;
      break;
    }
    __nanosleep(ns);
    if (ns < 1024) ns *= 2;
  }
  *recv_seq = want;
  if (dst) {
    const int32_t* ids = reinterpret_cast<const int32_t*>(static_cast<const char*>(box) + PEARL_MAILBOX_IDS_OFFSET);
    for (int i = 0; i < n_ids; ++i) dst[i] = ids[i];
  }
}

}  // namespace pearl

using namespace pearl;

extern "C" size_t pearl_mailbox_bytes(int n_rows, int V) {
  return PEARL_MAILBOX_ROWS_OFFSET + static_cast<size_t>(n_rows > 0 ? n_rows : 0) * (V > 0 ? V : 0) * sizeof(float);
}

extern "C" int pearl_mailbox_alloc(size_t bytes, void** dptr) {
  PEARL_ARG_CHECK(dptr && bytes >= PEARL_MAILBOX_ROWS_OFFSET, "bad mailbox size");
  void* p = nullptr;
  PEARL_CUDA_TRY(cudaMalloc(&p, bytes));
  PEARL_CUDA_TRY(cudaMemset(p, 0, bytes));
  PEARL_CUDA_TRY(cudaDeviceSynchronize());
  *dptr = p;
  return PEARL_OK;
}

extern "C" int pearl_mailbox_free(void* dptr) {
  if (dptr) PEARL_CUDA_TRY(cudaFree(dptr));
  return PEARL_OK;
}

extern "C" int pearl_ipc_export(void* dptr, void* handle_out) {
  PEARL_ARG_CHECK(dptr && handle_out, "bad ipc export arguments");
  cudaIpcMemHandle_t h;
  PEARL_CUDA_TRY(cudaIpcGetMemHandle(&h, dptr));
  static_assert(sizeof(h) == PEARL_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  return PEARL_OK;
}

extern "C" int pearl_ipc_import(const void* handle, void** dptr) {
  PEARL_ARG_CHECK(handle && dptr, "bad ipc import arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  PEARL_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *dptr = p;
  return PEARL_OK;
}

extern "C" int pearl_ipc_close(void* dptr) {
  if (dptr) PEARL_CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return PEARL_OK;
}

extern "C" int pearl_xfer_send(const pearl_xfer_send_args* args, void* stream) {
  PEARL_ARG_CHECK(args && args->peer_box && args->send_seq && args->arrive, "bad xfer_send arguments");
  PEARL_ARG_CHECK(args->n_ids >= 0 && args->n_ids <= PEARL_MAILBOX_MAX_IDS && (args->n_ids == 0 || args->ids),
                  "xfer_send: 0 <= n_ids <= PEARL_MAILBOX_MAX_IDS");
  PEARL_ARG_CHECK(args->n_rows >= 0 && (args->n_rows == 0 || (args->rows && args->V > 0)), "xfer_send: rows");
  PEARL_ARG_CHECK((reinterpret_cast<uintptr_t>(args->rows) & 15) == 0, "xfer_send: rows must be 16-byte aligned");
  const size_t n4 = static_cast<size_t>(args->n_rows) * args->V / 4;
  // ~4 float4 per thread per pass; at most one CTA per SM (148)
  int grid = static_cast<int>((n4 + 4 * kXferThreads - 1) / (4 * kXferThreads));
  grid = grid < 1 ? 1 : (grid > 148 ? 148 : grid);
  xfer_send_kernel<<<grid, kXferThreads, 0, static_cast<cudaStream_t>(stream)>>>(*args);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  return PEARL_OK;
}

__global__ void xfer_seq_kernel(unsigned long long* send_seq, unsigned long long* staging) {
  const unsigned long long seq = *send_seq + 1ull;
  *send_seq = seq;
  *staging = seq;
}

extern "C" int pearl_xfer_send_copy(const pearl_xfer_send_args* a, unsigned long long* staging, void* stream) {
  PEARL_ARG_CHECK(a && a->peer_box && a->send_seq && staging, "bad xfer_send_copy arguments");
  PEARL_ARG_CHECK(a->n_ids >= 0 && a->n_ids <= PEARL_MAILBOX_MAX_IDS && (a->n_ids == 0 || a->ids),
                  "xfer_send_copy: 0 <= n_ids <= PEARL_MAILBOX_MAX_IDS");
  PEARL_ARG_CHECK(a->n_rows >= 0 && (a->n_rows == 0 || (a->rows && a->V > 0)), "xfer_send_copy: rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* box = static_cast<char*>(a->peer_box);
  if (a->n_ids)
    PEARL_CUDA_TRY(cudaMemcpyAsync(box + PEARL_MAILBOX_IDS_OFFSET, a->ids, static_cast<size_t>(a->n_ids) * 4,
                                   cudaMemcpyDefault, st));
  if (a->n_rows)
    PEARL_CUDA_TRY(cudaMemcpyAsync(box + PEARL_MAILBOX_ROWS_OFFSET, a->rows,
                                   static_cast<size_t>(a->n_rows) * a->V * sizeof(float), cudaMemcpyDefault, st));
  xfer_seq_kernel<<<1, 1, 0, st>>>(a->send_seq, staging);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  PEARL_CUDA_TRY(cudaMemcpyAsync(box, staging, sizeof(unsigned long long), cudaMemcpyDefault, st));
  return PEARL_OK;
}

extern "C" int pearl_pci_bus_id(char* out, int len) {
  PEARL_ARG_CHECK(out && len >= 16, "pci bus id buffer too small");
  int dev = 0;
  PEARL_CUDA_TRY(cudaGetDevice(&dev));
  PEARL_CUDA_TRY(cudaDeviceGetPCIBusId(out, len, dev));
  return PEARL_OK;
}

extern "C" int pearl_peer_storable(const char* peer_pci_bus_id) {
  PEARL_ARG_CHECK(peer_pci_bus_id, "null pci bus id");
  int dev = 0, peer = -1, ok = 0;
  PEARL_CUDA_TRY(cudaGetDevice(&dev));
  if (cudaDeviceGetByPCIBusId(&peer, peer_pci_bus_id) != cudaSuccess) {
    cudaGetLastError();
    return 0;  // the peer GPU is not visible to this process: no direct stores
  }
  if (peer == dev) return 1;
  PEARL_CUDA_TRY(cudaDeviceCanAccessPeer(&ok, dev, peer));
  return ok ? 1 : 0;
}

extern "C" int pearl_xfer_wait(const void* box, unsigned long long* recv_seq, int32_t* dst_ids, int n_ids,
                               int32_t* status, long long timeout_ns, void* stream) {
  PEARL_ARG_CHECK(box && recv_seq, "bad xfer_wait arguments");
  PEARL_ARG_CHECK(n_ids >= 0 && n_ids <= PEARL_MAILBOX_MAX_IDS && (n_ids == 0 || dst_ids), "xfer_wait: n_ids");
  xfer_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(box, recv_seq, dst_ids, n_ids, status,
                                                                  timeout_ns);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  return PEARL_OK;
}
