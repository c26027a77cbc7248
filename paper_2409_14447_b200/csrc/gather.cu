// gather.cu -- fused all-gather plumbing for the sharded device path
// (SURVEY §8e): K2 stores every record into this rank's slot of every
// rank's gathered block over peer memory (PlanArgs.mirror_*), then publishes
// an epoch into each rank's flag array.  This file holds the flag wait and
// the CUDA IPC plumbing that maps the peers' blocks (one process per GPU).
#include <cuda_runtime.h>

#include <cstring>

#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// lane r waits until rank r's flag has reached `epoch` (bounded: a peer
// that never arrives sets *status and releases the stream instead of
// hanging it)
__global__ void gather_wait_kernel(const uint32_t* flags, int n, uint32_t epoch, long long timeout_ns,
                                   int* status) {
  const int r = threadIdx.x;
  if (r >= n) return;
  const unsigned long long t0 = global_ns();
  unsigned ns = 32;
  while ((int32_t)(ld_acquire_sys_u32(flags + r) - epoch) < 0) {
    if (timeout_ns > 0 && (long long)(global_ns() - t0) > timeout_ns) {
      atomicExch(status, PARVA_LAUNCH_ERROR);
      return;
    }
    __nanosleep(ns);
    ns = ns < 1024 ? 2 * ns : ns;
  }
}

}  // namespace parva

extern "C" {

int parva_gather_wait(const uint32_t* d_flags, int32_t n, uint32_t epoch, int64_t timeout_ns, int32_t* d_status,
                      void* stream) {
  if (!d_flags || !d_status || n < 1 || n > parva::kMaxMirror) return PARVA_BAD_INPUT;
  parva::gather_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_flags, n, epoch, (long long)timeout_ns, d_status);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int parva_ipc_alloc(size_t bytes, void** d_ptr) {
  if (!d_ptr || bytes == 0) return PARVA_BAD_INPUT;
  if (cudaMalloc(d_ptr, bytes) != cudaSuccess) { cudaGetLastError(); return PARVA_LAUNCH_ERROR; }
  if (cudaMemset(*d_ptr, 0, bytes) != cudaSuccess) { cudaGetLastError(); return PARVA_LAUNCH_ERROR; }
  return PARVA_OK;
}

int parva_ipc_free(void* d_ptr) {
  return cudaFree(d_ptr) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int parva_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int parva_ipc_handle(void* d_ptr, void* handle) {
  if (!d_ptr || !handle) return PARVA_BAD_INPUT;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, d_ptr) != cudaSuccess) { cudaGetLastError(); return PARVA_LAUNCH_ERROR; }
  std::memcpy(handle, &h, sizeof(h));
  return PARVA_OK;
}

int parva_ipc_open(const void* handle, void** d_ptr) {
  if (!handle || !d_ptr) return PARVA_BAD_INPUT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return PARVA_LAUNCH_ERROR;
  }
  return PARVA_OK;
}

int parva_ipc_close(void* d_ptr) {
  return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // extern "C"
