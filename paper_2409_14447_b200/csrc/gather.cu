// gather.cu -- fused all-gather plumbing for the sharded device path
// (SURVEY §8e): K2 stores every record into this rank's sections of a slot
// on every rank over peer memory (PlanArgs.mirror_*), then publishes the
// launch's epoch into its flag word of the slot on each rank.  This file
// holds the consumer side (exact-epoch flag wait + release of the slot into
// every producer's ack row) and the CUDA IPC plumbing that maps the peers'
// buffers (one process per GPU).
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

// lane r waits until rank r's flag word of the slot holds exactly `epoch`
// (bounded: a peer that never arrives -- or whose later epoch already
// overwrote the slot -- sets *status and releases the stream instead of
// hanging it); then, if `release`, lane m stores the epoch into this rank's
// ack word of the slot on rank m, so rank m's producer may reuse the slot.
struct GatherSlotArgs {
  const uint32_t* flags;
  uint32_t* ack[kMaxMirror];
  int n;
};

__global__ void gather_wait_kernel(GatherSlotArgs g, uint32_t epoch, int wait, int release, long long timeout_ns,
                                   int* status) {
  const int r = threadIdx.x;
  bool ok = true;
  if (wait && r < g.n) {
    const unsigned long long t0 = global_ns();
    unsigned ns = 32;
    while (ld_acquire_sys_u32(g.flags + r) != epoch) {
      if (timeout_ns > 0 && (long long)(global_ns() - t0) > timeout_ns) {
        atomicExch(status, PARVA_LAUNCH_ERROR);
        ok = false;
        break;
      }
      __nanosleep(ns);
      ns = ns < 1024 ? 2 * ns : ns;
    }
  }
  // every rank's records of the epoch have landed here (acquire above);
  // release the slot only when all of them did
  if (!__all_sync(0xffffffffu, ok) || !release) return;
  if (r < g.n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(g.ack[r]), "r"(epoch) : "memory");
}

// one thread waits until a host-written word (pinned, mapped) equals `value`
// (benchmark gate: queue a timed region behind it, then open it, so the
// region measures device execution without host launch gaps)
__global__ void host_gate_kernel(const volatile uint32_t* flag, uint32_t value, long long timeout_ns, int* status) {
  const unsigned long long t0 = global_ns();
  while (*flag != value) {
    if (timeout_ns > 0 && (long long)(global_ns() - t0) > timeout_ns) {
      if (status) atomicExch(status, PARVA_LAUNCH_ERROR);
      return;
    }
    __nanosleep(256);
  }
}

}  // namespace parva

extern "C" {

int parva_host_gate(const uint32_t* h_flag, uint32_t value, int64_t timeout_ns, int32_t* d_status, void* stream) {
  if (!h_flag) return PARVA_BAD_INPUT;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, const_cast<uint32_t*>(h_flag), 0) != cudaSuccess) {
    cudaGetLastError();
    return PARVA_BAD_INPUT;   // not pinned, mapped host memory
  }
  parva::host_gate_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((const volatile uint32_t*)d, value,
                                                              (long long)timeout_ns, (int*)d_status);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

static int gather_slot_launch(const parva_gather_slot* slot, uint32_t epoch, int wait, int release,
                              int64_t timeout_ns, int32_t* d_status, void* stream) {
  if (!slot || slot->n < 1 || slot->n > parva::kMaxMirror || epoch == 0) return PARVA_BAD_INPUT;
  if (wait && (!slot->d_flags || !d_status)) return PARVA_BAD_INPUT;
  parva::GatherSlotArgs g = {};
  g.flags = slot->d_flags;
  g.n = slot->n;
  for (int m = 0; m < slot->n; m++) {
    if (release && !slot->ack[m]) return PARVA_BAD_INPUT;
    g.ack[m] = slot->ack[m];
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = slot->pdl ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, parva::gather_wait_kernel, g, epoch, wait, release, (long long)timeout_ns,
                         (int*)d_status) != cudaSuccess)
    return PARVA_LAUNCH_ERROR;
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int parva_gather_wait(const parva_gather_slot* slot, uint32_t epoch, int32_t release, int64_t timeout_ns,
                      int32_t* d_status, void* stream) {
  return gather_slot_launch(slot, epoch, 1, release ? 1 : 0, timeout_ns, d_status, stream);
}

int parva_gather_release(const parva_gather_slot* slot, uint32_t epoch, void* stream) {
  return gather_slot_launch(slot, epoch, 0, 1, 0, nullptr, stream);
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
