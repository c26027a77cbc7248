// Can cp.async.bulk (TMA 1-D) read pinned, mapped host memory?  And how fast,
// with a few "DMA" CTAs streaming host -> smem -> device global in order?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc/tma_probe tools/zc/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SLICE, int NBUF>
__global__ void dma(const uint8_t* __restrict__ src, uint8_t* dst, int64_t bytes, unsigned* ticket) {
  extern __shared__ __align__(128) uint8_t buf[];
  __shared__ __align__(8) uint64_t bar[NBUF];
  if (threadIdx.x != 0) return;
  for (int b = 0; b < NBUF; b++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t n = (bytes + SLICE - 1) / SLICE;
  int64_t sl[NBUF];
  uint32_t phase[NBUF] = {};
  // prime
  for (int b = 0; b < NBUF; b++) {
    sl[b] = atomicAdd(ticket, 1u);
    if (sl[b] < n) {
      const uint32_t sz = (uint32_t)(bytes - sl[b] * SLICE < SLICE ? bytes - sl[b] * SLICE : SLICE);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[b])), "r"(sz) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(buf + b * SLICE)), "l"(src + sl[b] * SLICE), "r"(sz), "r"(sa(&bar[b])) : "memory");
    }
  }
  for (;;) {
    bool any = false;
    for (int b = 0; b < NBUF; b++) {
      if (sl[b] >= n) continue;
      any = true;
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                   ::"r"(sa(&bar[b])), "r"(phase[b]) : "memory");
      phase[b] ^= 1;
      const uint32_t sz = (uint32_t)(bytes - sl[b] * SLICE < SLICE ? bytes - sl[b] * SLICE : SLICE);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + sl[b] * SLICE),
                   "r"(sa(buf + b * SLICE)), "r"(sz) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      sl[b] = atomicAdd(ticket, 1u);
      if (sl[b] < n) {
        const uint32_t sz2 = (uint32_t)(bytes - sl[b] * SLICE < SLICE ? bytes - sl[b] * SLICE : SLICE);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[b])), "r"(sz2) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(buf + b * SLICE)), "l"(src + sl[b] * SLICE), "r"(sz2), "r"(sa(&bar[b])) : "memory");
      }
    }
    if (!any) break;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int64_t bytes = 2 << 20;
  uint8_t *h, *d;
  unsigned* t;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  for (int64_t i = 0; i < bytes; i++) h[i] = (uint8_t)(i * 7 + 3);
  cudaMalloc(&d, bytes);
  cudaMalloc(&t, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int slice, int nbuf, int ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, slice * nbuf);
    float best = 1e9;
    for (int r = 0; r < 20; r++) {
      cudaMemset(t, 0, 4); cudaMemset(d, 0, bytes);
      cudaEventRecord(a);
      kern<<<ctas, 32, slice * nbuf>>>(h, d, bytes, t);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    uint8_t* chk = (uint8_t*)malloc(bytes);
    cudaMemcpy(chk, d, bytes, cudaMemcpyDeviceToHost);
    int64_t bad = 0;
    for (int64_t i = 0; i < bytes; i++) bad += chk[i] != (uint8_t)(i * 7 + 3);
    free(chk);
    printf("slice %6d nbuf %d ctas %4d: %7.1f us  %5.1f GB/s  err %s  bad %lld\n", slice, nbuf, ctas, best * 1e3,
           bytes / (best * 1e-3) / 1e9, cudaGetErrorString(e), (long long)bad);
  };
  for (int ctas : {8, 16, 32, 64, 128}) {
    run(dma<8192, 2>, 8192, 2, ctas);
    run(dma<16384, 2>, 16384, 2, ctas);
    run(dma<16384, 4>, 16384, 4, ctas);
    run(dma<32768, 2>, 32768, 2, ctas);
  }
  return 0;
}
