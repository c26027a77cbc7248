// Zero-copy probe: kernel reads / writes pinned host memory directly over PCIe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc/zc_probe tools/zc/zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const uint4* __restrict__ src, size_t n16, unsigned long long* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = 1;
}

__global__ void wr(uint4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((unsigned)i, 1, 2, 3);
}

__global__ void rdwr(const uint4* __restrict__ src, uint4* dst, size_t n16, size_t m16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    if (i < m16) dst[i] = v;
  }
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t bytes : {64u << 10, 512u << 10, 2u << 20, 8u << 20, 32u << 20}) {
    void *h_in, *h_out;
    cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped);
    memset(h_in, 1, bytes);
    size_t n16 = bytes / 16;
    for (int grid : {148, 296, 592, 1184}) {
      float best_r = 1e9, best_w = 1e9, best_rw = 1e9;
      for (int rep = 0; rep < 20; rep++) {
        float ms;
        cudaEventRecord(a); rd<<<grid, 256>>>((const uint4*)h_in, n16, sink); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best_r) best_r = ms;
        cudaEventRecord(a); wr<<<grid, 256>>>((uint4*)h_out, n16); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best_w) best_w = ms;
        cudaEventRecord(a); rdwr<<<grid, 256>>>((const uint4*)h_in, (uint4*)h_out, n16, n16 * 3 / 4); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best_rw) best_rw = ms;
      }
      printf("%8zu KiB grid %5d  read %7.1f us (%5.1f GB/s)  write %7.1f us (%5.1f GB/s)  read+write.75 %7.1f us\n",
             bytes >> 10, grid, best_r * 1e3, bytes / (best_r * 1e-3) / 1e9, best_w * 1e3,
             bytes / (best_w * 1e-3) / 1e9, best_rw * 1e3);
    }
    cudaFreeHost(h_in); cudaFreeHost(h_out);
  }
  // latency: one thread, dependent loads
  return 0;
}
