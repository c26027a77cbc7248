// Host-write probe: bandwidth of kernel stores into pinned mapped host memory
// by store shape (the K2s record writes are 8-B config records, 11 per
// scenario, and 64-B plan records).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc/wr_probe tools/zc/wr_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// piece = bytes written per store group (lanes x 8 B or x 16 B); pieces are
// contiguous, taken by groups of `glanes` lanes in a grid-stride loop
template <int W>   // bytes per lane: 8 or 16
__global__ void wr_pieces(uint8_t* dst, size_t bytes, int piece, int glanes) {
  const int lane = threadIdx.x & 31, g = lane / glanes, gl = lane % glanes, gpw = 32 / glanes;
  const size_t n_pieces = bytes / piece;
  const size_t gid = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32 * gpw + g;
  const size_t ng = (size_t)gridDim.x * blockDim.x / 32 * gpw;
  for (size_t p = gid; p < n_pieces; p += ng) {
    for (int o = gl * W; o < piece; o += glanes * W) {
      if (W == 8) *reinterpret_cast<uint64_t*>(dst + p * piece + o) = p;
      else *reinterpret_cast<uint4*>(dst + p * piece + o) = make_uint4((unsigned)p, 1, 2, 3);
    }
  }
}

// bulk: each warp stages `piece` bytes in shared memory and one lane stores
// them with cp.async.bulk (shared -> global)
__global__ void wr_bulk(uint8_t* dst, size_t bytes, int piece) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint8_t* buf = sm + warp * piece;
  for (int o = lane * 16; o < piece; o += 512) *reinterpret_cast<uint4*>(buf + o) = make_uint4(o, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const size_t n_pieces = bytes / piece;
  const size_t nw = (size_t)gridDim.x * blockDim.x / 32;
  for (size_t p = blockIdx.x * (size_t)(blockDim.x / 32) + warp; p < n_pieces; p += nw) {
    if (lane == 0) {
      unsigned s = (unsigned)__cvta_generic_to_shared(buf);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + p * piece), "r"(s),
                   "r"(piece) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 1520000 / 2816 * 2816;   // ~1.5 MB, divisible by the pieces below
  uint8_t* h;
  cudaHostAlloc(&h, bytes + 4096, cudaHostAllocMapped);
  uint8_t* d;
  cudaHostGetDevicePointer((void**)&d, h, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(wr_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 2816);
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 30; r++) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r > 2 && ms < best) best = ms;
    }
    printf("%-44s %8.1f us  %6.1f GB/s  %s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int grid : {148, 296}) {
    printf("grid %d x 512\n", grid);
    timeit("8 B/lane, 88-B pieces (16-lane groups)", [&] { wr_pieces<8><<<grid, 512>>>(d, bytes, 88, 16); });
    timeit("16 B/lane, 64-B pieces (4 lanes)", [&] { wr_pieces<16><<<grid, 512>>>(d, bytes, 64, 4); });
    timeit("16 B/lane, 128-B pieces (8 lanes)", [&] { wr_pieces<16><<<grid, 512>>>(d, bytes, 128, 8); });
    timeit("16 B/lane, 512-B pieces (32 lanes)", [&] { wr_pieces<16><<<grid, 512>>>(d, bytes, 512, 32); });
    timeit("8 B/lane, 256-B pieces (32 lanes)", [&] { wr_pieces<8><<<grid, 512>>>(d, bytes, 256, 32); });
    timeit("bulk 704-B pieces", [&] { wr_bulk<<<grid, 512, 16 * 704>>>(d, bytes, 704); });
    timeit("bulk 2816-B pieces", [&] { wr_bulk<<<grid, 512, 16 * 2816>>>(d, bytes, 2816); });
  }
  return 0;
}
