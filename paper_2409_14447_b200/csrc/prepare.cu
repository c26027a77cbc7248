// prepare.cu — table preparation on the device.
//
// prepare_tables (pipeline.py:70-80) = filter_feasible (profiles.py:260-271:
// keep memory_required <= memory_map[size]) + optional
// restrict(process_counts=(1,)) (profiles.py:115-129), as kernel predicates
// over raw key-ordered segments: count kept points per segment (warp ballot),
// exclusive scan of the counts, then a stable warp-ballot compaction into the
// prepared (tp, lat) layout.  d_src keeps the raw index of every kept point
// so the host can decode winners' batch / process count.
#include <cuda_runtime.h>

#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

__device__ __forceinline__ bool keep_point(const parva_raw_tables& R, int64_t i, double cap, int single) {
  return R.d_mem[i] <= cap && (!single || R.d_procs[i] == 1);
}

__global__ void prep_count_kernel(parva_raw_tables R, const double* __restrict__ caps, int single,
                                  int32_t* __restrict__ seg_count_out) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= (int64_t)R.n_tables * 5) return;
  const double cap = caps[s % 5];
  const int64_t a = R.d_seg_start[s];
  const int n = R.d_seg_count[s];
  int cnt = 0;
  for (int j = 0; j < n; j += 32) {
    const bool k = j + lane < n && keep_point(R, a + j + lane, cap, single);
    cnt += __popc(__ballot_sync(0xffffffffu, k));
  }
  if (lane == 0) seg_count_out[s] = cnt;
}

__global__ void __launch_bounds__(1024) prep_scan_kernel(const int32_t* __restrict__ cnt, int64_t n,
                                                         int64_t* __restrict__ start, int64_t* __restrict__ total) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + tid;
    const int64_t v = i < n ? cnt[i] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int64_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      int64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += u;
      }
      warp_tot[lane] = wi - w;
    }
    __syncthreads();
    const int64_t c0 = carry_s;
    if (i < n) start[i] = c0 + warp_tot[warp] + incl - v;
    __syncthreads();
    if (tid == blockDim.x - 1) carry_s = c0 + warp_tot[warp] + incl;
    __syncthreads();
  }
  if (tid == 0) *total = carry_s;
}

__global__ void prep_scatter_kernel(parva_raw_tables R, const double* __restrict__ caps, int single,
                                    const int64_t* __restrict__ start, double2* __restrict__ pts,
                                    int32_t* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= (int64_t)R.n_tables * 5) return;
  const double cap = caps[s % 5];
  const int64_t a = R.d_seg_start[s];
  const int n = R.d_seg_count[s];
  int64_t o = start[s];
  for (int j = 0; j < n; j += 32) {
    const int64_t i = a + j + lane;
    const bool k = j + lane < n && keep_point(R, i, cap, single);
    const unsigned b = __ballot_sync(0xffffffffu, k);
    if (k) {
      const int64_t p = o + __popc(b & ((1u << lane) - 1u));
      pts[p] = make_double2(R.d_tp[i], R.d_lat[i]);
      src[p] = (int32_t)i;
    }
    o += __popc(b);
  }
}

}  // namespace parva

extern "C" int parva_prepare_tables(const parva_raw_tables* raw, const double* h_memcap5, int32_t single_process,
                                    double* d_pts, int64_t* d_seg_start, int32_t* d_seg_count, int32_t* d_src,
                                    int64_t* h_n_points, void* stream) {
  if (!raw || !h_memcap5 || !d_pts || !d_seg_start || !d_seg_count || !d_src || !h_n_points) return PARVA_BAD_INPUT;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nseg = (int64_t)raw->n_tables * 5;
  if (nseg == 0) { *h_n_points = 0; return PARVA_OK; }
  double* d_caps = nullptr;
  int64_t* d_total = nullptr;
  if (cudaMallocAsync(&d_caps, 5 * sizeof(double) + sizeof(int64_t), s) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  d_total = reinterpret_cast<int64_t*>(d_caps + 5);
  cudaMemcpyAsync(d_caps, h_memcap5, 5 * sizeof(double), cudaMemcpyHostToDevice, s);
  const int wpb = 8;
  const int grid = (int)((nseg + wpb - 1) / wpb);
  parva::prep_count_kernel<<<grid, wpb * 32, 0, s>>>(*raw, d_caps, single_process, d_seg_count);
  parva::prep_scan_kernel<<<1, 1024, 0, s>>>(d_seg_count, nseg, d_seg_start, d_total);
  parva::prep_scatter_kernel<<<grid, wpb * 32, 0, s>>>(*raw, d_caps, single_process, d_seg_start,
                                                      reinterpret_cast<double2*>(d_pts), d_src);
  int64_t tot = 0;
  cudaMemcpyAsync(&tot, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFreeAsync(d_caps, s);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return PARVA_LAUNCH_ERROR;
  *h_n_points = tot;
  return PARVA_OK;
}
