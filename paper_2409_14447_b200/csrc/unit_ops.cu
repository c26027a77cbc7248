// unit_ops.cu — batched single-function kernels behind the fine-grained
// API calls (select_optimal_segment, match_demand, propose_small_segments)
// on caller-ordered triplet lists.  The device functions are the same ones
// the fused kernels use; one thread per list.
#include <cuda_runtime.h>

#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

// select_optimal_segment (configurator.py:127-139) in caller order.
__device__ inline int select_optimal_list(const int32_t* size, const double* tp, int n) {
  int best = 0;
  for (int i = 1; i < n; i++) {
    const double lhs = __dmul_rn(tp[i], (double)size[best]);
    const double rhs = __dmul_rn(tp[best], (double)size[i]);
    if (lhs > rhs || (lhs == rhs && size[i] > size[best])) best = i;
  }
  return best;
}

__global__ void select_optimal_kernel(int n_lists, const int32_t* off, const int32_t* size, const double* tp,
                                      int32_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_lists) return;
  const int a = off[k], n = off[k + 1] - a;
  out[k] = n > 0 ? a + select_optimal_list(size + a, tp + a, n) : -1;
}

// match_demand (configurator.py:142-186) on an arbitrary best_triplets list.
__global__ void match_demand_kernel(int n_lists, const int32_t* off, const int32_t* size, const double* tp,
                                    const double* rate, int32_t* opt_out, int32_t* last_out,
                                    int64_t* count_out, double* cov_out, uint8_t* status_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_lists) return;
  const int a = off[k], n = off[k + 1] - a;
  opt_out[k] = -1; last_out[k] = -1; count_out[k] = 0; cov_out[k] = 0.0;
  if (n <= 0) { status_out[k] = PARVA_BAD_INPUT; return; }
  const int o = select_optimal_list(size + a, tp + a, n);
  const double topt = tp[a + o], r = rate[k];
  opt_out[k] = a + o;
  long long count = 0;
  if (r > 0.0) {
    const double q = floor(__ddiv_rn(r, topt));
    if (!(q <= kCountLimit)) { status_out[k] = PARVA_COUNT_OVERFLOW; return; }
    count = (long long)q;
  }
  double remaining = __dsub_rn(r, __dmul_rn((double)count, topt));
  const double m = (1.0 > r) ? 1.0 : r;
  if (remaining <= __dmul_rn(1e-9, m)) remaining = 0.0;
  int last = -1;
  if (remaining > 0.0) {
    // sorted(best_triplets, key=instance_size): stable selection by (size, position)
    int prev_size = -2147483647 - 1, prev_pos = -1;
    for (int step = 0; step < n && last < 0; step++) {
      int pick = -1;
      for (int i = 0; i < n; i++) {
        const bool after = size[a + i] > prev_size || (size[a + i] == prev_size && i > prev_pos);
        if (!after) continue;
        if (pick < 0 || size[a + i] < size[a + pick]) pick = i;
      }
      prev_size = size[a + pick]; prev_pos = pick;
      if (tp[a + pick] >= remaining) last = pick;
    }
    if (last < 0) {
      int fb = 0;
      for (int i = 1; i < n; i++) if (tp[a + i] > tp[a + fb]) fb = i;
      if (tp[a + fb] >= remaining) last = fb;
      else { status_out[k] = PARVA_RESIDUAL_UNCOVERABLE; return; }
    }
  }
  last_out[k] = last >= 0 ? a + last : -1;
  count_out[k] = count;
  cov_out[k] = coverage_sum(topt, count, last >= 0, last >= 0 ? tp[a + last] : 0.0);
  status_out[k] = PARVA_OK;
}

__global__ void propose_kernel(int n, const double* tp1, const double* tp2, const double* freed, int64_t* k2,
                               int64_t* k1, uint8_t* ok) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  long long a, b;
  ok[k] = propose_small(tp1[k], tp2[k], freed[k], a, b) ? 1 : 0;
  k2[k] = a;
  k1[k] = b;
}

}  // namespace parva

extern "C" {

int parva_select_optimal_lists(int32_t n_lists, const int32_t* d_off, const int32_t* d_size, const double* d_tp,
                               int32_t* d_out, void* stream) {
  if (n_lists <= 0) return PARVA_OK;
  parva::select_optimal_kernel<<<(n_lists + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n_lists, d_off, d_size,
                                                                                        d_tp, d_out);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int parva_match_demand_lists(int32_t n_lists, const int32_t* d_off, const int32_t* d_size, const double* d_tp,
                             const double* d_rate, int32_t* d_opt, int32_t* d_last, int64_t* d_count,
                             double* d_coverage, uint8_t* d_status, void* stream) {
  if (n_lists <= 0) return PARVA_OK;
  parva::match_demand_kernel<<<(n_lists + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      n_lists, d_off, d_size, d_tp, d_rate, d_opt, d_last, d_count, d_coverage, d_status);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int parva_propose_small_batch(int32_t n, const double* d_tp1, const double* d_tp2, const double* d_freed,
                              int64_t* d_k2, int64_t* d_k1, uint8_t* d_ok, void* stream) {
  if (n <= 0) return PARVA_OK;
  parva::propose_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, d_tp1, d_tp2, d_freed, d_k2, d_k1,
                                                                          d_ok);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // extern "C"
