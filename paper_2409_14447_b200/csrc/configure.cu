// configure.cu — K1 configure_sweep and K0 build_index (sm_100a).
//
// K1 replaces configure_service (configurator.py:189-191) for one query per
// row: decide_best_triplets (:93-124) as a streaming per-size argmax over the
// queried table, then select_optimal_segment + match_demand (:127-186).
// It is HBM-bound (16 B per prepared point): a producer warp streams each
// (table, size class) segment through a ring of shared-memory stages with
// 1-D bulk copies (cp.async.bulk -> UBLKCP) completing on mbarriers; eight
// consumer warps scan the stage and keep one running argmax per thread, then
// reduce with warp shuffles (exact: the comparator is a strict total order,
// SURVEY.md fact 4).
#include <cuda_runtime.h>

#include "parva_async.cuh"
#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

constexpr int SW_WARPS = 8;                    // consumer warps
constexpr int SW_THREADS = (SW_WARPS + 1) * 32;
constexpr int SW_CH = 2048;                    // points per chunk
constexpr int SW_STAGES = 3;

struct SweepSmem {
  double tp[SW_STAGES][SW_CH + 2];
  double lat[SW_STAGES][SW_CH + 2];
  uint64_t full[SW_STAGES];
  uint64_t empty[SW_STAGES];
  Cand wbest[SW_WARPS][5];
  Cand fin[5];
};

struct ChunkIter {
  int64_t a, b, s0;  // chunk [a, b) of segment starting at s0
};

__global__ void __launch_bounds__(SW_THREADS) configure_sweep_kernel(
    const double* __restrict__ tp, const double* __restrict__ lat,
    const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count, int n_tables,
    int nq, const int32_t* __restrict__ q_table, const double* __restrict__ q_rate,
    const double* __restrict__ q_bound, parva_config_record* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SweepSmem& S = *reinterpret_cast<SweepSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SW_STAGES; s++) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], SW_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == SW_WARPS) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      for (int q = blockIdx.x; q < nq; q += gridDim.x) {
        const int t = q_table[q];
        if (t < 0 || t >= n_tables) continue;
        for (int c = 0; c < 5; c++) {
          const int64_t s0 = seg_start[t * 5 + c];
          const int n = seg_count[t * 5 + c];
          for (int off = 0; off < n; off += SW_CH, it++) {
            const int64_t a = s0 + off, b = s0 + min(n, off + SW_CH);
            const int64_t a2 = a & ~int64_t(1), b2 = (b + 1) & ~int64_t(1);
            const uint32_t bytes = uint32_t(b2 - a2) * 8u;
            const int st = it % SW_STAGES;
            mbar_wait(&S.empty[st], ((it / SW_STAGES) & 1) ^ 1);
            mbar_arrive_expect_tx(&S.full[st], 2 * bytes);
            bulk_g2s(S.tp[st], tp + a2, bytes, &S.full[st], pol);
            bulk_g2s(S.lat[st], lat + a2, bytes, &S.full[st], pol);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int tid = threadIdx.x;  // 0 .. 255
  uint32_t it = 0;
  for (int q = blockIdx.x; q < nq; q += gridDim.x) {
    const int t = q_table[q];
    if (t < 0 || t >= n_tables) {
      if (tid == 0) {
        parva_config_record r = {};
        for (int c = 0; c < 5; c++) r.best[c] = -1;
        r.opt_sc = -1; r.last_sc = -1; r.status = PARVA_BAD_INPUT;
        out[q] = r;
      }
      continue;
    }
    const double bound = q_bound[q];
    for (int c = 0; c < 5; c++) {
      const int64_t s0 = seg_start[t * 5 + c];
      const int n = seg_count[t * 5 + c];
      Cand best{0.0, 0.0, -1};
      for (int off = 0; off < n; off += SW_CH, it++) {
        const int64_t a = s0 + off, b = s0 + min(n, off + SW_CH);
        const int64_t a2 = a & ~int64_t(1);
        const int st = it % SW_STAGES;
        mbar_wait(&S.full[st], (it / SW_STAGES) & 1);
        const double* stp = S.tp[st];
        const double* slat = S.lat[st];
        const int lo = int(a - a2), hi = int(b - a2);
#pragma unroll 4
        for (int j = lo + tid; j < hi; j += SW_WARPS * 32) {
          const double l = slat[j];
          if (l < bound) {
            Cand cnd{stp[j], l, int(a2 - s0) + j};
            if (better(cnd, best)) best = cnd;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[st]);
      }
      best = warp_argmax(best);
      if (lane == 0) S.wbest[warp][c] = best;
    }
    named_bar_sync(1, SW_WARPS * 32);
    if (tid < 5) {
      Cand b = S.wbest[0][tid];
      for (int w = 1; w < SW_WARPS; w++)
        if (better(S.wbest[w][tid], b)) b = S.wbest[w][tid];
      S.fin[tid] = b;
    }
    named_bar_sync(1, SW_WARPS * 32);
    if (tid == 0) {
      parva_config_record r = {};
      double tpc[5];
      for (int c = 0; c < 5; c++) {
        r.best[c] = (int16_t)S.fin[c].idx;
        tpc[c] = S.fin[c].idx >= 0 ? S.fin[c].tp : 0.0;
      }
      match_demand(tpc, q_rate[q], r);
      out[q] = r;
    }
  }
}

// ------------------------------------------------------------------- K0
// Latency-sorted prefix-argmax index per segment (one CTA per segment).
constexpr int IDX_MAX = 4096;

__global__ void __launch_bounds__(256) build_index_kernel(
    const double* __restrict__ tp, const double* __restrict__ lat,
    const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count,
    double* __restrict__ lat_sorted, uint16_t* __restrict__ best_out, int* __restrict__ err) {
  __shared__ double sl[IDX_MAX];
  __shared__ uint16_t order[IDX_MAX];
  const int s = blockIdx.x;
  const int64_t s0 = seg_start[s];
  const int n = seg_count[s];
  if (n > IDX_MAX) {
    if (threadIdx.x == 0) atomicExch(err, 1);
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) sl[i] = lat[s0 + i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double li = sl[i];
    int rank = 0;
    for (int j = 0; j < n; j++) {
      const double lj = sl[j];
      rank += (lj < li) || (lj == li && j < i);
    }
    order[rank] = (uint16_t)i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand b{0.0, 0.0, -1};
    for (int r = 0; r < n; r++) {
      const int i = order[r];
      Cand c{tp[s0 + i], sl[i], i};
      if (better(c, b)) b = c;
      lat_sorted[s0 + r] = sl[i];
      best_out[s0 + r] = (uint16_t)b.idx;
    }
  }
}

}  // namespace parva

// ------------------------------------------------------------------ launchers
namespace parva {

int launch_configure_sweep(const parva_tables* t, int nq, const int32_t* q_table,
                           const double* q_rate, const double* q_bound,
                           parva_config_record* out, cudaStream_t stream) {
  if (nq <= 0) return PARVA_OK;
  static int blocks_per_sm = -1, n_sm = 0;
  const size_t smem = sizeof(SweepSmem);
  if (blocks_per_sm < 0) {
    cudaFuncSetAttribute(configure_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, configure_sweep_kernel, SW_THREADS, smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int grid = n_sm * blocks_per_sm;
  if (grid > nq) grid = nq;
  configure_sweep_kernel<<<grid, SW_THREADS, smem, stream>>>(
      t->d_tp, t->d_lat, t->d_seg_start, t->d_seg_count, t->n_tables, nq, q_table, q_rate, q_bound, out);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int launch_build_index(const parva_tables* t, parva_index* idx, int* d_err, cudaStream_t stream) {
  const int nseg = t->n_tables * 5;
  if (nseg <= 0) return PARVA_OK;
  build_index_kernel<<<nseg, 256, 0, stream>>>(t->d_tp, t->d_lat, t->d_seg_start, t->d_seg_count,
                                               idx->d_lat_sorted, idx->d_best, d_err);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva
