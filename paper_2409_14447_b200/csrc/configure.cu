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

#ifndef PARVA_SW_WARPS
#define PARVA_SW_WARPS 14
#endif
#ifndef PARVA_SW_CH
#define PARVA_SW_CH 256
#endif
#ifndef PARVA_SW_STAGES
#define PARVA_SW_STAGES 4
#endif
constexpr int SW_WARPS = PARVA_SW_WARPS;       // warps per CTA, one table each at a time
constexpr int SW_THREADS = SW_WARPS * 32;
constexpr int SW_CH = PARVA_SW_CH;             // points per chunk (16 B each)
constexpr int SW_STAGES = PARVA_SW_STAGES;     // chunks in flight per warp

struct alignas(128) SweepWarpSmem {
  double2 pts[SW_STAGES][SW_CH];   // (tp, lat)
  uint64_t full[SW_STAGES];
};

// Walks (query, size class, chunk) for one warp: queries q0, q0+stride, ...
// The current table's 5 segment offsets/counts live in lanes 0..4.
struct ChunkCursor {
  int q, c, off, n;
  int64_t s0;
  int64_t lane_start;   // lane c: seg_start of the current table, class c
  int lane_count;       // lane c: seg_count
  bool valid;           // current q has a valid table

  __device__ void load_table(const int32_t* q_table, const int64_t* seg_start, const int32_t* seg_count,
                             int n_tables, int lane) {
    const int t = q_table[q];
    valid = t >= 0 && t < n_tables;
    lane_start = 0; lane_count = 0;
    if (valid && lane < 5) { lane_start = seg_start[t * 5 + lane]; lane_count = seg_count[t * 5 + lane]; }
  }
  __device__ void select(int cc) {
    c = cc;
    s0 = __shfl_sync(0xffffffffu, lane_start, cc);
    n = __shfl_sync(0xffffffffu, lane_count, cc);
  }
  // move to the next non-empty chunk at or after (q, c, off); false when done
  __device__ bool settle(const int32_t* q_table, const int64_t* seg_start, const int32_t* seg_count,
                         int n_tables, int nq, int stride, int lane) {
    while (q < nq) {
      if (valid) {
        while (c < 5) {
          if (off < n) return true;
          off = 0;
          if (c + 1 < 5) select(c + 1); else c = 5;
        }
      }
      q += stride;
      if (q >= nq) break;
      load_table(q_table, seg_start, seg_count, n_tables, lane);
      off = 0;
      select(0);
    }
    return false;
  }
};

__global__ void __launch_bounds__(SW_THREADS) configure_sweep_kernel(
    const double2* __restrict__ pts,
    const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count, int n_tables,
    int nq, const int32_t* __restrict__ q_table, const double* __restrict__ q_rate,
    const double* __restrict__ q_bound, parva_config_record* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SweepWarpSmem& S = reinterpret_cast<SweepWarpSmem*>(smem_raw)[warp];
  const int gw = blockIdx.x * SW_WARPS + warp;
  const int stride = gridDim.x * SW_WARPS;
  if (gw >= nq) return;

  if (lane == 0) {
    for (int s = 0; s < SW_STAGES; s++) mbar_init(&S.full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();

  // producer cursor: up to SW_STAGES chunks ahead of the consumer
  ChunkCursor P;
  P.q = gw; P.off = 0;
  P.load_table(q_table, seg_start, seg_count, n_tables, lane);
  P.select(0);
  bool p_ok = P.settle(q_table, seg_start, seg_count, n_tables, nq, stride, lane);
  uint32_t issued = 0;
  auto issue = [&]() {
    const int64_t a = P.s0 + P.off;
    const uint32_t bytes = uint32_t(min(P.n - P.off, SW_CH)) * 16u;
    const int st = issued % SW_STAGES;
    if (lane == 0) {
      mbar_arrive_expect_tx(&S.full[st], bytes);
      bulk_g2s(S.pts[st], pts + a, bytes, &S.full[st], pol);
    }
    issued++;
    P.off += SW_CH;
    p_ok = P.settle(q_table, seg_start, seg_count, n_tables, nq, stride, lane);
  };
  for (int k = 0; k < SW_STAGES && p_ok; k++) issue();

  // deferred epilogue: lane L holds the per-size winners of the L-th pending query
  int pend_q = -1;
  int p_idx0 = -1, p_idx1 = -1, p_idx2 = -1, p_idx3 = -1, p_idx4 = -1;
  double p_tp0 = 0, p_tp1 = 0, p_tp2 = 0, p_tp3 = 0, p_tp4 = 0;
  int npend = 0;
  auto flush = [&]() {
    if (pend_q >= 0) {
      parva_config_record r = {};
      r.best[0] = (int16_t)p_idx0; r.best[1] = (int16_t)p_idx1; r.best[2] = (int16_t)p_idx2;
      r.best[3] = (int16_t)p_idx3; r.best[4] = (int16_t)p_idx4;
      double tpc[5] = {p_idx0 >= 0 ? p_tp0 : 0.0, p_idx1 >= 0 ? p_tp1 : 0.0, p_idx2 >= 0 ? p_tp2 : 0.0,
                       p_idx3 >= 0 ? p_tp3 : 0.0, p_idx4 >= 0 ? p_tp4 : 0.0};
      match_demand(tpc, q_rate[pend_q], r);
      const uint4* src = reinterpret_cast<const uint4*>(&r);
      uint4* dst = reinterpret_cast<uint4*>(out + pend_q);
      dst[0] = src[0];
      dst[1] = src[1];
    }
    pend_q = -1; p_idx0 = p_idx1 = p_idx2 = p_idx3 = p_idx4 = -1;
    npend = 0;
  };

  // consumer cursor over the same sequence
  ChunkCursor Q;
  uint32_t consumed = 0;
  for (Q.q = gw; Q.q < nq; Q.q += stride) {
    Q.load_table(q_table, seg_start, seg_count, n_tables, lane);
    if (!Q.valid) {
      if (lane == 0) {
        parva_config_record r = {};
        for (int c = 0; c < 5; c++) r.best[c] = -1;
        r.opt_sc = -1; r.last_sc = -1; r.status = PARVA_BAD_INPUT;
        out[Q.q] = r;
      }
      continue;
    }
    const double bound = q_bound[Q.q];
    const int slot = npend++;
#pragma unroll 1
    for (int c = 0; c < 5; c++) {
      Q.select(c);
      // lane-local running best: a lane sees its points in increasing
      // position, so (tp desc, lat asc) decides and later equal points lose
      // on position; tp > 0, so btp = 0 means "none yet"
      double btp = 0.0, blat = 0.0;
      int bidx = -1;
      for (int off = 0; off < Q.n; off += SW_CH) {
        const int hi = min(Q.n - off, SW_CH);
        const int st = consumed % SW_STAGES;
        mbar_wait(&S.full[st], (consumed / SW_STAGES) & 1);
        const double2* sp = S.pts[st];
        if (hi == SW_CH) {
#pragma unroll
          for (int j0 = 0; j0 < SW_CH; j0 += 32) {
            const double2 v = sp[j0 + lane];
            const bool take = v.y < bound && (v.x > btp || (v.x == btp && v.y < blat));
            btp = take ? v.x : btp;
            blat = take ? v.y : blat;
            bidx = take ? off + j0 + lane : bidx;
          }
        } else {
          for (int j = lane; j < hi; j += 32) {
            const double2 v = sp[j];
            const bool take = v.y < bound && (v.x > btp || (v.x == btp && v.y < blat));
            btp = take ? v.x : btp;
            blat = take ? v.y : blat;
            bidx = take ? off + j : bidx;
          }
        }
        consumed++;
        __syncwarp();
        if (p_ok) issue();
      }
      Cand best{btp, blat, bidx};
      best = warp_argmax(best);
      if (lane == slot) {
        switch (c) {
          case 0: p_idx0 = best.idx; p_tp0 = best.tp; break;
          case 1: p_idx1 = best.idx; p_tp1 = best.tp; break;
          case 2: p_idx2 = best.idx; p_tp2 = best.tp; break;
          case 3: p_idx3 = best.idx; p_tp3 = best.tp; break;
          default: p_idx4 = best.idx; p_tp4 = best.tp; break;
        }
        pend_q = Q.q;
      }
    }
    if (npend == 32) flush();
  }
  flush();
}

// ------------------------------------------------------------------- K0
// Latency-sorted prefix-argmax index per segment (one CTA per segment).
constexpr int IDX_MAX = 4096;

__global__ void __launch_bounds__(256) build_index_kernel(
    const double2* __restrict__ pts,
    const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count,
    double* __restrict__ lat_sorted, uint16_t* __restrict__ best_out, double* __restrict__ tp_out,
    int* __restrict__ err) {
  __shared__ double sl[IDX_MAX];
  __shared__ uint16_t order[IDX_MAX];
  const int s = blockIdx.x;
  const int64_t s0 = seg_start[s];
  const int n = seg_count[s];
  if (n > IDX_MAX) {
    if (threadIdx.x == 0) atomicExch(err, 1);
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sl[i] = pts[s0 + i].y;
    tp_out[s0 + i] = pts[s0 + i].x;
  }
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
      Cand c{pts[s0 + i].x, sl[i], i};
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
  // per-device launch configuration (attributes are per device context)
  static int s_bps[kMaxDevices], s_nsm[kMaxDevices];
  const size_t smem = sizeof(SweepWarpSmem) * SW_WARPS;
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= kMaxDevices - 1;
  if (!s_nsm[dev]) {
    cudaFuncSetAttribute(configure_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaDeviceGetAttribute(&s_nsm[dev], cudaDevAttrMultiProcessorCount, dev);
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, configure_sweep_kernel, SW_THREADS, smem);
    s_bps[dev] = bps < 1 ? 1 : bps;
  }
  const int blocks_per_sm = s_bps[dev], n_sm = s_nsm[dev];
  int grid = n_sm * blocks_per_sm;
  const int need = (nq + SW_WARPS - 1) / SW_WARPS;
  if (grid > need) grid = need;
  configure_sweep_kernel<<<grid, SW_THREADS, smem, stream>>>(
      reinterpret_cast<const double2*>(t->d_pts), t->d_seg_start, t->d_seg_count, t->n_tables, nq, q_table, q_rate, q_bound, out);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int launch_build_index(const parva_tables* t, parva_index* idx, int* d_err, cudaStream_t stream) {
  const int nseg = t->n_tables * 5;
  if (nseg <= 0) return PARVA_OK;
  build_index_kernel<<<nseg, 256, 0, stream>>>(reinterpret_cast<const double2*>(t->d_pts), t->d_seg_start, t->d_seg_count,
                                               idx->d_lat_sorted, idx->d_best, idx->d_tp, d_err);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva
