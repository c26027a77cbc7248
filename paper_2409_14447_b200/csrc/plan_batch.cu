// plan_batch.cu — K2: fused per-scenario planner (sm_100a).
//
// Replaces plan_services' timed region (pipeline.py:95-103) for a batch of
// independent scenarios: configure_service x N (configurator.py:189-191),
// relocate_segments (allocator.py:292-316), optimize_allocation
// (allocator.py:362-443).  One warp plans one scenario:
//   * configure: lane = service; per size class a binary search over the
//     latency-sorted prefix-argmax index held in shared memory (exact:
//     the points with lat < bound are a prefix of the sorted order and the
//     argmax under a total order is prefix-decomposable);
//   * relocate / optimize: lane = GPU; a GPU is a 7-bit slot mask; first-fit
//     is one ballot over find_start(mask) (cursorless first-fit is
//     equivalent to the reference's cursors); the
//     freed_rate ledger lives in lane = service registers, snapshot/restore
//     is a register copy.
// Scenarios beyond the 128-byte record's limits report PARVA_CAPACITY and
// are re-planned by the general kernel (plan_general.cu).
#include <cuda_runtime.h>

#include "parva_async.cuh"
#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

constexpr int PB_WARPS = 16;
constexpr int PB_THREADS = PB_WARPS * 32;
constexpr int QCAP = 224;                 // > 31 GPUs x 7 slots: longer queues cannot fit

struct WarpScratch {
  double cat_tp[32 * 5];                  // best tp per (service, size class); 0 = absent
  uint16_t lst[32][8];                    // per GPU placement list: cat << 3 | slot
  uint16_t bak[32][8];                    // relocation result (regression fallback)
  uint8_t q2[QCAP];
  uint8_t q1[QCAP];
  uint8_t undo[2 * QCAP];
  uint16_t diag[32];                      // optimize diagnostics, in order
  parva_plan_record rec;
};


__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double unallocated(int total, int n) {
  if (n == 0) return 0.0;
  return __dsub_rn(1.0, __ddiv_rn((double)total, (double)(7 * n)));
}

// configure one service from the index: for each size class, count = number
// of points with lat < bound (binary search over the latency-sorted
// segment), winner = prefix argmax at count-1.  The five searches advance in
// lockstep (branch-free power-of-two steps) so their loads overlap.
__device__ __forceinline__ void configure_indexed(const double* lat_s, const uint16_t* best_s,
                                                  const double* tp, int tp_stride, const int* seg_s,
                                                  const int* seg_n, int t, double bound,
                                                  double rate, parva_config_record& r,
                                                  double tpc[5]) {
  int s0[5], n[5], lo[5];
  int nmax = 0;
#pragma unroll
  for (int c = 0; c < 5; c++) {
    s0[c] = seg_s[t * 5 + c];
    n[c] = seg_n[t * 5 + c];
    lo[c] = 0;
    nmax = max(nmax, n[c]);
  }
  for (int step = nmax ? 1 << (31 - __clz(nmax)) : 0; step > 0; step >>= 1) {
#pragma unroll
    for (int c = 0; c < 5; c++) {
      const int probe = lo[c] + step;
      if (probe <= n[c] && lat_s[s0[c] + probe - 1] < bound) lo[c] = probe;
    }
  }
#pragma unroll
  for (int c = 0; c < 5; c++) {
    const int b = lo[c] ? (int)best_s[s0[c] + lo[c] - 1] : -1;
    r.best[c] = (int16_t)b;
    tpc[c] = b >= 0 ? tp[(s0[c] + b) * tp_stride] : 0.0;
  }
  match_demand(tpc, rate, r);
  if (r.status == PARVA_INFEASIBLE_SLO) r.opt_sc = -1;
}

// one relocation size class (allocator.py:284-289): services in input order,
// opt copies then last; c is a compile-time constant in each instantiation
template <int c>
__device__ __forceinline__ void relocate_class(WarpScratch& W, int lane, int n, int my_opt, long long my_count,
                                               int my_last, uint32_t& mask, int& ngpc, int& len, int& ngpus,
                                               int& status) {
  const int my_reps = lane < n ? (my_opt == c ? (int)my_count : 0) + (my_last == c ? 1 : 0) : 0;
  unsigned pending = __ballot_sync(0xffffffffu, my_reps > 0);
  while (pending && status == PARVA_OK) {
    const int s = __ffs(pending) - 1;
    pending &= pending - 1;
    const int reps = __shfl_sync(0xffffffffu, my_reps, s);
    const uint16_t cat3 = (uint16_t)((s * 5 + c) << 3);
    for (int r = 0; r < reps; r++) {
      int st = lane < ngpus ? find_start(mask, c) : -1;
      const unsigned b = __ballot_sync(0xffffffffu, st >= 0);
      int g;
      if (b) g = __ffs(b) - 1;
      else {
        if (ngpus >= PARVA_PLAN_MAX_GPUS) { status = PARVA_CAPACITY; break; }
        g = ngpus++;
        st = find_start(0u, c);
      }
      if (lane == g) {
        mask |= footprint(c, st);
        ngpc += size_of_class(c);
        W.lst[g][len++] = (uint16_t)(cat3 | st);
      }
    }
  }
}

// Index view: segment tables always in shared memory; latency-sorted
// index + tp either bulk-copied into shared memory or read from global.
struct IndexView {
  const int* seg_s;
  const int* seg_n;
  const double* lat;
  const uint16_t* best;
  const double* tp;
  int tp_stride;
};

__device__ __forceinline__ IndexView load_index(const PlanArgs& A, uint8_t* base, bool need_lat_best,
                                                uint64_t* bar) {
  const int T5 = A.n_tables * 5;
  int* seg_s = reinterpret_cast<int*>(base);
  int* seg_n = seg_s + T5;
  for (int i = threadIdx.x; i < T5; i += blockDim.x) {
    seg_s[i] = (int)A.seg_start[i];
    seg_n[i] = A.seg_count[i];
  }
  IndexView V{seg_s, seg_n, A.idx_lat, A.idx_best, A.pts, 2};
  if (A.smem_index) {
    const size_t off = (size_t(T5) * 8 + 15) & ~size_t(15);
    const uint32_t b_dbl = uint32_t((A.n_points * 8 + 15) & ~int64_t(15));
    const uint32_t b_u16 = uint32_t((A.n_points * 2 + 15) & ~int64_t(15));
    double* tp_w = reinterpret_cast<double*>(base + off);
    double* lat_w = reinterpret_cast<double*>(base + off + b_dbl);
    uint16_t* best_w = reinterpret_cast<uint16_t*>(base + off + 2 * size_t(b_dbl));
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, b_dbl + (need_lat_best ? b_dbl + b_u16 : 0u));
      const uint64_t pol = policy_evict_last();
      bulk_g2s(tp_w, A.idx_tp, b_dbl, bar, pol);
      if (need_lat_best) {
        bulk_g2s(lat_w, A.idx_lat, b_dbl, bar, pol);
        bulk_g2s(best_w, A.idx_best, b_u16, bar, pol);
      }
    }
    __syncthreads();
    mbar_wait(bar, 0);
    V.tp = tp_w;
    V.tp_stride = 1;
    if (need_lat_best) { V.lat = lat_w; V.best = best_w; }
  }
  __syncthreads();
  return V;
}

__device__ __forceinline__ void store_config(const PlanArgs& A, int64_t i, const parva_config_record& r) {
  if (A.cfg_format == PARVA_CFG_TINY) {
    parva_config_tiny k;
#pragma unroll
    for (int c = 0; c < 5; c++) k.best[c] = r.best[c] < 0 ? 255 : (uint8_t)r.best[c];
    k.opt_last = (uint8_t)((r.opt_sc < 0 ? 15 : r.opt_sc) | (r.last_sc < 0 ? 15 : r.last_sc) << 4);
    k.status_flags = (uint8_t)(r.status | (r.count > 255 ? 0x80 : 0));
    k.count = (uint8_t)(r.count > 255 ? 255 : r.count);
    reinterpret_cast<uint2*>(A.cfg)[i] = *reinterpret_cast<const uint2*>(&k);
  } else if (A.cfg_format == PARVA_CFG_COMPACT) {
    parva_config_compact k;
#pragma unroll
    for (int c = 0; c < 5; c++) k.best[c] = r.best[c];
    k.opt_sc = r.opt_sc; k.last_sc = r.last_sc; k.status = r.status;
    k.flags = r.count > 65535 ? 1 : 0;
    k.count = (uint16_t)(r.count > 65535 ? 65535 : r.count);
    reinterpret_cast<uint4*>(A.cfg)[i] = *reinterpret_cast<const uint4*>(&k);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<parva_config_record*>(A.cfg) + i);
    dst[0] = reinterpret_cast<const uint4*>(&r)[0];
    dst[1] = reinterpret_cast<const uint4*>(&r)[1];
  }
}

// K2a: configure_service for every service of the batch, one thread each
// (configurator.py:189-191 via the prefix-argmax index).
constexpr int CF_THREADS = 256;
__global__ void __launch_bounds__(CF_THREADS) configure_services_kernel(PlanArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t bar;
  // let K2b's CTAs be scheduled now: they load their index while we work and
  // wait for our records at griddepcontrol.wait (programmatic dependent launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const IndexView V = load_index(A, smem_raw, true, &bar);
  const int64_t lo = A.scen_off[0], hi = lo + A.n_svc;
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    parva_config_record r = {};
    double tpc[5];
    const int t = A.svc_table16 ? (int)A.svc_table16[i] : A.svc_table[i];
    if (t < 0 || t >= A.n_tables) {
      for (int c = 0; c < 5; c++) r.best[c] = -1;
      r.opt_sc = -1; r.last_sc = -1; r.status = PARVA_BAD_INPUT;
    } else {
      configure_indexed(V.lat, V.best, V.tp, V.tp_stride, V.seg_s, V.seg_n, t, A.svc_bound[i], A.svc_rate[i], r, tpc);
    }
    store_config(A, i, r);
  }
}

// K2b: relocate + optimize, one warp per scenario, from the config records.
__global__ void __launch_bounds__(PB_THREADS, 2) plan_batch_kernel(PlanArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  WarpScratch* scratch = reinterpret_cast<WarpScratch*>(smem_raw);
  __shared__ uint64_t bar;
  const IndexView V = load_index(A, smem_raw + sizeof(WarpScratch) * PB_WARPS, false, &bar);
  // config records come from K2a (launched before us with PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpScratch& W = scratch[warp];
  const int gwarps = gridDim.x * PB_WARPS;

  for (int k = blockIdx.x * PB_WARPS + warp; k < A.n_scen; k += gwarps) {
    const int a0 = A.scen_off[k];
    const int n = A.scen_off[k + 1] - a0;
    reinterpret_cast<uint32_t*>(&W.rec)[lane] = 0u;

    // ------------------------------------------------ configured services
    int err_status = 0, err_svc = 0;
    int my_opt = -1, my_last = -1;
    long long my_count = 0;
    if (n <= PARVA_PLAN_MAX_SERVICES) {
      int st = PARVA_OK;
      if (lane < n) {
        const int i = a0 + lane;
        int16_t best[5];
        if (A.cfg_format == PARVA_CFG_TINY) {
          const parva_config_tiny r = reinterpret_cast<const parva_config_tiny*>(A.cfg)[i];
#pragma unroll
          for (int c = 0; c < 5; c++) best[c] = r.best[c] == 255 ? -1 : (int16_t)r.best[c];
          my_opt = (r.opt_last & 15) == 15 ? -1 : (r.opt_last & 15);
          my_last = (r.opt_last >> 4) == 15 ? -1 : (r.opt_last >> 4);
          my_count = (r.status_flags & 0x80) ? (long long)1 << 40 : r.count;   // saturated: cannot fit
          st = r.status_flags & 0x7F;
        } else if (A.cfg_format == PARVA_CFG_COMPACT) {
          const parva_config_compact r = reinterpret_cast<const parva_config_compact*>(A.cfg)[i];
#pragma unroll
          for (int c = 0; c < 5; c++) best[c] = r.best[c];
          my_opt = r.opt_sc; my_last = r.last_sc; my_count = r.count; st = r.status;
        } else {
          const parva_config_record r = reinterpret_cast<const parva_config_record*>(A.cfg)[i];
#pragma unroll
          for (int c = 0; c < 5; c++) best[c] = r.best[c];
          my_opt = r.opt_sc; my_last = r.last_sc; my_count = r.count; st = r.status;
        }
        const int t = A.svc_table16 ? (int)A.svc_table16[i] : A.svc_table[i];
#pragma unroll
        for (int c = 0; c < 5; c++)
          W.cat_tp[lane * 5 + c] =
              (st != PARVA_BAD_INPUT && best[c] >= 0) ? V.tp[(V.seg_s[t * 5 + c] + best[c]) * V.tp_stride] : 0.0;
      }
      const unsigned bad = __ballot_sync(0xffffffffu, lane < n && st != PARVA_OK);
      if (bad) {
        err_svc = __ffs(bad) - 1;
        err_status = __shfl_sync(0xffffffffu, st, err_svc);
      }
    }
    __syncwarp();

    int status = PARVA_OK;
    bool spill = false;
    if (n > PARVA_PLAN_MAX_SERVICES) status = PARVA_CAPACITY;
    else if (err_status) status = err_status;
    else {
      const long long segs = warp_sum_ll(lane < n ? my_count + (my_last >= 0) : 0);
      if (segs > 32 * 7) status = PARVA_CAPACITY;
    }

    // per-lane GPU state (lane = GPU index) and ledger state (lane = service)
    uint32_t mask = 0;
    int ngpc = 0, len = 0, ngpus = 0;
    double freed = 0.0;
    int order = 0;
    bool fallback = false;
    int nd = 0, n_before = 0;

    if (status == PARVA_OK) {
      // --------------------------------------------- relocate_segments
      // queue order (allocator.py:46-51): size classes 7,4,3,2,1
      relocate_class<4>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, status);
      if (status == PARVA_OK) relocate_class<3>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, status);
      if (status == PARVA_OK) relocate_class<2>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, status);
      if (status == PARVA_OK) relocate_class<1>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, status);
      if (status == PARVA_OK) relocate_class<0>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, status);
    }
    __syncwarp();

    if (status == PARVA_OK) {
      n_before = ngpus;
      const int total_before = warp_sum_i(lane < ngpus ? ngpc : 0);
      *reinterpret_cast<uint4*>(W.bak[lane]) = *reinterpret_cast<const uint4*>(W.lst[lane]);
      const int bak_len = len, bak_ngpc = ngpc;
      const uint32_t bak_mask = mask;

      if (A.optimize) {
        // ----------------------------------------- optimize_allocation
        int next = 0;
        for (int index = ngpus - 1; index >= 0; index--) {
          const int nl = __shfl_sync(0xffffffffu, len, index);
          const int ng = __shfl_sync(0xffffffffu, ngpc, index);
          if (nl == 0 || ng > A.threshold) continue;
          const double sv_freed = freed;
          const int sv_order = order, sv_next = next;
          int q2n = 0, q1n = 0, fail = -1, fsvc = 0, rot = nl;
          bool qover = false;
          for (int kk = 0; kk < nl; kk++) {
            const int cat = W.lst[index][kk] >> 3;
            const int s = cat / 5;
            const double tpp = W.cat_tp[cat];
            const bool newkey = __shfl_sync(0xffffffffu, order, s) == 0;
            if (newkey) next++;
            if (lane == s) {
              if (newkey) { order = next; freed = __dadd_rn(0.0, tpp); }
              else freed = __dadd_rn(freed, tpp);
            }
            const double f = __shfl_sync(0xffffffffu, freed, s);
            const double t1 = W.cat_tp[s * 5 + 0], t2 = W.cat_tp[s * 5 + 1];
            long long k2, k1;
            if (!propose_small(t1, t2, f, k2, k1)) { fail = PARVA_DIAG_SMALL_UNAVAILABLE; fsvc = s; rot = kk + 1; break; }
            if (lane == s) {
              for (long long j = 0; j < k2; j++) freed = __dsub_rn(freed, t2);
              for (long long j = 0; j < k1; j++) freed = __dsub_rn(freed, t1);
            }
            if (qover || q2n + k2 > QCAP || q1n + k1 > QCAP) qover = true;
            else {
              for (int j = lane; j < k2; j += 32) W.q2[q2n + j] = (uint8_t)(s * 5 + 1);
              for (int j = lane; j < k1; j += 32) W.q1[q1n + j] = (uint8_t)(s * 5 + 0);
              q2n += (int)k2; q1n += (int)k1;
            }
          }
          __syncwarp();
          if (fail < 0) {
            if (qover) fail = PARVA_DIAG_NEED_NEW_GPU;
            else {
              int nu = 0;
              for (int j = 0; j < q2n + q1n; j++) {
                const int cat = j < q2n ? W.q2[j] : W.q1[j - q2n];
                const int c = cat % 5;
                const int st = (lane < ngpus && lane != index) ? find_start(mask, c) : -1;
                const unsigned b = __ballot_sync(0xffffffffu, st >= 0);
                if (!b) { fail = PARVA_DIAG_NEED_NEW_GPU; break; }
                const int g = __ffs(b) - 1;
                if (lane == g) {
                  mask |= footprint(c, st);
                  ngpc += size_of_class(c);
                  W.lst[g][len++] = (uint16_t)(cat << 3 | st);
                }
                if (lane == 0) W.undo[nu] = (uint8_t)g;
                nu++;
              }
              __syncwarp();
              if (fail >= 0) {  // all-or-nothing undo (allocator.py:272-277)
                for (int j = nu - 1; j >= 0; j--) {
                  const int g = W.undo[j];
                  if (lane == g) {
                    const int e = W.lst[g][--len];
                    mask &= ~footprint((e >> 3) % 5, e & 7);
                    ngpc -= size_of_class((e >> 3) % 5);
                  }
                }
              }
            }
          }
          if (fail >= 0) {
            // restore drained placements (allocator.py:415-417): the ones not yet
            // removed keep their order, the removed ones are re-appended
            if (lane == index && rot != nl) {
              uint16_t e[8];
#pragma unroll
              for (int j = 0; j < 8; j++) e[j] = W.lst[index][j];
#pragma unroll
              for (int j = 0; j < 8; j++) {
                if (j < nl) {
                  int src = j + rot;
                  if (src >= nl) src -= nl;
                  uint16_t v = e[0];
#pragma unroll
                  for (int u = 1; u < 8; u++) if (u == src) v = e[u];
                  W.lst[index][j] = v;
                }
              }
            }
            freed = sv_freed; order = sv_order; next = sv_next;
            if (lane == 0)
              W.diag[nd] = (uint16_t)(index << 7 | fail << 5 | (fail == PARVA_DIAG_SMALL_UNAVAILABLE ? fsvc : 0));
            nd++;
          } else if (lane == index) {
            len = 0; mask = 0; ngpc = 0;
          }
          __syncwarp();
        }
        // compaction + regression check (allocator.py:423-435)
        const int n_after = __popc(__ballot_sync(0xffffffffu, lane < ngpus && len > 0));
        const int total_after = warp_sum_i(lane < ngpus ? ngpc : 0);
        const double ua_before = unallocated(total_before, n_before);
        const double ua_after = unallocated(total_after, n_after);
        if (n_after > n_before || ua_after > __dadd_rn(ua_before, 1e-12)) {
          fallback = true;
          *reinterpret_cast<uint4*>(W.lst[lane]) = *reinterpret_cast<const uint4*>(W.bak[lane]);
          len = bak_len; ngpc = bak_ngpc; mask = bak_mask;
          freed = 0.0; order = 0; nd = 0;
        }
      }
      __syncwarp();

      // ------------------------------------------------------- emit record
      const bool good = lane < ngpus && len > 0;
      const int mine = good ? len : 0;
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int n_place = __shfl_sync(0xffffffffu, incl, 31);
      const int n_final = __popc(__ballot_sync(0xffffffffu, good));
      const int n_led = __popc(__ballot_sync(0xffffffffu, lane < n && order > 0));
      const int led_off = (2 * (n_place + nd) + 7) & ~7;
      const int need = led_off + 10 * n_led;
      if (need > PARVA_PLAN_PAYLOAD) {
        status = PARVA_CAPACITY;
      } else {
        spill = A.plan_bytes == 64 && need > 64 - 8;
        uint16_t* pay16 = reinterpret_cast<uint16_t*>(W.rec.payload);
        for (int j = 0; j < mine; j++) pay16[incl - mine + j] = (uint16_t)(lane << 11 | W.lst[lane][j]);
        if (lane < nd) pay16[n_place + lane] = W.diag[lane];
        if (lane < n && order > 0) {
          reinterpret_cast<double*>(W.rec.payload + led_off)[order - 1] = freed;
          reinterpret_cast<uint16_t*>(W.rec.payload + led_off + 8 * n_led)[order - 1] = (uint16_t)(lane | order << 8);
        }
        if (lane == 0) {
          W.rec.n_gpus = (uint8_t)n_final;
          W.rec.n_gpus_unopt = (uint8_t)n_before;
          W.rec.n_place = (uint8_t)n_place;
          W.rec.n_diag = (uint8_t)nd;
          W.rec.n_ledger = (uint8_t)n_led;
          W.rec.flags = fallback ? PARVA_FLAG_FALLBACK : 0;
        }
      }
      // reset this lane's GPU list slots for the next scenario
      *reinterpret_cast<uint4*>(W.lst[lane]) = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    if (status != PARVA_OK) {
      reinterpret_cast<uint32_t*>(&W.rec)[lane] = 0u;
      __syncwarp();
      if (lane == 0) {
        W.rec.status = (uint8_t)status;
        W.rec.err_service = (uint8_t)(status == PARVA_CAPACITY ? 0 : err_svc);
      }
    }
    __syncwarp();
    uint8_t* dst = reinterpret_cast<uint8_t*>(A.plan) + (size_t)k * A.plan_bytes;
    if (status == PARVA_OK && spill) {
      // 64-byte records: the full record goes to the spill list
      int slot = 0;
      if (lane == 0) slot = atomicAdd(A.spill_count, 1);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (slot < A.spill_cap) {
        uint8_t* e = A.spill + (size_t)slot * kSpillEntry;
        if (lane == 0) *reinterpret_cast<int4*>(e) = make_int4(k, 0, 0, 0);
        if (lane < 8) reinterpret_cast<uint4*>(e + 16)[lane] = reinterpret_cast<const uint4*>(&W.rec)[lane];
        if (lane < 4) reinterpret_cast<uint4*>(dst)[lane] = lane == 0 ? make_uint4(PARVA_SPILLED, 0, 0, 0) : make_uint4(0, 0, 0, 0);
      } else if (lane < 4) {
        reinterpret_cast<uint4*>(dst)[lane] = lane == 0 ? make_uint4(PARVA_CAPACITY, 0, 0, 0) : make_uint4(0, 0, 0, 0);
      }
    } else if (lane < A.plan_bytes / 16) {
      reinterpret_cast<uint4*>(dst)[lane] = reinterpret_cast<const uint4*>(&W.rec)[lane];
    }
    __syncwarp();
  }
}


size_t index_smem_bytes(int n_tables, int64_t n_points, bool smem_index, bool lat_best) {
  size_t b = (size_t(n_tables) * 5 * 8 + 15) & ~size_t(15);
  if (smem_index) {
    b += size_t((n_points * 8 + 15) & ~int64_t(15));
    if (lat_best) b += size_t((n_points * 8 + 15) & ~int64_t(15)) + size_t((n_points * 2 + 15) & ~int64_t(15));
  }
  return (b + 15) & ~size_t(15);
}

struct LaunchCfg {
  int grid_a, grid_b;
  size_t smem_a, smem_b;
};

static bool plan_launch_config(const PlanArgs& A, LaunchCfg* L) {
  const size_t smem_b = sizeof(WarpScratch) * PB_WARPS + index_smem_bytes(A.n_tables, A.n_points, A.smem_index, false);
  const size_t smem_a = index_smem_bytes(A.n_tables, A.n_points, A.smem_index, true);
  // per-device caches: smem attribute set, occupancy for the smem size used
  struct DevCfg { size_t conf_a, conf_b, occ_a, occ_b; int n_sm, per_a, per_b; };
  static DevCfg s_cfg[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  DevCfg& D = s_cfg[dev & (kMaxDevices - 1)];
  if (smem_b > D.conf_b) {
    cudaFuncSetAttribute(plan_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
    D.conf_b = smem_b;
  }
  if (smem_a > D.conf_a) {
    cudaFuncSetAttribute(configure_services_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
    D.conf_a = smem_a;
  }
  if (!D.n_sm) cudaDeviceGetAttribute(&D.n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (smem_b != D.occ_b) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.per_b, plan_batch_kernel, PB_THREADS, smem_b);
    D.occ_b = smem_b;
  }
  if (smem_a != D.occ_a) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.per_a, configure_services_kernel, CF_THREADS, smem_a);
    D.occ_a = smem_a;
  }
  const int n_sm = D.n_sm, per_a = D.per_a, per_b = D.per_b;
  if (per_b < 1 || per_a < 1) return false;
  int gb = (A.n_scen + PB_WARPS - 1) / PB_WARPS;
  if (gb > n_sm * per_b) gb = n_sm * per_b;
  int ga = (int)((A.n_svc + CF_THREADS - 1) / CF_THREADS);
  if (ga > n_sm * per_a) ga = n_sm * per_a;
  L->grid_a = ga < 1 ? 1 : ga;
  L->grid_b = gb < 1 ? 1 : gb;
  L->smem_a = smem_a;
  L->smem_b = smem_b;
  return true;
}

int launch_plan_batch(const PlanArgs& A, cudaStream_t stream) {
  if (A.n_scen <= 0) return PARVA_OK;
  LaunchCfg L;
  if (!plan_launch_config(A, &L)) return PARVA_LAUNCH_ERROR;
  const bool two = !A.cfg_given && A.n_svc > 0;
  if (two) configure_services_kernel<<<L.grid_a, CF_THREADS, L.smem_a, stream>>>(A);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid_b);
  cfg.blockDim = dim3(PB_THREADS);
  cfg.dynamicSmemBytes = L.smem_b;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = two ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, plan_batch_kernel, A) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int add_plan_batch_node(cudaGraph_t g, const PlanArgs& A, const cudaGraphNode_t* deps, size_t ndeps,
                        cudaGraphNode_t* node) {
  LaunchCfg L;
  if (!plan_launch_config(A, &L)) return PARVA_LAUNCH_ERROR;
  PlanArgs copy = A;
  void* args[] = {&copy};
  cudaKernelNodeParams p = {};
  cudaGraphNode_t na;
  const cudaGraphNode_t* d = deps;
  size_t nd = ndeps;
  if (!A.cfg_given && A.n_svc > 0) {
    p.func = (void*)configure_services_kernel;
    p.gridDim = dim3(L.grid_a);
    p.blockDim = dim3(CF_THREADS);
    p.sharedMemBytes = (unsigned)L.smem_a;
    p.kernelParams = args;
    if (cudaGraphAddKernelNode(&na, g, deps, ndeps, &p) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    d = &na;
    nd = 1;
  }
  p.func = (void*)plan_batch_kernel;
  p.gridDim = dim3(L.grid_b);
  p.blockDim = dim3(PB_THREADS);
  p.sharedMemBytes = (unsigned)L.smem_b;
  p.kernelParams = args;
  if (d != deps) {
    // K2a -> K2b as a programmatic edge (PDL inside the graph)
    if (cudaGraphAddKernelNode(node, g, nullptr, 0, &p) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    cudaGraphEdgeData ed = {};
    ed.from_port = cudaGraphKernelNodePortProgrammatic;
    ed.type = cudaGraphDependencyTypeProgrammatic;
    return cudaGraphAddDependencies_v2(g, &na, node, &ed, 1) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
  }
  return cudaGraphAddKernelNode(node, g, d, nd, &p) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva
