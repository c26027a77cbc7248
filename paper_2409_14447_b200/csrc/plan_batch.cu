// plan_batch.cu — K2: fused per-scenario planner (sm_100a).
//
// Replaces plan_services' timed region (pipeline.py:95-103) for a batch of
// independent scenarios: configure_service x N (configurator.py:189-191),
// relocate_segments (allocator.py:292-316), optimize_allocation
// (allocator.py:362-443).  A lane group (half warp; a full warp for the
// rare scenario wider than 16 services / GPUs) plans one scenario:
//   * configure: thread = service (tile kernel) or lane = service (streamed
//     kernel); per size class a binary search over the latency-sorted
//     prefix-argmax index, staged in shared memory, or read through L1 by
//     back-to-back overlapped launches (exact: the points with lat < bound
//     are a prefix of the sorted order and the argmax under a total order is
//     prefix-decomposable);
//   * relocate / optimize: lane = GPU; a GPU is a 7-bit slot mask; first-fit
//     is one ballot over find_start(mask) (cursorless first-fit is
//     equivalent to the reference's cursors); the
//     freed_rate ledger lives in lane = service registers, snapshot/restore
//     is a register copy.
// Three kernels: plan_thread_kernel (plan_thread.cuh; device-resident
// batches, the default: one thread per scenario; the <true> instantiation
// also copies each chunk's records into every rank's gathered block over
// peer memory), plan_batch_kernel (the tile kernel: lane groups per
// scenario; used when K1's config records are given, i.e. for tables too
// large for the index) and plan_warp_kernel (the zero-copy entry: loader
// CTAs stream the input over PCIe with TMA while the other warps plan).  Scenarios beyond the 128-byte record's limits
// report PARVA_CAPACITY and are re-planned by the general kernel
// (plan_general.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "parva_async.cuh"
#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

// 12 warps x 3 CTAs per SM (56 registers, 36 warps resident) measured best
// for K2 among 8-16 warps x 2-4 CTAs (tools/k2_variants.py)
#ifndef PARVA_PB_WARPS
#define PARVA_PB_WARPS 12
#endif
#ifndef PARVA_PB_MINB
#define PARVA_PB_MINB 2
#endif
constexpr int PB_WARPS = PARVA_PB_WARPS;
constexpr int PB_THREADS = PB_WARPS * 32;
// the tile kernel's CTA shape (K2, device-resident batches)
#ifndef PARVA_TK_WARPS
#define PARVA_TK_WARPS PARVA_PB_WARPS
#endif
constexpr int TK_WARPS = PARVA_TK_WARPS;
constexpr int TK_THREADS = TK_WARPS * 32;
// Per-group scratch of the warp planner; G lanes = G GPUs at most.  The
// refill queues hold G*7 segments: more than the other G-1 GPUs' 7(G-1)
// slots cannot fit anyway (the drain then needs a new GPU).
template <int G>
struct alignas(16) GScratch {
  uint16_t lst[G][8];                     // per GPU placement list: cat << 3 | slot
  uint16_t bak[G][8];                     // relocation result (regression fallback)
  uint8_t q2[G * 7];
  uint8_t q1[G * 7];
  uint8_t undo[2 * G * 7];
  uint16_t diag[G];                       // optimize diagnostics, in order
  parva_plan_record rec;
};
// a warp's scratch (tile and streamed kernels): two half-warp groups, or (overflow
// pass) one full-warp group over the same bytes
constexpr size_t kWarpArea = 2 * sizeof(GScratch<16>) > sizeof(GScratch<32>) ? 2 * sizeof(GScratch<16>)
                                                                             : sizeof(GScratch<32>);


// A lane group that plans one scenario: the whole warp (G = 32) or one half
// (G = 16; two scenarios per warp).  All collectives are restricted to the
// group's member mask; ballots come back shifted to the group's lanes.
template <int G>
struct Grp {
  unsigned m;
  int sh;
  __device__ __forceinline__ unsigned ballot(bool p) const {
    return G == 32 ? __ballot_sync(m, p) : (__ballot_sync(m, p) >> sh) & 0xFFFFu;
  }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(m, p); }
  __device__ __forceinline__ bool all(bool p) const { return __all_sync(m, p); }
  template <typename T> __device__ __forceinline__ T shfl(T v, int s) const { return __shfl_sync(m, v, s, G); }
  template <typename T> __device__ __forceinline__ T shfl_up(T v, int o) const { return __shfl_up_sync(m, v, o, G); }
  template <typename T> __device__ __forceinline__ T shfl_xor(T v, int o) const { return __shfl_xor_sync(m, v, o, G); }
  __device__ __forceinline__ void sync() const { __syncwarp(m); }
};

template <int G>
__device__ __forceinline__ int warp_sum_i(int v, const Grp<G>& gp) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += gp.shfl_xor(v, o);
  return v;
}
template <int G>
__device__ __forceinline__ long long warp_sum_ll(long long v, const Grp<G>& gp) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += gp.shfl_xor(v, o);
  return v;
}

__device__ __forceinline__ double unallocated(int total, int n) {
  if (n == 0) return 0.0;
  return __dsub_rn(1.0, __ddiv_rn((double)total, (double)(7 * n)));
}

// ------------------------------------------------------------ slot tickets
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
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

// One thread per CTA, before the CTA's first store: every scenario of the
// slot's earlier launches is done (completion counter >= wait) and, for the
// fused all-gather, every rank has released the slot's previous epoch.
// Launches into one slot are therefore serialized however many overlapped
// grids are in flight.  No deadlock: a programmatic dependent launch starts
// only after every CTA of its predecessor has started, so every earlier grid
// is resident or finished.  Returns false after the timeout (error recorded).
__device__ __noinline__ bool ticket_wait(const unsigned long long* count, unsigned long long wait,
                                         const uint32_t* acks, int n_acks, uint32_t ack_prev,
                                         unsigned long long timeout_ns, int32_t* err) {
  // relaxed polls: nothing the earlier launches wrote is read, only
  // overwritten, and no store is issued before the poll has returned.  (An
  // acquire at gpu scope invalidates the SM's L1 -- and with it the index
  // the SM's overlapped CTAs read through L1: +2 us per C2 step.)
  const unsigned long long t0 = global_ns();
  for (unsigned ns = 32;; ns = ns < 1024 ? 2 * ns : ns) {
    unsigned long long c;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(count) : "memory");
    bool ok = c >= wait;
    if (ok && acks && ack_prev)
      for (int m = 0; m < n_acks && ok; m++) {
        uint32_t a;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(a) : "l"(acks + m) : "memory");
        ok = (int32_t)(a - ack_prev) >= 0;
      }
    if (ok) return true;
    if (global_ns() - t0 > timeout_ns) {
      if (err) atomicExch(err, (int32_t)PARVA_LAUNCH_ERROR);
      return false;
    }
    __nanosleep(ns);
  }
}

// configure one service from the index: for each size class, count = number
// of points with lat < bound (binary search over the latency-sorted
// segment), winner = prefix argmax at count-1.  The five searches advance in
// lockstep (branch-free power-of-two steps) so their loads overlap.
template <typename SegT>
__device__ __forceinline__ void configure_indexed(const double* lat_s, const uint16_t* best_s,
                                                  const double* tp, int tp_stride, const SegT* seg_s,
                                                  const int* seg_n, int t, double bound,
                                                  double rate, parva_config_record& r,
                                                  double tpc[5], bool with_coverage = true) {
  int s0[5], n[5], lo[5];
  int nmax = 0;
#pragma unroll
  for (int c = 0; c < 5; c++) {
    s0[c] = (int)seg_s[t * 5 + c];
    n[c] = seg_n[t * 5 + c];
    lo[c] = 0;
    nmax = max(nmax, n[c]);
  }
#ifndef PARVA_QUAD_SEARCH   // (A/B builds: a 4-ary form, 3 rounds of 15 loads -- measured slower: the
                            // kernel is issue-bound, the extra probes cost more than the rounds saved)
  for (int step = nmax ? 1 << (31 - __clz(nmax)) : 0; step > 0; step >>= 1) {
#pragma unroll
    for (int c = 0; c < 5; c++) {
      const int probe = lo[c] + step;
      if (probe <= n[c] && lat_s[s0[c] + probe - 1] < bound) lo[c] = probe;
    }
  }
#else
  // 4-ary: three probes per class and round (15 independent loads in
  // flight), so a segment of <= 63 points takes 3 dependent rounds instead
  // of 6.  The probes' outcomes are monotone (sorted latencies), so the
  // count advances by step x (number of true probes).
  for (int step = nmax ? 1 << (2 * ((31 - __clz(nmax)) >> 1)) : 0; step > 0; step >>= 2) {
#pragma unroll
    for (int c = 0; c < 5; c++) {
      const int p1 = lo[c] + step, p2 = p1 + step, p3 = p2 + step;
      const double* a = lat_s + s0[c] - 1;
      const int t = (p1 <= n[c] && a[p1] < bound) + (p2 <= n[c] && a[p2] < bound) + (p3 <= n[c] && a[p3] < bound);
      lo[c] += step * t;
    }
  }
#endif
#pragma unroll
  for (int c = 0; c < 5; c++) {
    const int b = lo[c] ? (int)best_s[s0[c] + lo[c] - 1] : -1;
    r.best[c] = (int16_t)b;
    tpc[c] = b >= 0 ? tp[(s0[c] + b) * tp_stride] : 0.0;
  }
  match_demand(tpc, rate, r, with_coverage);
  if (r.status == PARVA_INFEASIBLE_SLO) r.opt_sc = -1;
}

// Greedy capacity of a GPU (slot mask m) for size class c: how many
// segments repeated find_start + place accept (mig.py:114-149).  The
// preference-ordered footprints of one class are disjoint, so it is a count.
__device__ __forceinline__ int class_capacity(uint32_t m, int c) {
  switch (c) {
    case 4: return m == 0;
    case 3: return (m & 0x0Fu) == 0;
    case 2: return ((m & 0x70u) == 0) + ((m & 0x0Fu) == 0);
    case 1: return ((m & 0x03u) == 0) + ((m & 0x0Cu) == 0) + ((m & 0x30u) == 0);
    default: return __popc(~m & 0x7Fu);
  }
}

template <int G>
__device__ __forceinline__ int warp_incl_scan(int v, int lane, const Grp<G>& gp) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) {
    const int t = gp.shfl_up(v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// One relocation size class (allocator.py:284-289 queue order: services in
// input order, opt copies then last; c is a compile-time constant).
// First-fit within one class fills GPUs strictly in list order: a placement
// changes only its own GPU, so the first accepting GPU keeps accepting until
// it is full, and a new GPU is appended only when none accepts
// (allocator.py:194-251, 280-281).  GPU g (lane g; lanes >= ngpus are the
// GPUs that would be appended, mask 0) therefore takes queue items
// [C_g - cap_g, min(C_g, R)), C = inclusive prefix of capacities -- the same
// placements, in the same per-GPU list order, as R sequential first-fits.
// The queue is walked service by service (warp-uniform); each lane places
// its share of the service's items.  For the first three classes the
// capacity prefix has a closed form: relocation starts from an empty map,
// so when size 4 is queued every existing GPU holds one size-7 segment, and
// when size 3 is queued the n7 first GPUs are full and the rest hold 4@0.
template <int c, int G>
__device__ __forceinline__ void relocate_class(GScratch<G>& W, int lane, int n, int my_opt, long long my_count,
                                               int my_last, uint32_t& mask, int& ngpc, int& len, int& ngpus,
                                               int& n7, int& status, const Grp<G>& gp) {
  // total segments <= 224 was checked, so per-service counts fit an int
  const int my_reps = lane < n ? (my_opt == c ? (int)my_count : 0) + (my_last == c ? 1 : 0) : 0;
  unsigned pending = gp.ballot(my_reps > 0);
  if (!pending) return;
  int cap, incl;
  if (c == 4) {                      // empty map
    cap = 1; incl = lane + 1;
  } else if (c == 3) {               // GPUs [0, ngpus) full
    cap = lane >= ngpus; incl = max(0, lane + 1 - ngpus);
  } else if (c == 2) {               // [0, n7) full, [n7, ngpus) hold 4@0 (slot 4 free), then empty
    cap = lane < n7 ? 0 : lane < ngpus ? 1 : 2;
    incl = lane < n7 ? 0 : lane < ngpus ? lane + 1 - n7 : ngpus - n7 + 2 * (lane + 1 - ngpus);
  } else {
    cap = class_capacity(mask, c);
    incl = warp_incl_scan(cap, lane, gp);
  }
  const int excl = incl - cap;
  int e = 0;                         // queue position of the current service's first item
  do {
    const int s = __ffs(pending) - 1;
    pending &= pending - 1;
    const int reps = gp.shfl(my_reps, s);
    const int hi = min(incl, e + reps);
    const uint16_t cat3 = (uint16_t)((s * 5 + c) << 3);
    int j = max(excl, e);
    if (c >= 3) {                    // capacity 1: at most one item per GPU
      if (j < hi) {
        mask |= footprint(c, 0);
        ngpc += size_of_class(c);
        W.lst[lane][len++] = cat3;
      }
    } else {
#pragma unroll 1
      for (; j < hi; j++) {
        const int st = find_start(mask, c);
        mask |= footprint(c, st);
        ngpc += size_of_class(c);
        W.lst[lane][len++] = (uint16_t)(cat3 | st);
      }
    }
    e += reps;
  } while (pending);
  if (e > gp.shfl(incl, G - 1)) { status = PARVA_CAPACITY; return; }  // needs GPU index >= G
  ngpus = max(ngpus, 32 - __clz(gp.ballot(excl < e && cap > 0)));
  if (c == 4) n7 = ngpus;
}

// propose_small_segments over a lane group (see propose_small_warp in
// parva_common.cuh: k2 candidates spread over the lanes, exact lexicographic
// min reduction)
template <int G>
__device__ __forceinline__ bool propose_small_grp(double tp1, double tp2, double freed, long long& k2o,
                                                 long long& k1o, int lane, const Grp<G>& gp) {
  k2o = 0; k1o = 0;
  if (freed <= 0.0) return true;
  if (tp1 == 0.0 && tp2 == 0.0) return false;
  long long max_k2 = 0;
  if (tp2 != 0.0) max_k2 = (long long)ceil(__dsub_rn(__ddiv_rn(freed, tp2), 1e-12));
  const double m = (1.0 > freed) ? 1.0 : freed;
  const double thr = __dmul_rn(1e-12, m);
  bool have = false;
  long long bg = 0, bc = 0, bn = 0;
  // (gpcs, count, -k2) packs order-preserving into one u64 when every field
  // fits 21 bits: key = gpcs << 42 | count << 21 | (2^21 - 1 - k2)
  const bool packed = max_k2 < (1ll << 19);
  for (long long base = 0; base <= max_k2; base += G) {
    const long long k2 = base + lane;
    bool ok = k2 <= max_k2;
    long long k1 = 0;
    if (ok) {
      const double covered = tp2 != 0.0 ? __dmul_rn((double)k2, tp2) : 0.0;
      const double sh = __dsub_rn(freed, covered);
      if (sh <= thr) k1 = 0;
      else if (tp1 != 0.0) {
        k1 = (long long)ceil(__dsub_rn(__ddiv_rn(sh, tp1), 1e-12));
        if (k1 < 1) k1 = 1;
      } else ok = false;
    }
    long long g, cn, nk;
    // warp-uniform choice (the reductions are collective)
    if (packed && gp.all(!ok || 2 * k2 + k1 < (1ll << 21))) {
      unsigned long long key = ok ? ((unsigned long long)(2 * k2 + k1) << 42) |
                                        ((unsigned long long)(k2 + k1) << 21) |
                                        (unsigned long long)((1ll << 21) - 1 - k2)
                                  : ~0ull;
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const unsigned long long k = gp.shfl_xor(key, o);
        key = k < key ? k : key;
      }
      if (key == ~0ull) { g = cn = nk = LLONG_MAX; }
      else {
        g = (long long)(key >> 42);
        cn = (long long)((key >> 21) & ((1ull << 21) - 1));
        nk = (long long)(key & ((1ull << 21) - 1)) - ((1ll << 21) - 1);
      }
    } else {
      g = ok ? 2 * k2 + k1 : LLONG_MAX; cn = ok ? k2 + k1 : LLONG_MAX; nk = ok ? -k2 : LLONG_MAX;
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const long long g2 = gp.shfl_xor(g, o);
        const long long c2 = gp.shfl_xor(cn, o);
        const long long n2 = gp.shfl_xor(nk, o);
        if (g2 < g || (g2 == g && (c2 < cn || (c2 == cn && n2 < nk)))) { g = g2; cn = c2; nk = n2; }
      }
    }
    if (g != LLONG_MAX && (!have || g < bg || (g == bg && (cn < bc || (cn == bc && nk < bn))))) {
      have = true; bg = g; bc = cn; bn = nk;
    }
  }
  if (!have) return false;
  k2o = -bn;
  k1o = bc + bn;
  return true;
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

// config record store, words assembled in registers (no local copy)
__device__ __forceinline__ void store_config(const PlanArgs& A, int64_t i, const parva_config_record& r) {
  void* cfg = A.cfg;
#if defined(PARVA_NO_OUT) || defined(PARVA_NO_CFG_OUT)
  if (A.stream_src) return;   // development probe: PCIe reads without the record writes
#endif
  const uint32_t b01 = (uint16_t)r.best[0] | (uint32_t)(uint16_t)r.best[1] << 16;
  const uint32_t b23 = (uint16_t)r.best[2] | (uint32_t)(uint16_t)r.best[3] << 16;
  const uint32_t b4ol = (uint16_t)r.best[4] | (uint32_t)(uint8_t)r.opt_sc << 16 | (uint32_t)(uint8_t)r.last_sc << 24;
  if (A.cfg_format == PARVA_CFG_TINY) {
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) lo |= (uint32_t)(r.best[c] < 0 ? 255 : (uint8_t)r.best[c]) << (8 * c);
    const uint32_t ol = (uint32_t)((r.opt_sc < 0 ? 15 : r.opt_sc) | (r.last_sc < 0 ? 15 : r.last_sc) << 4);
    const uint32_t sf = (uint32_t)(r.status | (r.count > 255 ? 0x80 : 0));
    const uint32_t cn = (uint32_t)(r.count > 255 ? 255 : r.count);
    hi = (uint32_t)(r.best[4] < 0 ? 255 : (uint8_t)r.best[4]) | ol << 8 | sf << 16 | cn << 24;
    reinterpret_cast<uint2*>(cfg)[i] = make_uint2(lo, hi);
  } else if (A.cfg_format == PARVA_CFG_COMPACT) {
    const uint32_t w3 = (uint32_t)r.status | (uint32_t)(r.count > 65535 ? 1 : 0) << 8 |
                        (uint32_t)(r.count > 65535 ? 65535 : r.count) << 16;
    reinterpret_cast<uint4*>(cfg)[i] = make_uint4(b01, b23, b4ol, w3);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<parva_config_record*>(cfg) + i);
    const unsigned long long cbits = (unsigned long long)r.count;
    const unsigned long long vbits = (unsigned long long)__double_as_longlong(r.coverage);
    dst[0] = make_uint4(b01, b23, b4ol, (uint32_t)r.status | (uint32_t)r.flags << 8);
    dst[1] = make_uint4((uint32_t)cbits, (uint32_t)(cbits >> 32), (uint32_t)vbits, (uint32_t)(vbits >> 32));
  }
}

// ------------------------------------------------------------------ K2
// One kernel, tile by tile.  A CTA owns a contiguous block of scenarios and
// walks it in tiles of at most kTileSvc services: all threads configure the
// tile's services (thread per service, configurator.py:189-191 through the
// prefix-argmax index in shared memory), the per-service results stay in
// shared memory, then the CTA's half warps plan the tile's scenarios (taken
// from a shared counter so that uneven scenarios balance inside the CTA).
// 256-service tiles keep three CTAs per SM within shared memory.
#ifndef PARVA_TILE_SVC
#define PARVA_TILE_SVC 256
#endif
constexpr int kTileSvc = PARVA_TILE_SVC;

#ifdef PARVA_PHASE_TIMING
// development probe (tools/k2_probe.py): per-CTA phase timestamps and per-warp
// finish times / scenario counts; not built into the product library
__device__ unsigned long long g_phase[1024][4];
__device__ unsigned long long g_warp_end[1024][PB_WARPS][2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PHASE(i) do { if (threadIdx.x == 0 && blockIdx.x < 1024) g_phase[blockIdx.x][i] = gtimer(); } while (0)
__device__ unsigned long long g_warp_cyc[1024][PB_WARPS][4];
__device__ unsigned long long g_warp_wait[1024][PB_WARPS][4];
#define WCYC_START long long wc_t = clock64();
#define WCYC(i) do { const long long wc_n = clock64(); \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) g_warp_cyc[blockIdx.x][threadIdx.x >> 5][i] += wc_n - wc_t; \
    wc_t = wc_n; } while (0)
#else
#define PHASE(i) do { } while (0)
#define WCYC_START
#define WCYC(i) do { } while (0)
#endif

struct alignas(16) TileSmem {
  double tp[kTileSvc * 5];                // best tp per (tile service, size class); 0 = absent
  uint64_t meta[kTileSvc];                // count | opt << 48 | last << 52 | status << 56 (15 = none)
  int32_t off[TK_THREADS + 1];            // tile scenario offsets (absolute service index)
  int32_t next;                           // next tile scenario to plan (half-warp pass)
  int32_t next_over;                      // next overflow entry (full-warp pass)
  int32_t n_over;
  int32_t go;                             // slot ticket granted (first tile)
  int16_t over[TK_THREADS];               // tile scenarios beyond a half-warp's width
};

__device__ __forceinline__ uint64_t pack_meta(int opt, int last, int status, long long count) {
  const uint64_t c = (uint64_t)(count < 0 ? 0 : count > (1ll << 40) ? (1ll << 40) : count);
  return c | (uint64_t)(opt < 0 ? 15 : opt) << 48 | (uint64_t)(last < 0 ? 15 : last) << 52 |
         (uint64_t)(status & 0xFF) << 56;
}

// configure one service (table t, request rate, internal latency bound) and
// store its config record at index out_i
__device__ __forceinline__ uint64_t svc_configure(const PlanArgs& A, const IndexView& V, int t, double rate,
                                                  double bound, int64_t out_i, double tpc[5]) {
  parva_config_record r = {};
  if (t < 0 || t >= A.n_tables) {
#pragma unroll
    for (int c = 0; c < 5; c++) { r.best[c] = -1; tpc[c] = 0.0; }
    r.opt_sc = -1; r.last_sc = -1; r.status = PARVA_BAD_INPUT;
  } else {
    configure_indexed(V.lat, V.best, V.tp, V.tp_stride, V.seg_s, V.seg_n, t, bound, rate, r, tpc,
                      A.cfg_format == PARVA_CFG_FULL);
  }
  store_config(A, out_i, r);
  return pack_meta(r.opt_sc, r.last_sc, r.status, r.count);
}

// configure (or load the given config record of) absolute service i; returns
// the per-size-class tp (0 = absent) and the packed meta word
__device__ __forceinline__ uint64_t tile_service(const PlanArgs& A, const IndexView& V, int64_t i, double tpc[5]) {
  const int t = A.svc_table16 ? (int)A.svc_table16[i] : A.svc_table[i];
  const bool bad_t = t < 0 || t >= A.n_tables;
  if (!A.cfg_given) return svc_configure(A, V, t, A.svc_rate[i], A.svc_bound[i], i, tpc);
  // preconfigured (K1 sweep records)
  int16_t best[5];
  int opt, last, st;
  long long count;
  if (A.cfg_format == PARVA_CFG_TINY) {
    const parva_config_tiny r = reinterpret_cast<const parva_config_tiny*>(A.cfg)[i];
#pragma unroll
    for (int c = 0; c < 5; c++) best[c] = r.best[c] == 255 ? -1 : (int16_t)r.best[c];
    opt = (r.opt_last & 15) == 15 ? -1 : (r.opt_last & 15);
    last = (r.opt_last >> 4) == 15 ? -1 : (r.opt_last >> 4);
    count = (r.status_flags & 0x80) ? (long long)1 << 40 : r.count;   // saturated: cannot fit
    st = r.status_flags & 0x7F;
  } else if (A.cfg_format == PARVA_CFG_COMPACT) {
    const parva_config_compact r = reinterpret_cast<const parva_config_compact*>(A.cfg)[i];
#pragma unroll
    for (int c = 0; c < 5; c++) best[c] = r.best[c];
    opt = r.opt_sc; last = r.last_sc; count = r.count; st = r.status;
  } else {
    const parva_config_record r = reinterpret_cast<const parva_config_record*>(A.cfg)[i];
#pragma unroll
    for (int c = 0; c < 5; c++) best[c] = r.best[c];
    opt = r.opt_sc; last = r.last_sc; count = r.count; st = r.status;
  }
#pragma unroll
  for (int c = 0; c < 5; c++)
    tpc[c] = (!bad_t && st != PARVA_BAD_INPUT && best[c] >= 0) ? V.tp[(V.seg_s[t * 5 + c] + best[c]) * V.tp_stride]
                                                               : 0.0;
  return pack_meta(opt, last, st, count);
}

// relocate + optimize + emit for scenario k (scenario-local services [0, n),
// their tile results at cat_tp / meta); one warp.
// Returns false (writing nothing) when a half-warp group (G = 16) meets a
// limit of its width -- more than 16 services or GPUs -- so that a full warp
// re-plans the scenario; for G = 32 those limits are the record's (CAPACITY).
template <int G>
__device__ __forceinline__ bool plan_scenario_warp(const PlanArgs& A, GScratch<G>& W, int k, int n,
                                                   const double* cat_tp, const uint64_t* meta, bool in_tile,
                                                   int lane, const Grp<G>& gp) {
  WCYC_START
  for (int w = lane; w < 32; w += G) reinterpret_cast<uint32_t*>(&W.rec)[w] = 0u;

  // ------------------------------------------------ configured services
  int err_status = 0, err_svc = 0;
  int my_opt = -1, my_last = -1;
  long long my_count = 0;
  if (n <= PARVA_PLAN_MAX_SERVICES && in_tile) {
    int st = PARVA_OK;
    if (lane < n) {
      const uint64_t m = meta[lane];
      my_count = (long long)(m & ((1ull << 48) - 1));
      my_opt = (int)(m >> 48 & 15); if (my_opt == 15) my_opt = -1;
      my_last = (int)(m >> 52 & 15); if (my_last == 15) my_last = -1;
      st = (int)(m >> 56);
    }
    const unsigned bad = gp.ballot(lane < n && st != PARVA_OK);
    if (bad) {
      err_svc = __ffs(bad) - 1;
      err_status = gp.shfl(st, err_svc);
    }
  }

  int status = PARVA_OK;
  bool spill = false;
  if (G < 32 && (n > G || !in_tile)) return false;
  if (n > PARVA_PLAN_MAX_SERVICES) status = PARVA_CAPACITY;
  else if (!in_tile) status = PARVA_BAD_INPUT;
  else if (err_status) status = err_status;
  else {
    const long long segs = warp_sum_ll(lane < n ? my_count + (my_last >= 0) : 0, gp);
    if (segs > G * 7) {
      if (G < 32) return false;
      status = PARVA_CAPACITY;
    }
  }

  // per-lane GPU state (lane = GPU index) and ledger state (lane = service)
  uint32_t mask = 0;
  int ngpc = 0, len = 0, ngpus = 0;
  double freed = 0.0;
  int order = 0;
  bool fallback = false;
  int nd = 0, n_before = 0;

  WCYC(0);
  int n7 = 0;
  if (status == PARVA_OK) {
    // --------------------------------------------- relocate_segments
    // queue order (allocator.py:46-51): size classes 7,4,3,2,1
    relocate_class<4>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, n7, status, gp);
    if (status == PARVA_OK) relocate_class<3>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, n7, status, gp);
    if (status == PARVA_OK) relocate_class<2>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, n7, status, gp);
    if (status == PARVA_OK) relocate_class<1>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, n7, status, gp);
    if (status == PARVA_OK) relocate_class<0>(W, lane, n, my_opt, my_count, my_last, mask, ngpc, len, ngpus, n7, status, gp);
  }
  gp.sync();
  WCYC(1);
  if (G < 32 && status == PARVA_CAPACITY) return false;   // would need more than G GPUs

  if (status == PARVA_OK) {
    n_before = ngpus;
    const int total_before = warp_sum_i(lane < ngpus ? ngpc : 0, gp);
    *reinterpret_cast<uint4*>(W.bak[lane]) = *reinterpret_cast<const uint4*>(W.lst[lane]);
    const int bak_len = len, bak_ngpc = ngpc;
    const uint32_t bak_mask = mask;

    if (A.optimize) {
      // ----------------------------------------- optimize_allocation
      int next = 0;
      // GPUs last -> first (allocator.py:382): the next GPU to drain is the
      // highest-index one below the last that is non-empty with <= threshold
      // GPCs (skipped GPUs are not touched, so checking them now is the same)
      for (int index = ngpus; ;) {
        const unsigned cand = gp.ballot(lane < index && len > 0 && ngpc <= A.threshold);
        if (!cand) break;
        index = 31 - __clz(cand);
        const int nl = gp.shfl(len, index);
        const double sv_freed = freed;
        const int sv_order = order, sv_next = next;
        int q2n = 0, q1n = 0, fail = -1, fsvc = 0, rot = nl;
        bool qover = false;
        for (int kk = 0; kk < nl; kk++) {
          const int cat = W.lst[index][kk] >> 3;
          const int s = cat / 5;
          const double tpp = cat_tp[cat];
          const bool newkey = gp.shfl(order, s) == 0;
          if (newkey) next++;
          if (lane == s) {
            if (newkey) { order = next; freed = __dadd_rn(0.0, tpp); }
            else freed = __dadd_rn(freed, tpp);
          }
          const double f = gp.shfl(freed, s);
          const double t1 = cat_tp[s * 5 + 0], t2 = cat_tp[s * 5 + 1];
          long long k2, k1;
          if (!propose_small_grp(t1, t2, f, k2, k1, lane, gp)) { fail = PARVA_DIAG_SMALL_UNAVAILABLE; fsvc = s; rot = kk + 1; break; }
          if (lane == s) {
            for (long long j = 0; j < k2; j++) freed = __dsub_rn(freed, t2);
            for (long long j = 0; j < k1; j++) freed = __dsub_rn(freed, t1);
          }
          if (qover || q2n + k2 > G * 7 || q1n + k1 > G * 7) qover = true;
          else {
            for (int j = lane; j < k2; j += 32) W.q2[q2n + j] = (uint8_t)(s * 5 + 1);
            for (int j = lane; j < k1; j += 32) W.q1[q1n + j] = (uint8_t)(s * 5 + 0);
            q2n += (int)k2; q1n += (int)k1;
          }
        }
        gp.sync();
        if (fail < 0) {
          if (qover) fail = PARVA_DIAG_NEED_NEW_GPU;
          else {
            int nu = 0;
            for (int j = 0; j < q2n + q1n; j++) {
              const int cat = j < q2n ? W.q2[j] : W.q1[j - q2n];
              const int c = cat % 5;
              const int st = (lane < ngpus && lane != index) ? find_start(mask, c) : -1;
              const unsigned b = gp.ballot(st >= 0);
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
            gp.sync();
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
        gp.sync();
      }
      // compaction + regression check (allocator.py:423-435)
      const int n_after = __popc(gp.ballot(lane < ngpus && len > 0));
      const int total_after = warp_sum_i(lane < ngpus ? ngpc : 0, gp);
#ifdef PARVA_FLOAT_REGRESSION   // (A/B builds: the reference's float form)
      const double ua_before = unallocated(total_before, n_before);
      const double ua_after = unallocated(total_after, n_after);
      const bool regressed = n_after > n_before || ua_after > __dadd_rn(ua_before, 1e-12);
#else
      // allocator.py:428-430 in integers: unallocated = 1 - t / (7 n) (0 for
      // n = 0).  With n <= 32 GPUs two different values differ by at least
      // 1 / 224^2 >> 1e-12, and equal rationals round to the same double, so
      // "after > before + 1e-12" is exactly t_after n_before < t_before n_after.
      const bool regressed = n_after > n_before ||
                             (n_after > 0 && n_before > 0 && total_after * n_before < total_before * n_after);
#endif
      if (regressed) {
        fallback = true;
        *reinterpret_cast<uint4*>(W.lst[lane]) = *reinterpret_cast<const uint4*>(W.bak[lane]);
        len = bak_len; ngpc = bak_ngpc; mask = bak_mask;
        freed = 0.0; order = 0; nd = 0;
      }
    }
    gp.sync();
    WCYC(2);

    // ------------------------------------------------------- emit record
    const bool good = lane < ngpus && len > 0;
    const int mine = good ? len : 0;
    int incl = mine;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int v = gp.shfl_up(incl, o);
      if (lane >= o) incl += v;
    }
    const int n_place = gp.shfl(incl, G - 1);
    const int n_final = __popc(gp.ballot(good));
    const int n_led = __popc(gp.ballot(lane < n && order > 0));
    const int led_off = (2 * (n_place + nd) + 7) & ~7;
    const int need = led_off + 10 * n_led;
    if (need > PARVA_PLAN_PAYLOAD) {
      status = PARVA_CAPACITY;
    } else {
      spill = A.plan_bytes == 64 && need > 64 - 8;
      uint16_t* pay16 = reinterpret_cast<uint16_t*>(W.rec.payload);
      {
        uint16_t* dst16 = pay16 + (incl - mine);
#pragma unroll
        for (int j = 0; j < 7; j++)
          if (j < mine) dst16[j] = (uint16_t)(lane << 11 | W.lst[lane][j]);
      }
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
  gp.sync();
  if (status != PARVA_OK) {
    for (int w = lane; w < 32; w += G) reinterpret_cast<uint32_t*>(&W.rec)[w] = 0u;
    gp.sync();
    if (lane == 0) {
      W.rec.status = (uint8_t)status;
      W.rec.err_service = (uint8_t)((status == PARVA_CAPACITY || (status == PARVA_BAD_INPUT && !in_tile)) ? 0 : err_svc);
    }
  }
  gp.sync();
  uint8_t* dst = reinterpret_cast<uint8_t*>(A.plan) + (size_t)k * A.plan_bytes;
#if defined(PARVA_NO_OUT) || defined(PARVA_NO_PLAN_OUT)
  if (A.stream_src) { gp.sync(); return true; }
#endif
  if (status == PARVA_OK && spill && A.spill_direct) {
    // 64-byte records, streamed mode: the full record goes to its scenario's
    // slot of the overflow area
    if (lane < 8) reinterpret_cast<uint4*>(A.spill + (size_t)k * 128)[lane] = reinterpret_cast<const uint4*>(&W.rec)[lane];
    if (lane < 4) reinterpret_cast<uint4*>(dst)[lane] = lane == 0 ? make_uint4(PARVA_SPILLED, 0, 0, 0) : make_uint4(0, 0, 0, 0);
  } else if (status == PARVA_OK && spill) {
    // 64-byte records: the full record goes to the spill list
    int slot = 0;
    if (lane == 0) slot = atomicAdd(A.spill_count, 1);
    slot = gp.shfl(slot, 0);
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
  gp.sync();
  WCYC(3);
  return true;
}

// Where a tile loop reads its scenarios: offsets indexable at [k, k1], the
// per-service inputs, and the record index bases.  Streamed inputs were
// written during this kernel, so they are read through L2 (ld.cg).
struct TileSrc {
  const int32_t* off;
  const uint16_t* t16;            // table ids as u16 (packed formats), else t32
  const int32_t* t32;
  const double* rate;
  const double* bound;
  int scen_base;                  // plan record index = scen_base + k
  int64_t svc_base;               // config record index = svc_base + i
  bool cg;
};

template <typename T>
__device__ __forceinline__ T src_ld(const T* p, bool cg) { return cg ? __ldcg(p) : *p; }

// configure service i of a tile source (or load its given config record)
__device__ __forceinline__ uint64_t src_service(const PlanArgs& A, const IndexView& V, const TileSrc& S, int i,
                                                double tpc[5]) {
  if (A.cfg_given) return tile_service(A, V, S.svc_base + i, tpc);
  const int t = S.t16 ? (int)src_ld(S.t16 + i, S.cg) : src_ld(S.t32 + i, S.cg);
  return svc_configure(A, V, t, src_ld(S.rate + i, S.cg), src_ld(S.bound + i, S.cg), S.svc_base + i, tpc);
}

// Configure-then-plan over scenarios [k, k1) of a source, tile by tile: all
// threads configure a tile's services into shared memory, then the warps
// plan its scenarios (taken from a shared counter, so uneven scenarios
// balance inside the CTA).  All threads of the CTA call it.
// With a slot ticket (A.slot_count), thread 0 waits for it while the first
// tile's offsets load, before the tile barrier (no store precedes it);
// returns false (nothing stored) if the wait timed out.
template <bool kMirror>
__device__ __forceinline__ bool run_tiles(const PlanArgs& A, const IndexView& V, TileSmem& T, uint8_t* area,
                                          const TileSrc& S, int k, const int k1, int tid, int lane) {
#ifdef PARVA_PHASE_TIMING
  int dbg_n = 0;
  bool dbg_first = true;
#endif
  bool first = true;
  while (k < k1) {
    // tile = the longest run of scenarios from k with <= kTileSvc services
    // (at least one scenario; offsets are non-decreasing)
    const int a0 = src_ld(S.off + k, S.cg);
    const int e = k + 1 + tid;
    const int off_e = e <= k1 ? src_ld(S.off + e, S.cg) : 0;
    const bool fits = e <= k1 && (tid == 0 || off_e - a0 <= kTileSvc);
    if (e <= k1) T.off[tid + 1] = off_e;
    if (tid == 0) {
      T.off[0] = a0; T.next = 0; T.next_over = 0; T.n_over = 0;
#if !defined(PARVA_AB_NO_TICKET) && !defined(PARVA_AB_NO_WAIT)   // (A/B builds only: tools/k2_ab.py)
      if (first && A.slot_count)
        T.go = ticket_wait(A.slot_count, A.slot_wait, A.ack_row, A.n_mirror, A.ack_prev, A.ticket_timeout_ns,
                           A.err_word);
#endif
    }
    const int n_tile = __syncthreads_count(fits);
    if (first) {
      first = false;
      if (A.slot_count && !T.go) return false;   // timed out: store nothing
    }
    const int a_end = T.off[n_tile];

    // configure the tile's services
    for (int i = a0 + tid; i < a_end; i += TK_THREADS) {
      double tpc[5];
      const uint64_t m = src_service(A, V, S, i, tpc);
      const int li = i - a0;
      if (li < kTileSvc) {
#pragma unroll
        for (int c = 0; c < 5; c++) T.tp[li * 5 + c] = tpc[c];
        T.meta[li] = m;
      }
    }
    __syncthreads();
#ifdef PARVA_PHASE_TIMING
    if (dbg_first) PHASE(2);
    dbg_first = false;
#endif

    // plan the tile's scenarios, two per warp: each half-warp takes
    // scenarios from the shared counter; one that needs more than 16
    // services or GPUs goes to the overflow list, re-planned by full warps
    {
      const int h = lane >> 4, hl = lane & 15;
      const Grp<16> gh{0xFFFFu << (16 * h), 16 * h};
      GScratch<16>& Wh = reinterpret_cast<GScratch<16>*>(area)[h];
      for (;;) {
        int j = 0;
        if (hl == 0) j = atomicAdd(&T.next, 1);
        j = gh.shfl(j, 0);
        if (j >= n_tile) break;
        const int b = T.off[j] - a0;
        const int n = T.off[j + 1] - T.off[j];
        const bool in_tile = b >= 0 && n >= 0 && b + n <= kTileSvc;
        if (!plan_scenario_warp<16>(A, Wh, S.scen_base + k + j, n, T.tp + (in_tile ? b * 5 : 0),
                                    T.meta + (in_tile ? b : 0), in_tile, hl, gh)) {
          if (hl == 0) T.over[atomicAdd(&T.n_over, 1)] = (int16_t)j;
        }
#ifdef PARVA_PHASE_TIMING
        dbg_n++;
#endif
      }
    }
    __syncthreads();
    for (;;) {
      int x = 0;
      if (lane == 0) x = atomicAdd(&T.next_over, 1);
      x = __shfl_sync(0xffffffffu, x, 0);
      if (x >= T.n_over) break;
      const int j = T.over[x];
      const int b = T.off[j] - a0;
      const int n = T.off[j + 1] - T.off[j];
      const bool in_tile = b >= 0 && n >= 0 && b + n <= kTileSvc;
      plan_scenario_warp<32>(A, *reinterpret_cast<GScratch<32>*>(area), S.scen_base + k + j, n,
                             T.tp + (in_tile ? b * 5 : 0), T.meta + (in_tile ? b : 0),
                             in_tile, lane, Grp<32>{0xffffffffu, 0});
    }
#ifdef PARVA_PHASE_TIMING
    if (lane == 0 && blockIdx.x < 1024) {
      g_warp_end[blockIdx.x][threadIdx.x >> 5][0] = gtimer();
      g_warp_end[blockIdx.x][threadIdx.x >> 5][1] = dbg_n;
    }
#endif
    __syncthreads();
    if (kMirror) {
      // fused all-gather: the tile's records (contiguous plan and config
      // ranges, written by this CTA, visible after the barrier) go to this
      // rank's slot on every rank as coalesced 16-B / 8-B peer stores
      const int cfg_b = A.cfg_format == PARVA_CFG_TINY ? 8 : A.cfg_format == PARVA_CFG_COMPACT ? 16 : 32;
      const size_t p0 = (size_t)(S.scen_base + k) * A.plan_bytes, pn = (size_t)n_tile * A.plan_bytes / 16;
      const size_t c0 = (size_t)(S.svc_base + a0) * cfg_b, cn = (size_t)(a_end - a0) * cfg_b / 8;
      const uint4* ps = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(A.plan) + p0);
      const uint2* cs = reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(A.cfg) + c0);
      for (int m = 0; m < A.n_mirror; m++) {
        uint4* pd = reinterpret_cast<uint4*>(A.mirror_plan[m] + p0);
        uint2* cd = reinterpret_cast<uint2*>(A.mirror_cfg[m] + c0);
        if (pd == ps) continue;   // this rank's own part of the slot is the launch's output
        for (size_t x = tid; x < pn; x += TK_THREADS) pd[x] = ps[x];
        for (size_t x = tid; x < cn; x += TK_THREADS) cd[x] = cs[x];
      }
      if (A.plan_bytes == 64) {
        // 64-byte records: a spilled scenario's full record (overflow area,
        // same index) follows it; one warp per scenario of the tile
        for (int j = tid >> 5; j < n_tile; j += TK_WARPS) {
          const size_t kk = (size_t)(S.scen_base + k + j);
          if (reinterpret_cast<const uint8_t*>(A.plan)[kk * 64] == PARVA_SPILLED && lane < 8) {
            const uint4 v = reinterpret_cast<const uint4*>(A.spill + kk * 128)[lane];
            for (int m = 0; m < A.n_mirror; m++)
              if (A.mirror_spill[m] != A.spill) reinterpret_cast<uint4*>(A.mirror_spill[m] + kk * 128)[lane] = v;
          }
        }
      }
    }
    k += n_tile;
  }
  return true;
}

#ifndef PARVA_TILE_MINB
#define PARVA_TILE_MINB 3
#endif
// kMirror: the fused all-gather instantiation (parva_plan_batch_fused)
template <bool kMirror>
__global__ void __launch_bounds__(TK_THREADS, PARVA_TILE_MINB) plan_batch_kernel(PlanArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  TileSmem& T = *reinterpret_cast<TileSmem*>(smem_raw + kWarpArea * TK_WARPS);
  __shared__ uint64_t bar;
  // an overlapped successor (parva_plan_batch_overlapped / _fused) may take
  // SM slots as this grid's CTAs retire; the slot ticket keeps it from
  // storing into an output slot a launch still in flight writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  PHASE(0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) T.go = 1;
  const IndexView V = load_index(A, smem_raw + kWarpArea * TK_WARPS + sizeof(TileSmem), !A.cfg_given, &bar);
  PHASE(1);
  // this CTA's contiguous block of scenarios
  const int per = (A.n_scen + gridDim.x - 1) / gridDim.x;
  const int k = blockIdx.x * per, k1 = min(A.n_scen, k + per);
  const TileSrc S{A.scen_off, A.svc_table16, A.svc_table, A.svc_rate, A.svc_bound, 0, 0, false};
  if (!run_tiles<kMirror>(A, V, T, smem_raw + kWarpArea * warp, S, k, k1, tid, lane)) return;
  PHASE(3);
#if !defined(PARVA_AB_NO_TICKET) && !defined(PARVA_AB_NO_DONE)
  if (A.slot_count) {
    // completion: the CTA's stores are ordered before thread 0's release
    // reduction (barrier; a release is cumulative over what the barrier
    // made visible to thread 0; peer stores: every thread fences at system
    // scope first).  Fused: the last CTA resets the CTA counter and publishes
    // the epoch into this rank's flag word of the slot on every rank.
    if (kMirror) __threadfence_system();
    __syncthreads();
    if (tid == 0) {
      if (kMirror && atomicAdd(A.done_ctas, 1u) == gridDim.x - 1) {
        atomicExch(A.done_ctas, 0u);
        __threadfence_system();
        for (int m = 0; m < A.n_mirror; m++)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.peer_flag[m]), "r"(A.flag_epoch) : "memory");
      }
      const unsigned long long mine = k1 > k ? (unsigned long long)(k1 - k) : 0ull;
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(A.slot_count), "l"(mine) : "memory");
    }
  }
#endif
}

// K2, warp-autonomous form: every half warp takes scenarios one at a time
// from a device counter (work[0]) and configures its own scenario (lane =
// service, the same prefix-argmax search) before planning it -- no block
// barriers, so loads, configuration and planning of different warps overlap
// freely.  Per-group service staging:
template <int G>
struct alignas(16) GSvc {
  double tp[G * 5];                       // best tp per (service, size class); 0 = absent
  uint64_t meta[G];
};
using WarpSvc = GSvc<32>;
static_assert(2 * sizeof(GSvc<16>) == sizeof(WarpSvc), "two half-warp staging areas fill one warp's");

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streamed mode: one thread per loader CTA is a DMA engine.  It takes input
// slices in ticket order (work[2]) and moves each host -> shared memory with
// a TMA bulk copy (cp.async.bulk reads the pinned, mapped host block over
// PCIe), then shared -> device staging with a bulk store, double-buffered;
// a slice is published (slice_flag[s] = epoch, release) once its store has
// completed.  A handful of loaders keeps ~n_loaders * 16 KB in flight: full
// PCIe bandwidth while the slices still land nearly in order.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Two warps of a loader CTA: warp 0 (one lane) issues the host -> shared
// loads and never fences, so its PCIe reads stay in flight; warp 1 (one lane)
// stores each landed slice to device memory, waits for the store, publishes
// the slice flag and hands the buffer back (full / empty mbarrier pairs;
// separate warps, so the store waits never block the load issue).
__device__ __forceinline__ void stream_loader(const PlanArgs& A, uint8_t* buf, uint64_t* bars, int role) {
  const int64_t n_slices = (A.stream_bytes + kStreamSlice - 1) / kStreamSlice;
  const int nl = A.n_loaders;
  uint64_t* full = bars;
  uint64_t* empty = bars + kLoaderBufs;
  // loader L moves slices L, L + nl, L + 2 nl, ... (all loaders advance at
  // PCIe pace, so the slices land in order)
  if (role == 0) {
    int i = 0;
    for (int64_t s = blockIdx.x; s < n_slices; s += nl, i++) {
      const int b = i % kLoaderBufs;
      if (i >= kLoaderBufs) mbar_wait(&empty[b], (uint32_t)((i / kLoaderBufs - 1) & 1));
      const int64_t o = s * kStreamSlice;
      const uint32_t sz = (uint32_t)min((int64_t)kStreamSlice, A.stream_bytes - o);
      mbar_arrive_expect_tx(&full[b], sz);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(buf + b * kStreamSlice)),
          "l"(A.stream_src + o), "r"(sz), "r"(smem_addr(&full[b]))
          : "memory");
    }
  } else {
    int i = 0;
    for (int64_t s = blockIdx.x; s < n_slices; s += nl, i++) {
      const int b = i % kLoaderBufs;
      mbar_wait(&full[b], (uint32_t)((i / kLoaderBufs) & 1));
      const int64_t o = s * kStreamSlice;
      bulk_s2g(A.stream_dst + o, buf + b * kStreamSlice, (uint32_t)min((int64_t)kStreamSlice, A.stream_bytes - o));
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");      // slice s is in device memory
      asm volatile("fence.proxy.async.global;" ::: "memory");
      st_release_u32(&A.slice_flag[s], A.epoch);
      mbar_arrive(&empty[b]);
    }
#ifdef PARVA_PHASE_TIMING
    if (blockIdx.x < 1024) g_phase[blockIdx.x][2] = gtimer();   // this loader's last slice published
#endif
  }
}

// Streamed mode: wait (this thread) until the input bytes [lo, hi) have landed.
__device__ __forceinline__ void stream_wait_thread(const PlanArgs& A, const void* p_lo, const void* p_hi) {
  const int64_t lo = (const uint8_t*)p_lo - A.stream_dst, hi = (const uint8_t*)p_hi - A.stream_dst;
  if (hi > lo)
    for (int64_t s = lo / kStreamSlice; s <= (hi - 1) / kStreamSlice; s++) {
      // exponential back-off keeps thousands of waiting warps from
      // hammering the flag lines in L2 while the loaders stream
      for (unsigned ns = 64; ld_acquire_u32(&A.slice_flag[s]) != A.epoch; ns = ns < 512 ? 2 * ns : ns)
        __nanosleep(ns);
    }
}

// the same for a lane group (its lane 0 waits)
template <int G>
__device__ __forceinline__ void group_wait(const PlanArgs& A, const void* p_lo, const void* p_hi, int gl,
                                           const Grp<G>& gp) {
  if (gl == 0) stream_wait_thread(A, p_lo, p_hi);
  gp.sync();
}

// A group's current chunk of the streamed input (a header, i.e. the chunk
// table, followed by chunk blocks; scenarios ascend per group).
struct ChunkCursor {
  int c = -1, scen_lo = 0, svc_lo = 0, tmpl = 0;   // tmpl > 0: one table-id sequence for the chunk
  const int32_t* off = nullptr;
  const double* rate = nullptr;
  const double* bound = nullptr;
  const uint16_t* table = nullptr;
};

// Configure and plan streamed scenario j with one lane group.  A half warp
// returns false (no plan written) for a scenario with more than 16 services
// and plan_scenario_warp<16>'s false (more than 16 GPUs / 112 segments): the
// whole warp re-plans it.
template <int G>
__device__ __forceinline__ bool stream_plan_one(const PlanArgs& A, const IndexView& V, GScratch<G>& W,
                                                GSvc<G>& S, ChunkCursor& C, int j, int n_ch, int ch_scen,
                                                int gl, const Grp<G>& gp) {
#ifdef PARVA_PHASE_TIMING
  const long long wt0 = clock64();
#endif
  const int cj = min(j / ch_scen, n_ch - 1);      // chunks hold ch_scen scenarios (the last one fewer)
  if (cj != C.c) {
    C.c = cj;
    const parva_stream_chunk* tab = reinterpret_cast<const parva_stream_chunk*>(A.stream_dst + 16);
    C.scen_lo = __ldcg(&tab[cj].scen_lo);
    C.svc_lo = __ldcg(&tab[cj].svc_lo);
    const int kc = __ldcg(&tab[cj].k), mc = __ldcg(&tab[cj].m);
    const uint8_t* blk = A.stream_dst + __ldcg(&tab[cj].offset);
    C.tmpl = __ldcg(&tab[cj].tmpl);
    // template chunks carry no offsets: scenario k owns [k tmpl, (k+1) tmpl)
    const int64_t rate_off = C.tmpl > 0 ? 0 : ((int64_t)(kc + 1) * 4 + 15) & ~int64_t(15);
    C.off = reinterpret_cast<const int32_t*>(blk);
    C.rate = reinterpret_cast<const double*>(blk + rate_off);
    C.bound = C.rate + mc;
    C.table = reinterpret_cast<const uint16_t*>(C.bound + mc);
    group_wait<G>(A, blk, C.table + (C.tmpl > 0 ? C.tmpl : mc), gl, gp);  // the whole chunk block has landed
  }
  const int jl = j - C.scen_lo;
  const int a0 = C.tmpl > 0 ? jl * C.tmpl : __ldcg(C.off + jl);
  const int n = C.tmpl > 0 ? C.tmpl : __ldcg(C.off + jl + 1) - a0;
  if (G < 32 && n > G) return false;
#ifdef PARVA_PHASE_TIMING
  const long long wt1 = clock64();
#endif
  for (int b = 0; b < n; b += G) {
    if (b + gl < n) {
      const int i = a0 + b + gl;
      double tpc[5];
      const int t = (int)__ldcg(C.table + (C.tmpl > 0 ? b + gl : i));
      const uint64_t m = svc_configure(A, V, t, __ldcg(C.rate + i), __ldcg(C.bound + i), (int64_t)C.svc_lo + i, tpc);
      if (b == 0) {
#pragma unroll
        for (int cc = 0; cc < 5; cc++) S.tp[gl * 5 + cc] = tpc[cc];
        S.meta[gl] = m;
      }
    }
  }
  gp.sync();
#ifdef PARVA_PHASE_TIMING
  const long long wt2 = clock64();
  const bool ok = plan_scenario_warp<G>(A, W, j, n, S.tp, S.meta, n >= 0, gl, gp);
  if (gl == 0 && blockIdx.x < 1024) {
    unsigned long long* w = g_warp_wait[blockIdx.x][threadIdx.x >> 5];
    atomicAdd(&w[0], (unsigned long long)(wt1 - wt0));
    atomicAdd(&w[1], (unsigned long long)(wt2 - wt1));
    atomicAdd(&w[2], (unsigned long long)(clock64() - wt2));
    atomicAdd(&w[3], 1ull);
  }
  return ok;
#else
  return plan_scenario_warp<G>(A, W, j, n, S.tp, S.meta, n >= 0, gl, gp);
#endif
}

__global__ void __launch_bounds__(PB_THREADS, PARVA_PB_MINB) plan_warp_kernel(PlanArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint64_t loader_bars[2 * kLoaderBufs];
  __shared__ int stop_flag[PB_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) stop_flag[warp] = 0;
  // a dependent streamed call (its own scratch and blocks) may start as soon
  // as SM space frees up; nothing here waits for a predecessor
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint8_t* area = smem_raw + kWarpArea * warp;
  WarpSvc* wsvc = reinterpret_cast<WarpSvc*>(smem_raw + kWarpArea * PB_WARPS);
  uint8_t* loader_buf = smem_raw + (kWarpArea + sizeof(WarpSvc)) * PB_WARPS;
  PHASE(0);
  if ((int)blockIdx.x < A.n_loaders && threadIdx.x == 0) {
    for (int b = 0; b < 2 * kLoaderBufs; b++) mbar_init(&loader_bars[b], 1);
    fence_mbar_init();
  }
  // (load_index's block barriers also publish the loader mbarrier inits)
  const IndexView V = load_index(A, loader_buf + kLoaderBufs * kStreamSlice, true, &bar);
  // loader roles (warps 0 and 1 of the first n_loaders CTAs), then they plan
  // too; the CTAs' other warps start planning right away
  if ((int)blockIdx.x < A.n_loaders && warp < 2) {
    if (lane == 0) stream_loader(A, loader_buf, loader_bars, warp);
    __syncwarp();
  }
  PHASE(1);
  const Grp<32> gw{0xffffffffu, 0};
  group_wait<32>(A, A.stream_dst, A.stream_dst + 16, lane, gw);
  const int n_ch = __ldcg(reinterpret_cast<const int32_t*>(A.stream_dst));
  const int ch_scen = max(1, __ldcg(reinterpret_cast<const int32_t*>(A.stream_dst) + 1));
  group_wait<32>(A, A.stream_dst, A.stream_dst + parva_stream_header_bytes(n_ch), lane, gw);

  // Each half warp takes scenarios from the ticket counter.  A half that
  // meets a scenario it cannot plan (more than 16 services / GPUs) raises
  // the warp's stop flag; once its sibling has finished its current
  // scenario the whole warp plans the pending one(s), then both halves go on.
  {
    const int h = lane >> 4, hl = lane & 15;
    const Grp<16> gh{0xFFFFu << (16 * h), 16 * h};
    GScratch<16>& Wh = reinterpret_cast<GScratch<16>*>(area)[h];
    GSvc<16>& Sh = reinterpret_cast<GSvc<16>*>(&wsvc[warp])[h];
    int* stop = &stop_flag[warp];       // cross-half signal: shared-memory atomics (no plain racing accesses)
    ChunkCursor C, Cw;
    bool out = false;                                  // this half saw the tickets run out
    for (;;) {
      int pend = -1;
      while (!out && !atomicAdd(stop, 0)) {
        int j = 0;
        if (hl == 0) j = (int)atomicAdd(&A.work[0], 1u);
        j = gh.shfl(j, 0);
        if (j >= A.n_scen) { out = true; break; }
        if (!stream_plan_one<16>(A, V, Wh, Sh, C, j, n_ch, ch_scen, hl, gh)) {
          pend = j;
          if (hl == 0) atomicExch(stop, 1);
        }
      }
      __syncwarp();
      const int p0 = __shfl_sync(0xffffffffu, pend, 0), p1 = __shfl_sync(0xffffffffu, pend, 16);
      if (p0 >= 0)
        stream_plan_one<32>(A, V, *reinterpret_cast<GScratch<32>*>(area), wsvc[warp], Cw, p0, n_ch, ch_scen, lane, gw);
      if (p1 >= 0)
        stream_plan_one<32>(A, V, *reinterpret_cast<GScratch<32>*>(area), wsvc[warp], Cw, p1, n_ch, ch_scen, lane, gw);
      if (__all_sync(0xffffffffu, out)) break;
      if (lane == 0) atomicExch(stop, 0);
      __syncwarp();
    }
  }
#ifdef PARVA_PHASE_TIMING
  if (lane == 0 && blockIdx.x < 1024) g_warp_end[blockIdx.x][warp][0] = gtimer();
#endif
  // every lane's record stores are ordered before the warp counts itself
  // done (system scope when the host polls done_word instead of the stream)
  if (A.done_word) __threadfence_system();
  else __threadfence();
  __syncwarp();
  if (lane == 0) {
    // last warp of the grid resets the counters for the next launch and
    // publishes completion
    if (atomicAdd(&A.work[1], 1u) == gridDim.x * PB_WARPS - 1) {
      atomicExch(&A.work[0], 0u);
      atomicExch(&A.work[2], 0u);
      atomicExch(&A.work[1], 0u);
      if (A.done_word) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.done_word), "r"(A.epoch) : "memory");
      }
    }
  }
}

#include "plan_thread.cuh"

size_t index_smem_bytes(int n_tables, int64_t n_points, bool smem_index, bool lat_best) {
  size_t b = (size_t(n_tables) * 5 * 8 + 15) & ~size_t(15);
  if (smem_index) {
    b += size_t((n_points * 8 + 15) & ~int64_t(15));
    if (lat_best) b += size_t((n_points * 8 + 15) & ~int64_t(15)) + size_t((n_points * 2 + 15) & ~int64_t(15));
  }
  return (b + 15) & ~size_t(15);
}

struct LaunchCfg {
  int grid;
  size_t smem;
};

// device-resident batches: the thread-per-scenario kernel (PARVA_K2_THREAD,
// default) or the tile kernel (configure a tile with every thread, then
// plan with lane groups); K1's config records given: the tile kernel;
// streamed batches: the warp-autonomous kernel
#ifndef PARVA_K2_THREAD
#define PARVA_K2_THREAD 1
#endif
static bool warp_mode(const PlanArgs& A) { return A.stream_src != nullptr; }
static bool thread_mode(const PlanArgs& A) { return PARVA_K2_THREAD && !warp_mode(A) && !A.cfg_given; }

struct KernelSel {
  const void* fn;
  int kind, threads, per_cta;   // per_cta: scenarios one CTA takes per pass (grid sizing)
};

static KernelSel plan_kernel(const PlanArgs& A) {
  if (warp_mode(A)) return {(const void*)plan_warp_kernel, 1, PB_THREADS, PB_WARPS};
  const bool mir = A.n_mirror > 0;
  if (thread_mode(A))
    return {mir ? (const void*)plan_thread_kernel<true> : (const void*)plan_thread_kernel<false>, mir ? 4 : 3,
            TH_THREADS, 32 * TH_WARPS};
  return {mir ? (const void*)plan_batch_kernel<true> : (const void*)plan_batch_kernel<false>, mir ? 2 : 0,
          TK_THREADS, TK_WARPS};
}

static bool plan_launch_config(const PlanArgs& A, LaunchCfg* L) {
  const bool wm = warp_mode(A);
  const KernelSel K = plan_kernel(A);
  const size_t smem = K.kind >= 3 ? sizeof(ThWarp) * TH_WARPS
                                  : (wm ? (kWarpArea + sizeof(WarpSvc)) * PB_WARPS + size_t(kLoaderBufs) * kStreamSlice
                                        : kWarpArea * TK_WARPS + sizeof(TileSmem)) +
                                        index_smem_bytes(A.n_tables, A.n_points, A.smem_index, !A.cfg_given);
  // per-device caches: smem attribute set, occupancy for the smem size used
  struct DevCfg { size_t conf, occ; int n_sm, per; };
  static DevCfg s_cfg[kMaxDevices][5];
  int dev = 0;
  cudaGetDevice(&dev);
  DevCfg& D = s_cfg[dev & (kMaxDevices - 1)][K.kind];
  if (smem > D.conf) {
    if (cudaFuncSetAttribute(K.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return false;
    D.conf = smem;
  }
  if (!D.n_sm) cudaDeviceGetAttribute(&D.n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (smem != D.occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.per, K.fn, K.threads, smem);
    D.occ = smem;
  }
  if (D.per < 1) return false;
  int per = D.per;
  if (wm) {
    // streamed calls: one CTA per SM (PARVA_STREAM_PER_SM; 0 = all that
    // fit), so a dependent call's CTAs find SM space while this one is still
    // planning (PCIe, not the planners, bounds a streamed call); every loader
    // CTA must exist
    static int s_env = -1;
    if (s_env < 0) {
      const char* e = std::getenv("PARVA_STREAM_PER_SM");
      s_env = e ? std::max(0, std::atoi(e)) : 1;
    }
    if (s_env > 0) per = std::min(per, s_env);
  }
  int g = (A.n_scen + K.per_cta - 1) / K.per_cta;
  if (wm) g = std::max(g, A.n_loaders);
  if (g > D.n_sm * per) g = D.n_sm * per;
  L->grid = g < 1 ? 1 : g;
  L->smem = smem;
  return true;
}

int plan_batch_grid(const PlanArgs& A) {
  LaunchCfg L;
  return plan_launch_config(A, &L) ? L.grid : 0;
}

int launch_plan_batch(const PlanArgs& A, cudaStream_t stream) {
  // the tiny record stores point positions in a byte (255 = absent)
  if (A.cfg_format == PARVA_CFG_TINY && !A.cfg_given && (A.max_seg_points < 0 || A.max_seg_points > 254))
    return PARVA_BAD_INPUT;
  if (A.n_scen <= 0) return PARVA_OK;
  if (A.stream_src && !A.work) return PARVA_BAD_INPUT;
  LaunchCfg L;
  if (!plan_launch_config(A, &L)) return PARVA_LAUNCH_ERROR;
  if (warp_mode(A)) {
    PlanArgs B = A;
    B.n_loaders = std::min(A.n_loaders, L.grid);   // loaders are the first CTAs
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(PB_THREADS);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = A.pdl ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, plan_warp_kernel, B) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  } else {
    const KernelSel K = plan_kernel(A);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(K.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = A.pdl ? 1 : 0;
    void* args[] = {const_cast<PlanArgs*>(&A)};
    if (cudaLaunchKernelExC(&cfg, K.fn, args) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  }
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int add_plan_batch_node(cudaGraph_t g, const PlanArgs& A, const cudaGraphNode_t* deps, size_t ndeps,
                        cudaGraphNode_t* node) {
  LaunchCfg L;
  if (!plan_launch_config(A, &L)) return PARVA_LAUNCH_ERROR;
  PlanArgs copy = A;
  void* args[] = {&copy};
  cudaKernelNodeParams p = {};
  const KernelSel K = plan_kernel(A);
  p.func = const_cast<void*>(K.fn);
  p.gridDim = dim3(L.grid);
  p.blockDim = dim3(K.threads);
  p.sharedMemBytes = (unsigned)L.smem;
  p.kernelParams = args;
  return cudaGraphAddKernelNode(node, g, deps, ndeps, &p) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva

#ifdef PARVA_PHASE_TIMING
extern "C" int parva_dbg_phase(unsigned long long* phase, unsigned long long* warp_end, unsigned long long* cyc) {
  cudaMemcpyFromSymbol(phase, parva::g_phase, sizeof(parva::g_phase));
  cudaMemcpyFromSymbol(cyc, std::getenv("PARVA_DBG_WAIT") ? parva::g_warp_wait : parva::g_warp_cyc,
                       sizeof(parva::g_warp_cyc));
  return cudaMemcpyFromSymbol(warp_end, parva::g_warp_end, sizeof(parva::g_warp_end)) == cudaSuccess ? 0 : 1;
}
#endif
