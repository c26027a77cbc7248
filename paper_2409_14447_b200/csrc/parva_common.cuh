// parva_common.cuh — device building blocks shared by the sm_100a kernels.
//
// Bit-exactness rules: every double operation that the
// reference performs in CPython is done here with an explicitly rounded
// intrinsic (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn), and the whole
// library is compiled with --fmad=false, so no FMA contraction can change a
// residual (configurator.py:156, allocator.py:339-340).
#pragma once

#include <stdint.h>
#include <climits>
#include "../../include/parva_b200.h"

namespace parva {

__host__ __device__ constexpr int size_of_class(int c) { return c == 4 ? 7 : c + 1; }

// ---------------------------------------------------------------- geometry
// A GPU is a 7-bit mask of occupied-or-blocked slots.  find_start replaces
// GpuState.find_start (mig.py:114-122) over _START_OPTIONS (mig.py:41-54);
// the num_gpcs early exit (:116-117) is implied by the footprint test.
__device__ __forceinline__ int find_start(uint32_t m, int c) {
  switch (c) {
    case 4: return m == 0 ? 0 : -1;                       // size 7 @0
    case 3: return (m & 0x0Fu) == 0 ? 0 : -1;             // size 4 @0
    case 2:                                              // size 3 @4, then @0 (blocks 3)
      return (m & 0x70u) == 0 ? 4 : ((m & 0x0Fu) == 0 ? 0 : -1);
    case 1:                                              // size 2 @0, @2, @4
      return (m & 0x03u) == 0 ? 0 : (m & 0x0Cu) == 0 ? 2 : (m & 0x30u) == 0 ? 4 : -1;
    default: {                                           // size 1: lowest free slot
      uint32_t f = ~m & 0x7Fu;
      return f ? __ffs(f) - 1 : -1;
    }
  }
}

// occupied + blocked cells of a placement (size class c at start slot st)
__device__ __forceinline__ uint32_t footprint(int c, int st) {
  switch (c) {
    case 4: return 0x7Fu;
    case 3: return 0x0Fu;
    case 2: return st == 4 ? 0x70u : 0x0Fu;
    case 1: return 0x3u << st;
    default: return 0x1u << st;
  }
}

// ------------------------------------------------------------ comparisons
// _better_triplet (configurator.py:116-124) within one size class: the
// point's position in its key-ordered segment stands for (batch, procs).
struct Cand {
  double tp, lat;
  int idx;  // -1 = none
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.idx < 0) return false;
  if (b.idx < 0) return true;
  if (a.tp != b.tp) return a.tp > b.tp;
  if (a.lat != b.lat) return a.lat < b.lat;
  return a.idx < b.idx;
}

__device__ __forceinline__ Cand warp_argmax(Cand c, unsigned mask = 0xffffffffu) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand d;
    d.tp = __shfl_xor_sync(mask, c.tp, o);
    d.lat = __shfl_xor_sync(mask, c.lat, o);
    d.idx = __shfl_xor_sync(mask, c.idx, o);
    if (better(d, c)) c = d;
  }
  return c;
}

// ------------------------------------------------------ configurator math
// Service.coverage (configurator.py:60-62): CPython 3.12 sum() with int
// start 0 -> first item, then Neumaier compensation (bltinmodule.c).
__device__ __forceinline__ double neumaier_step(double f, double v, double& c) {
  double t = __dadd_rn(f, v);
  if (fabs(f) >= fabs(v)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), v));
  else c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), f));
  return t;
}

__device__ inline double coverage_sum(double topt, long long count, bool has_last, double tlast) {
  if (count == 0 && !has_last) return 0.0;
  double f, c = 0.0;
  long long i0;
  if (count > 0) { f = topt; i0 = 1; } else { f = tlast; i0 = 0; has_last = false; }
  for (long long i = i0; i < count; i++) f = neumaier_step(f, topt, c);
  if (has_last) f = neumaier_step(f, tlast, c);
  if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
  return f;
}

constexpr double kCountLimit = 1099511627776.0;  // 2^40 segments per service

// select_optimal_segment + match_demand (configurator.py:127-186) given the
// per-size-class best throughputs (tp[c] > 0 iff size class c present).
// Fills opt_sc, last_sc, count, coverage, status of a config record.  Only
// constant indices into tp[] (after unrolling), so it stays in registers.
// with_coverage = false skips Service.coverage (for the record formats that
// do not carry it: compact and tiny).
__device__ inline void match_demand(const double tp[5], double rate, parva_config_record& r,
                                    bool with_coverage = true) {
  int o = -1;
  double topt = 0.0;
#pragma unroll
  for (int c = 0; c < 5; c++) {
    if (!(tp[c] > 0.0)) continue;
    if (o < 0) { o = c; topt = tp[c]; continue; }
    // ascending size order: t.size > best.size always, so lhs >= rhs wins
    const double lhs = __dmul_rn(tp[c], (double)size_of_class(o));
    const double rhs = __dmul_rn(topt, (double)size_of_class(c));
    if (lhs > rhs || lhs == rhs) { o = c; topt = tp[c]; }
  }
  r.opt_sc = (int8_t)o;
  r.last_sc = -1;
  r.count = 0;
  r.coverage = 0.0;
  if (o < 0) { r.status = PARVA_INFEASIBLE_SLO; r.opt_sc = -1; return; }
  long long count = 0;
  if (rate > 0.0) {
    const double q = floor(__ddiv_rn(rate, topt));
    if (!(q <= kCountLimit)) { r.status = PARVA_COUNT_OVERFLOW; return; }
    count = (long long)q;
  }
  double remaining = __dsub_rn(rate, __dmul_rn((double)count, topt));
  const double m = (1.0 > rate) ? 1.0 : rate;
  if (remaining <= __dmul_rn(1e-9, m)) remaining = 0.0;
  int last = -1;
  double tlast = 0.0;
  if (remaining > 0.0) {
#pragma unroll
    for (int c = 0; c < 5; c++)
      if (last < 0 && tp[c] > 0.0 && tp[c] >= remaining) { last = c; tlast = tp[c]; }
    if (last < 0) {  // configurator.py:166-176 (unreachable in practice)
      int fb = -1;
      double tfb = 0.0;
#pragma unroll
      for (int c = 0; c < 5; c++)
        if (tp[c] > 0.0 && (fb < 0 || tp[c] > tfb)) { fb = c; tfb = tp[c]; }
      if (tfb >= remaining) { last = fb; tlast = tfb; }
      else { r.status = PARVA_RESIDUAL_UNCOVERABLE; return; }
    }
  }
  r.last_sc = (int8_t)last;
  r.count = count;
  r.coverage = with_coverage ? coverage_sum(topt, count, last >= 0, tlast) : 0.0;
  r.status = PARVA_OK;
}

// propose_small_segments (allocator.py:319-359).  tp1/tp2 == 0 -> absent.
// Returns false for SmallSegmentsUnavailableError.
__device__ inline bool propose_small(double tp1, double tp2, double freed, long long& k2o,
                                     long long& k1o) {
  k2o = 0; k1o = 0;
  if (freed <= 0.0) return true;
  if (tp1 == 0.0 && tp2 == 0.0) return false;
  long long max_k2 = 0;
  if (tp2 != 0.0) max_k2 = (long long)ceil(__dsub_rn(__ddiv_rn(freed, tp2), 1e-12));
  double m = (1.0 > freed) ? 1.0 : freed;
  double thr = __dmul_rn(1e-12, m);
  bool have = false;
  long long bg = 0, bc = 0, bn = 0;
  for (long long k2 = 0; k2 <= max_k2; k2++) {
    double covered = tp2 != 0.0 ? __dmul_rn((double)k2, tp2) : 0.0;
    double sh = __dsub_rn(freed, covered);
    long long k1;
    if (sh <= thr) k1 = 0;
    else if (tp1 != 0.0) {
      k1 = (long long)ceil(__dsub_rn(__ddiv_rn(sh, tp1), 1e-12));
      if (k1 < 1) k1 = 1;
    } else continue;
    long long g = 2 * k2 + k1, cn = k2 + k1, nk = -k2;
    if (!have || g < bg || (g == bg && (cn < bc || (cn == bc && nk < bn)))) {
      have = true; bg = g; bc = cn; bn = nk;
    }
  }
  if (!have) return false;
  k2o = -bn;
  k1o = bc + bn;
  return true;
}

// propose_small_segments with the k2 candidates spread over the warp: lane j
// evaluates k2 = base + j, then a lexicographic-min reduction over
// (2*k2+k1, k2+k1, -k2) -- a strict total order (k2 unique), so the result is
// the sequential loop's.  All 32 lanes must call it with the same arguments.
__device__ inline bool propose_small_warp(double tp1, double tp2, double freed, long long& k2o, long long& k1o,
                                          int lane) {
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
  for (long long base = 0; base <= max_k2; base += 32) {
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
    // warp-uniform choice (the reductions are collective).  Small fields:
    // key = gpcs << 20 | count << 10 | (1023 - k2) in 32 bits, one redux.
    if (__all_sync(0xffffffffu, !ok || (2 * k2 + k1 < 4095 && k2 + k1 < 1024 && k2 < 1024))) {
      const unsigned key = ok ? (unsigned)(2 * k2 + k1) << 20 | (unsigned)(k2 + k1) << 10 | (unsigned)(1023 - k2)
                              : 0xFFFFFFFFu;
      const unsigned m = __reduce_min_sync(0xffffffffu, key);
      if (m == 0xFFFFFFFFu) { g = cn = nk = LLONG_MAX; }
      else {
        g = (long long)(m >> 20);
        cn = (long long)((m >> 10) & 1023u);
        nk = (long long)(m & 1023u) - 1023;
      }
    } else if (packed && __all_sync(0xffffffffu, !ok || 2 * k2 + k1 < (1ll << 21))) {
      unsigned long long key = ok ? ((unsigned long long)(2 * k2 + k1) << 42) |
                                        ((unsigned long long)(k2 + k1) << 21) |
                                        (unsigned long long)((1ll << 21) - 1 - k2)
                                  : ~0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long k = __shfl_xor_sync(0xffffffffu, key, o);
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
      for (int o = 16; o > 0; o >>= 1) {
        const long long g2 = __shfl_xor_sync(0xffffffffu, g, o);
        const long long c2 = __shfl_xor_sync(0xffffffffu, cn, o);
        const long long n2 = __shfl_xor_sync(0xffffffffu, nk, o);
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

}  // namespace parva
