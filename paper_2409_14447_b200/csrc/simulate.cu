// simulate.cu — batched run_simulation, sm_100a.
//
// Replaces the reference simulator's arrival generation and heap-driven
// event loop (evaluation.py:207-226, 327-416) for many (deployment,
// workload, seed) runs at once.  Services never interact in that loop: a
// service's events only touch its own queue, lanes and segments, and the
// global (time, seq) heap order restricted to one service is the order of
// that service's own pushes.  So every service is an independent sequential
// simulation: one warp each, in two stages.
//
// * Arrivals, from the service's own numpy generator state (PCG64 XSL-RR
//   128/64, seeded on the host by SeedSequence(seed).spawn(n)[i] exactly as
//   the reference does): Generator.exponential(1/rate, size=chunk) gaps by
//   numpy's ziggurat (tables in numpy_ziggurat.h), per-chunk cumsum plus the
//   previous chunk's last time, stop at the horizon; or the deterministic
//   grid i * step.  Draws are generated 32 at a time by the warp's lanes
//   (PCG64 jump-ahead), gaps consumed lazily in the order the loop ingests.
// * The event loop: the FIFO queue is the index range [qh, ptr) of the
//   ingested arrivals; ingest() moves arrivals <= now into the buffer
//   (searchsorted(side="right") on a monotone clock); pending events are one
//   completion per busy lane plus at most one arrival wakeup, popped by
//   (time, seq); dispatch() gives the first segment (deployment-map order)
//   with a free lane min(batch, queue) requests.  Batch latencies overwrite
//   the consumed prefix of the buffer (batch b is written after >= b + 1
//   arrivals left the queue).
// Every floating-point operation is the reference's, one rounding each
// (--fmad=false; explicit __fma_rn only where glibc's log1p fuses).
#include <cuda_runtime.h>

#include "numpy_ziggurat.h"
#include "parva_common.cuh"

namespace parva {

constexpr int kSimLanes = 64;     // pending completions per service (its total lanes)
constexpr int kSimSegs = 32;      // segments per service
// One service per WARP: every service's event loop takes its own
// data-dependent path, so services sharing a warp would serialise (a warp
// of 32 services ran ~20x slower than its arithmetic); a warp each also
// spreads the few thousand services over every SM, and its lanes generate
// the service's random draws 32 at a time.
constexpr int kSimWarps = 4;      // services (warps) per CTA
constexpr int kRing = 32;         // last ingested arrivals per service, in shared memory

// ------------------------------------------------------------- numpy PCG64
struct Pcg64 {
  uint64_t hi, lo, inc_hi, inc_lo;

  __device__ __forceinline__ uint64_t next64() {
    // state = state * 0x2360ED051FC65DA44385DF649FCCF645 + inc (mod 2^128), then XSL-RR
    const uint64_t mlo = 0x4385DF649FCCF645ull, mhi = 0x2360ED051FC65DA4ull;
    uint64_t nlo = lo * mlo;
    uint64_t nhi = __umul64hi(lo, mlo) + hi * mlo + lo * mhi;
    nlo += inc_lo;
    nhi += inc_hi + (nlo < inc_lo ? 1ull : 0ull);
    lo = nlo;
    hi = nhi;
    const uint64_t x = nhi ^ nlo;
    const unsigned rot = (unsigned)(nhi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  __device__ __forceinline__ double next_double() {
    return __dmul_rn((double)(next64() >> 11), 1.0 / 9007199254740992.0);
  }
};

// glibc's log1p (sysdeps/ieee754/dbl-64/s_log1p.c, the FMA build its ifunc
// picks on x86-64 hosts) for x in (-1, 0]: the argument numpy's exponential
// tail passes (evaluation's ziggurat: r - log1p(-U)).  Same operations and
// the same fused multiply-adds, so the value is bit-identical (checked on
// 2.2e8 random inputs against the host libm, tools/sim/log1p_check).
__device__ __forceinline__ double glibc_log1p_neg(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = (int32_t)(__double_as_longlong(x) >> 32);
  const int32_t ax = hx & 0x7fffffff;
  if (ax < 0x3e200000) {                                  // |x| < 2^-29
    if (ax < 0x3c900000) return x;
    return __fma_rn(-__dmul_rn(x, x), 0.5, x);
  }
  int k = 0;
  double f, c = 0.0;
  int32_t hu;
  if (hx < (int32_t)0xbfd2bec4) {                          // sqrt(2)/2- <= 1+x: k = 0, f = x
    f = x;
    hu = 1;
  } else {
    const double u0 = __dadd_rn(x, 1.0);
    hu = (int32_t)(__double_as_longlong(u0) >> 32);
    k = (hu >> 20) - 1023;
    c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u0, x)) : __dsub_rn(x, __dsub_rn(u0, 1.0));
    c = __ddiv_rn(c, u0);
    hu &= 0x000fffff;
    const uint64_t lo32 = (uint64_t)__double_as_longlong(u0) & 0xffffffffull;
    double u;
    if (hu < 0x6a09e) {
      u = __longlong_as_double((long long)(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | lo32));
    } else {
      k += 1;
      u = __longlong_as_double((long long)(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | lo32));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    }
    const double R = __dmul_rn(__fma_rn(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double sr = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, sr));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(dk, ln2_lo, c), sr)), f));
}

// numpy random_standard_exponential (distributions.c, ziggurat method)
__device__ __forceinline__ double standard_exponential(Pcg64& g) {
  for (;;) {
    uint64_t ri = g.next64() >> 3;
    const int idx = (int)(ri & 0xFF);
    ri >>= 8;
    const double x = __dmul_rn((double)ri, __ldg(&kZigWe[idx]));
    if (ri < __ldg(&kZigKe[idx])) return x;
    if (idx == 0) return __dsub_rn(kZigExpR, glibc_log1p_neg(-g.next_double()));
    const double fe1 = __ldg(&kZigFe[idx - 1]), fe0 = __ldg(&kZigFe[idx]);
    if (__dadd_rn(__dmul_rn(__dsub_rn(fe1, fe0), g.next_double()), fe0) < exp(-x)) return x;
  }
}

// ------------------------------------------------ warp-cooperative arrivals
// A service's arrivals are a strictly sequential stream (PCG64 draws -> the
// ziggurat -> per-chunk cumsum), but the draws themselves are an affine
// recurrence mod 2^128, so a warp takes 32 at once: lane L jumps the base
// state by L + 1 steps (s' = A_L s + C_L, (A_L, C_L) = the (L+1)-fold step,
// from a warp scan at service start), maps its draw through the ziggurat's
// fast path, and the rare slow draws (about 1 in 80: the tail or a wedge
// test, each consuming the next draw as its uniform) are resolved in stream
// order by walking the ballot of slow lanes.  The gaps land in shared memory
// in draw order; the event loop -- run by all 32 lanes in lockstep on
// identical values -- consumes them one by one.
struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  return U128{__umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi, a.lo * b.lo};
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  const uint64_t lo = a.lo + b.lo;
  return U128{a.hi + b.hi + (lo < a.lo ? 1ull : 0ull), lo};
}
__device__ __forceinline__ U128 shfl128(U128 v, int src) {
  return U128{__shfl_sync(0xffffffffu, v.hi, src), __shfl_sync(0xffffffffu, v.lo, src)};
}
__device__ __forceinline__ U128 shfl_up128(U128 v, int o) {
  return U128{__shfl_up_sync(0xffffffffu, v.hi, o), __shfl_up_sync(0xffffffffu, v.lo, o)};
}
__device__ __forceinline__ uint64_t xsl_rr(U128 st) {
  const uint64_t x = st.hi ^ st.lo;
  const unsigned rot = (unsigned)(st.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double draw_double(uint64_t o) {
  return __dmul_rn((double)(o >> 11), 1.0 / 9007199254740992.0);
}
// the slow branch of random_standard_exponential for draw (idx, x) and the
// next draw's uniform u: the tail value, or x if the wedge test accepts
__device__ __forceinline__ bool zig_slow(int idx, double x, double u, double& e) {
  if (idx == 0) { e = __dsub_rn(kZigExpR, glibc_log1p_neg(-u)); return true; }
  const double fe1 = __ldg(&kZigFe[idx - 1]), fe0 = __ldg(&kZigFe[idx]);
  if (__dadd_rn(__dmul_rn(__dsub_rn(fe1, fe0), u), fe0) < exp(-x)) { e = x; return true; }
  return false;
}

// per-warp (per-service) shared state: generated gaps, the queue-head ring,
// pending completions and the segments (one copy; every lane reads and
// writes the same values)
struct alignas(16) SimWarp {
  double smp[64];                 // scale * exponential draws, in stream order
  double tm[32];                  // next arrival times (ms), in order
  double ring[kRing];             // last kRing ingested arrivals (ms)
  double ev_t[kSimLanes];         // pending completions, one FIFO per segment
  uint32_t ev_q[kSimLanes];       // (segment g's slots: [sg_lo, sg_lo + lanes_g), lane g's registers)
};

// Arrival stream of one service (evaluation.py:207-226): Poisson = numpy
// exponential gaps, per-chunk cumsum plus the previous chunk's last time;
// deterministic = i * step.  Times in seconds; next() returns ms, false at the
// horizon (times are monotone, so the rest would be filtered out).
struct WarpArrivals {
  U128 st;                        // base PCG64 state (uniform)
  U128 ja, jc;                    // this lane's jump: L + 1 steps
  double scale, horizon_s, cs, total, pend_x;
  int64_t chunk, i;
  int kind, head, cnt, pend_idx, lane;
  int th, tn;                     // W.tm[th, tn): arrival times not yet ingested
  bool done, pend;

  __device__ __forceinline__ void init(const uint64_t* pcg, int kind_, double scale_, double hs, int64_t count,
                                       int lane_) {
    st = U128{pcg[0], pcg[1]};
    const U128 inc{pcg[2], pcg[3]};
    lane = lane_;
    // (A, C) of one step is (M, inc); inclusive warp scan of the composition
    // (A, C) o (A', C') = (A A', A C' + C): lane L ends with L + 1 steps
    ja = U128{0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
    jc = inc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const U128 pa = shfl_up128(ja, o), pc = shfl_up128(jc, o);
      if (lane >= o) {
        jc = add128(mul128(ja, pc), jc);
        ja = mul128(ja, pa);
      }
    }
    kind = kind_;
    scale = scale_;
    horizon_s = hs;
    cs = 0.0;
    total = 0.0;
    chunk = count;
    i = kind == 1 ? chunk : 0;
    done = kind != 1 && kind != 2;
    head = cnt = 0;
    th = tn = 0;
    pend = false;
    pend_idx = 0;
    pend_x = 0.0;
  }

  // 32 more draws -> the gaps they complete, in order (warp-collective)
  __device__ __noinline__ void refill(SimWarp& W) {
    __syncwarp();                  // every lane's reads of the old samples precede the overwrite
    cnt = 0;
    head = 0;
    do {
      const U128 s = add128(mul128(ja, st), jc);
      const uint64_t out = xsl_rr(s);
      st = shfl128(s, 31);
      uint64_t ri = out >> 3;
      const int idx = (int)(ri & 0xFF);
      ri >>= 8;
      const double x = __dmul_rn((double)ri, __ldg(&kZigWe[idx]));
      const unsigned slow = __ballot_sync(0xffffffffu, !(ri < __ldg(&kZigKe[idx])));
      int pos = 0;
      if (pend) {                 // the last batch ended on a slow draw: its uniform is draw 0
        const double u = draw_double(__shfl_sync(0xffffffffu, out, 0));
        double e;
        if (zig_slow(pend_idx, pend_x, u, e)) W.smp[cnt++] = __dmul_rn(scale, e);
        pend = false;
        pos = 1;
      }
      while (pos < 32) {
        const unsigned m = slow & (0xffffffffu << pos);
        const int sl = m ? __ffs(m) - 1 : 32;
        if (lane >= pos && lane < sl) W.smp[cnt + lane - pos] = __dmul_rn(scale, x);
        cnt += sl - pos;
        if (sl >= 31) {
          if (sl == 31) {
            pend = true;
            pend_idx = __shfl_sync(0xffffffffu, idx, 31);
            pend_x = __shfl_sync(0xffffffffu, x, 31);
          }
          break;
        }
        const double u = draw_double(__shfl_sync(0xffffffffu, out, sl + 1));
        const int si = __shfl_sync(0xffffffffu, idx, sl);
        const double sx = __shfl_sync(0xffffffffu, x, sl);
        double e;
        if (zig_slow(si, sx, u, e)) W.smp[cnt++] = __dmul_rn(scale, e);
        pos = sl + 2;
      }
    } while (cnt == 0);
    __syncwarp();
  }

  // the next up to 32 arrival times (ms) into W.tm[0, tn): the reference's
  // per-chunk cumsum plus the previous chunk's last time (a sequential
  // chain), or the grid i * step; false once the horizon is reached
  __device__ __noinline__ bool fill(SimWarp& W) {
    __syncwarp();                  // every lane's reads of the old times precede the overwrite
    th = tn = 0;
    while (!done && tn == 0) {
      if (kind == 1) {
        while (tn < 32) {
          if (i == chunk) {              // the reference draws another chunk while total < horizon
            if (!(total < horizon_s)) { done = true; break; }
            i = 0;
          }
          if (head == cnt) refill(W);
          const double gap = W.smp[head++];
          cs = i == 0 ? gap : __dadd_rn(cs, gap);
          const double t = __dadd_rn(cs, total);
          if (i == chunk - 1) total = t;
          i++;
          if (t >= horizon_s) { done = true; break; }
          W.tm[tn++] = __dmul_rn(t, 1000.0);
        }
      } else if (kind == 2) {
        while (tn < 32) {
          if (i >= chunk) { done = true; break; }
          i++;
          const double t = __dmul_rn((double)i, scale);
          if (!(t < horizon_s)) { done = true; break; }
          W.tm[tn++] = __dmul_rn(t, 1000.0);
        }
      } else {
        done = true;
      }
    }
    __syncwarp();
    return tn > 0;
  }

  // next arrival not yet ingested: its time, or false if there is none
  __device__ __forceinline__ bool peek(SimWarp& W, double& t_ms) {
    if (th == tn && !fill(W)) return false;
    t_ms = W.tm[th];
    return true;
  }
};

// One service per warp.  Every lane runs the event loop on identical values
// (so the generator's collectives are always converged); lane 0 alone
// writes global memory.
__global__ void __launch_bounds__(kSimWarps * 32) simulate_kernel(parva_sim_problem P, parva_sim_result R) {
  __shared__ SimWarp sw[kSimWarps];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SimWarp& W = sw[wi];
  for (int s = blockIdx.x * kSimWarps + wi; s < P.n_services; s += gridDim.x * kSimWarps) {
    const int64_t b0 = P.d_buf_off[s];
    const int64_t cap = P.d_buf_off[s + 1] - b0;
    double* buf = R.d_buf + b0;            // ingested arrivals (ms), later the batch latencies
    const int kind = P.d_kind[s];
    WarpArrivals gen;
    gen.init(P.d_pcg + 4 * s, kind, P.d_scale[s], P.d_horizon_s[s], P.d_count[s], lane);
    const int g0 = P.d_seg_off[s];
    const int ns = P.d_seg_off[s + 1] - g0;
    if (ns > kSimSegs) {
      if (lane == 0) R.d_status[s] = PARVA_CAPACITY;
      continue;
    }
    // segment g's state lives in lane g's registers: free lanes, busy time,
    // service time, batch size, and its completion FIFO (slots [sg_lo,
    // sg_lo + sg_lanes) of W.ev_*, head cached in head_t / head_q)
    const bool own = lane < ns;
    const int sg_lanes = own ? P.d_seg_lanes[g0 + lane] : 0;
    const double sg_ms = own ? P.d_seg_ms[g0 + lane] : 0.0;
    const int64_t sg_batch = own ? (int64_t)P.d_seg_batch[g0 + lane] : 0;
    int sg_lo = sg_lanes;                  // exclusive prefix of the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, sg_lo, o);
      if (lane >= o) sg_lo += v;
    }
    const int lanes_total = __shfl_sync(0xffffffffu, sg_lo, 31);
    sg_lo -= sg_lanes;
    if (lanes_total > kSimLanes) {
      if (lane == 0) R.d_status[s] = PARVA_CAPACITY;
      continue;
    }
    int sg_free = sg_lanes, sg_head = 0, sg_n = 0;
    double sg_busy = 0.0, head_t = 0.0;
    uint32_t head_q = 0;
    const double H = P.d_horizon_ms[s];
    const double slo = P.d_slo[s];
    // reduction rounds that cover the segments (lane g = segment g)
    const int seg_rounds = ns <= 1 ? 0 : 32 - __clz(ns - 1);
    int free_lanes = lanes_total;
    int64_t ptr = 0, qh = 0, batches = 0, served = 0, violations = 0;
    uint32_t seq = 0;
    bool wake = false, overflow = false;
    double wake_t = 0.0;
    uint32_t wake_q = 0;
    double nt = 0.0;                       // next arrival not yet ingested (arr[ptr])
    bool have = gen.peek(W, nt);

    auto schedule_wakeup = [&]() {        // evaluation.py:362-366
      if (wake || !have) return;
      wake = true;
      wake_t = nt;
      wake_q = seq++;
    };
    auto ingest = [&](double now) {       // evaluation.py:353-360
      // arrivals <= now, a batch of up to 32 per step: times are monotone, so
      // the lanes whose time is <= now are a prefix
      while (have && nt <= now) {
        const int rem = gen.tn - gen.th;
        const unsigned le = __ballot_sync(0xffffffffu, lane < rem && W.tm[gen.th + lane] <= now);
        int take = __popc(le);
        if (take > cap - ptr) { take = (int)(cap - ptr); overflow = true; }
        if (lane < take) {
          const double v = W.tm[gen.th + lane];
          buf[ptr + lane] = v;
          W.ring[(ptr + lane) & (kRing - 1)] = v;
        }
        __syncwarp();
        ptr += take;
        gen.th += take;
        if (overflow) { have = false; break; }
        have = gen.peek(W, nt);
      }
    };
    auto dispatch = [&](double now) {     // evaluation.py:368-388
      if (now >= H) return;
      while (qh < ptr && free_lanes > 0) {
        const int g = __ffs(__ballot_sync(0xffffffffu, own && sg_free > 0)) - 1;
        const double ms = __shfl_sync(0xffffffffu, sg_ms, g);
        const int64_t qn = ptr - qh;
        const int64_t b = __shfl_sync(0xffffffffu, sg_batch, g);
        const int64_t n = b < qn ? b : qn;
        const double first = ptr - qh <= kRing ? W.ring[qh & (kRing - 1)] : buf[qh];
        qh += n;
        const double latency = __dadd_rn(__dsub_rn(now, first), ms);
        __syncwarp();                      // every lane has read buf[qh] before lane 0 overwrites a slot
        if (lane == 0) buf[batches] = latency;   // slot < qh: that arrival has left the queue
        batches++;
        served += n;
        if (latency > slo) violations++;
        free_lanes--;
        const double rem = __dsub_rn(H, now);
        const double m = ms < rem ? ms : rem;
        const double t_done = __dadd_rn(now, ms);
        const uint32_t q = seq++;
        if (lane == g) {
          sg_free--;
          sg_busy = __dadd_rn(sg_busy, m > 0.0 ? m : 0.0);
          // a segment's completions are pushed in (time, seq) order (now is
          // monotone, ms fixed), so each segment's pending events are a FIFO
          int slot = sg_head + sg_n;
          if (slot >= sg_lanes) slot -= sg_lanes;
          W.ev_t[sg_lo + slot] = t_done;
          W.ev_q[sg_lo + slot] = q;
          if (sg_n == 0) { head_t = t_done; head_q = q; }
          sg_n++;
        }
      }
    };

    if (ns > 0) schedule_wakeup();
    for (;;) {                             // evaluation.py:395-416
      // pop the (time, seq)-smallest pending event: the smallest FIFO head
      // over the segments (lane g = segment g, argmin over the lanes that
      // cover the segments; seqs are unique, so it is exact)
      int best = -1;
      double bt = 0.0;
      uint32_t bq = 0;
      if (free_lanes < lanes_total) {
        int ei = -1;
        double et = 0.0;
        uint32_t eq = 0xFFFFFFFFu;
        if (own && sg_n > 0) { et = head_t; eq = head_q; ei = lane; }
        for (int r = 0; r < seg_rounds; r++) {
          const int o = 1 << r;
          const double t2 = __shfl_xor_sync(0xffffffffu, et, o);
          const uint32_t q2 = __shfl_xor_sync(0xffffffffu, eq, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, ei, o);
          if (i2 >= 0 && (ei < 0 || t2 < et || (t2 == et && q2 < eq))) { et = t2; eq = q2; ei = i2; }
        }
        best = __shfl_sync(0xffffffffu, ei, 0);
        bt = __shfl_sync(0xffffffffu, et, 0);
        bq = __shfl_sync(0xffffffffu, eq, 0);
      }
      const bool take_wake = wake && (best < 0 || wake_t < bt || (wake_t == bt && wake_q < bq));
      if (best < 0 && !take_wake) break;
      if (take_wake) {
        const double now = wake_t;
        wake = false;
        ingest(now);
        dispatch(now);
        if (free_lanes > 0) schedule_wakeup();
      } else {
        const double now = bt;
        if (lane == best) {
          sg_head = sg_head + 1 == sg_lanes ? 0 : sg_head + 1;
          sg_n--;
          sg_free++;
          if (sg_n > 0) { head_t = W.ev_t[sg_lo + sg_head]; head_q = W.ev_q[sg_lo + sg_head]; }
        }
        free_lanes++;
        if (now < H) {
          ingest(now);
          dispatch(now);
          if (qh == ptr) schedule_wakeup();
        }
      }
    }
    // arrivals never ingested still count (ServiceSimStats.arrived)
    int64_t arrived = ptr;
    if (have) {
      arrived += gen.tn - gen.th;
      while (gen.fill(W)) arrived += gen.tn;
    }
    if (lane == 0) {
      R.d_arrived[s] = arrived;
      R.d_served[s] = served;
      R.d_batches[s] = batches;
      R.d_violations[s] = violations;

      R.d_status[s] = overflow ? PARVA_CAPACITY : PARVA_OK;
    }
    if (own) R.d_busy_ms[g0 + lane] = sg_busy;
    __syncwarp();
  }
}

// glibc log1p check kernel (tests): out[i] = glibc_log1p_neg(x[i])
__global__ void log1p_kernel(const double* x, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = glibc_log1p_neg(x[i]);
}

// numpy exponential check kernel (tests): draws of Generator.exponential(scale)
__global__ void exponential_kernel(const uint64_t* pcg, double scale, int64_t n, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  Pcg64 g{pcg[0], pcg[1], pcg[2], pcg[3]};
  for (int64_t i = 0; i < n; i++) out[i] = __dmul_rn(scale, standard_exponential(g));
}

}  // namespace parva

extern "C" int parva_simulate(const parva_sim_problem* p, const parva_sim_result* r, void* stream) {
  if (!p || !r || p->n_services < 0) return PARVA_BAD_INPUT;
  if (p->n_services == 0) return PARVA_OK;
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  // one warp per service (lane 0), kSimWarps services per CTA
  int blocks = (p->n_services + parva::kSimWarps - 1) / parva::kSimWarps;
  if (blocks > n_sm * 16) blocks = n_sm * 16;
  parva::simulate_kernel<<<blocks, parva::kSimWarps * 32, 0, (cudaStream_t)stream>>>(*p, *r);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

extern "C" int parva_sim_log1p(const double* d_x, double* d_out, int64_t n, void* stream) {
  if (n < 0) return PARVA_BAD_INPUT;
  if (n == 0) return PARVA_OK;
  parva::log1p_kernel<<<592, 256, 0, (cudaStream_t)stream>>>(d_x, d_out, n);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

extern "C" int parva_sim_exponential(const uint64_t* d_pcg, double scale, int64_t n, double* d_out, void* stream) {
  if (n < 0) return PARVA_BAD_INPUT;
  if (n == 0) return PARVA_OK;
  parva::exponential_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_pcg, scale, n, d_out);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}
