// simulate.cu — batched run_simulation, sm_100a.
//
// Replaces the reference simulator's arrival generation and heap-driven
// event loop (evaluation.py:207-226, 327-416) for many (deployment,
// workload, seed) runs at once.  Services never interact in that loop: a
// service's events only touch its own queue, lanes and segments, and the
// global (time, seq) heap order restricted to one service is the order of
// that service's own pushes.  So every service is an independent sequential
// simulation: one thread each, in two stages.
//
// * Arrivals, from the service's own numpy generator state (PCG64 XSL-RR
//   128/64, seeded on the host by SeedSequence(seed).spawn(n)[i] exactly as
//   the reference does): Generator.exponential(1/rate, size=chunk) gaps by
//   numpy's ziggurat (tables in numpy_ziggurat.h), per-chunk cumsum plus the
//   previous chunk's last time, stop at the horizon; or the deterministic
//   grid i * step.  Generated lazily, in the order the loop ingests them.
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
// One service per WARP (lane 0): every service's event loop takes its own
// data-dependent path, so services sharing a warp would serialise (a warp
// of 32 services ran ~20x slower than its arithmetic); a warp each also
// spreads the few thousand services over every SM.
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

// A service's arrival stream, generated lazily in order (the event loop
// consumes arrivals strictly in order, so the next one is always a register,
// never a dependent load).  Poisson: numpy exponential gaps, per-chunk cumsum
// plus the previous chunk's last time (evaluation.py:218-226); deterministic:
// i * step (:213-217).  Times in seconds; next() returns ms, false at the
// horizon (times are monotone, so the rest would be filtered out).
struct ArrivalGen {
  Pcg64 g;
  double scale, horizon_s, cs, total;
  int64_t chunk, i;
  int kind;
  bool done;

  __device__ __forceinline__ bool next(double& t_ms) {
    if (done) return false;
    if (kind == 1) {
      if (i == chunk) {                  // the reference draws another chunk while total < horizon
        if (!(total < horizon_s)) { done = true; return false; }
        i = 0;
      }
      const double gap = __dmul_rn(scale, standard_exponential(g));
      cs = i == 0 ? gap : __dadd_rn(cs, gap);
      const double t = __dadd_rn(cs, total);
      if (i == chunk - 1) total = t;
      i++;
      if (t >= horizon_s) { done = true; return false; }
      t_ms = __dmul_rn(t, 1000.0);
      return true;
    }
    if (kind == 2) {
      if (i < chunk) {
        i++;
        const double t = __dmul_rn((double)i, scale);
        if (t < horizon_s) { t_ms = __dmul_rn(t, 1000.0); return true; }
      }
    }
    done = true;
    return false;
  }
};

__global__ void __launch_bounds__(kSimWarps * 32) simulate_kernel(parva_sim_problem P, parva_sim_result R) {
  // the queue head (the oldest waiting arrival) is nearly always one of the
  // last kRing ingested: read it from shared memory, not back from L2
  __shared__ double ring[kRing][kSimWarps];
  const int tx = threadIdx.x >> 5;
  if (threadIdx.x & 31) return;
  for (int s = blockIdx.x * kSimWarps + tx; s < P.n_services; s += gridDim.x * kSimWarps) {
    const int64_t b0 = P.d_buf_off[s];
    const int64_t cap = P.d_buf_off[s + 1] - b0;
    double* buf = R.d_buf + b0;            // ingested arrivals (ms), later the batch latencies
    const int kind = P.d_kind[s];
    ArrivalGen gen;
    gen.g = Pcg64{P.d_pcg[4 * s], P.d_pcg[4 * s + 1], P.d_pcg[4 * s + 2], P.d_pcg[4 * s + 3]};
    gen.scale = P.d_scale[s];
    gen.horizon_s = P.d_horizon_s[s];
    gen.cs = 0.0;
    gen.total = 0.0;
    gen.chunk = P.d_count[s];
    gen.i = kind == 1 ? gen.chunk : 0;
    gen.kind = kind;
    gen.done = kind != 1 && kind != 2;
    const int g0 = P.d_seg_off[s];
    const int ns = P.d_seg_off[s + 1] - g0;
    int lanes_total = 0;
    for (int g = 0; g < ns; g++) lanes_total += P.d_seg_lanes[g0 + g];
    if (ns > kSimSegs || lanes_total > kSimLanes) {
      R.d_status[s] = PARVA_CAPACITY;
      continue;
    }
    const double H = P.d_horizon_ms[s];
    const double slo = P.d_slo[s];
    int free_seg[kSimSegs];
    double busy[kSimSegs];
    for (int g = 0; g < ns; g++) { free_seg[g] = P.d_seg_lanes[g0 + g]; busy[g] = 0.0; }
    double ev_t[kSimLanes];
    uint32_t ev_q[kSimLanes];
    uint8_t ev_g[kSimLanes];
    int n_ev = 0;
    int free_lanes = lanes_total;
    int64_t ptr = 0, qh = 0, batches = 0, served = 0, violations = 0;
    uint32_t seq = 0;
    bool wake = false, overflow = false;
    double wake_t = 0.0;
    uint32_t wake_q = 0;
    double nt = 0.0;                       // next arrival not yet ingested (arr[ptr])
    bool have = gen.next(nt);

    auto schedule_wakeup = [&]() {        // evaluation.py:362-366
      if (wake || !have) return;
      wake = true;
      wake_t = nt;
      wake_q = seq++;
    };
    auto ingest = [&](double now) {       // evaluation.py:353-360
      while (have && nt <= now) {
        if (ptr == cap) { overflow = true; have = false; break; }
        buf[ptr] = nt;
        ring[ptr & (kRing - 1)][tx] = nt;
        ptr++;
        have = gen.next(nt);
      }
    };
    auto dispatch = [&](double now) {     // evaluation.py:368-388
      if (now >= H) return;
      while (qh < ptr && free_lanes > 0) {
        int g = 0;
        while (free_seg[g] == 0) g++;
        const double ms = P.d_seg_ms[g0 + g];
        const int64_t qn = ptr - qh;
        const int64_t b = P.d_seg_batch[g0 + g];
        const int64_t n = b < qn ? b : qn;
        const double first = ptr - qh <= kRing ? ring[qh & (kRing - 1)][tx] : buf[qh];
        qh += n;
        const double latency = __dadd_rn(__dsub_rn(now, first), ms);
        buf[batches++] = latency;          // slot < qh: that arrival has left the queue
        served += n;
        if (latency > slo) violations++;
        free_seg[g]--;
        free_lanes--;
        const double rem = __dsub_rn(H, now);
        const double m = ms < rem ? ms : rem;
        busy[g] = __dadd_rn(busy[g], m > 0.0 ? m : 0.0);
        ev_t[n_ev] = __dadd_rn(now, ms);
        ev_q[n_ev] = seq++;
        ev_g[n_ev] = (uint8_t)g;
        n_ev++;
      }
    };

    if (ns > 0) schedule_wakeup();
    for (;;) {                             // evaluation.py:395-416
      // pop the (time, seq)-smallest pending event
      int best = -1;
      double bt = 0.0;
      uint32_t bq = 0;
      for (int e = 0; e < n_ev; e++)
        if (best < 0 || ev_t[e] < bt || (ev_t[e] == bt && ev_q[e] < bq)) { best = e; bt = ev_t[e]; bq = ev_q[e]; }
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
        const int g = ev_g[best];
        ev_t[best] = ev_t[n_ev - 1];
        ev_q[best] = ev_q[n_ev - 1];
        ev_g[best] = ev_g[n_ev - 1];
        n_ev--;
        free_seg[g]++;
        free_lanes++;
        if (now < H) {
          ingest(now);
          dispatch(now);
          if (qh == ptr) schedule_wakeup();
        }
      }
    }
    // arrivals never ingested still count (ServiceSimStats.arrived)
    int64_t arrived = ptr + (have ? 1 : 0);
    if (have) {
      double t;
      while (gen.next(t)) arrived++;
    }
    R.d_arrived[s] = arrived;
    R.d_served[s] = served;
    R.d_batches[s] = batches;
    R.d_violations[s] = violations;
    for (int g = 0; g < ns; g++) R.d_busy_ms[g0 + g] = busy[g];
    R.d_status[s] = overflow ? PARVA_CAPACITY : PARVA_OK;
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
