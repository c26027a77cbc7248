// simulate.cu — batched run_simulation event loops, sm_100a.
//
// Replaces the heap-driven event loop of the reference simulator
// (evaluation.py:337-416) for many (deployment, workload, seed) runs at once.
// Services never interact in that loop: a service's events only touch its
// own queue, lanes and segments, and the global (time, seq) heap order
// restricted to one service is the order of that service's own pushes.  So
// every service is an independent sequential simulation: one thread each.
//
// Per service (thread):
//   * arrivals: the service's arrival times in ms (sorted; generated on the
//     host with the reference's numpy RNG, evaluation.py:207-226, 327-335);
//     the FIFO queue is the index range [qh, ptr) of that array, ingest()
//     advances ptr (searchsorted(side="right") on a monotone clock);
//   * pending events: one completion per busy lane (time, seq, segment) and
//     at most one arrival wakeup, popped by (time, seq) with a linear scan;
//   * dispatch(): first segment (in dmap order) with a free lane takes
//     min(batch, queue) requests; latency = (now - first) + service_ms;
//     busy_ms += max(0, min(service_ms, horizon - now)).
// Floating-point operations are the reference's, one rounding each
// (--fmad=false), so latencies and busy times are bit-identical.
#include <cuda_runtime.h>

#include "parva_common.cuh"

namespace parva {

constexpr int kSimLanes = 64;     // pending completions per service (its total lanes)
constexpr int kSimSegs = 32;      // segments per service

__global__ void simulate_kernel(parva_sim_problem P, parva_sim_result R) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P.n_services; s += gridDim.x * blockDim.x) {
    const int64_t a0 = P.d_arr_off[s];
    const int64_t na = P.d_arr_off[s + 1] - a0;
    const double* arr = P.d_arrivals + a0;
    const int g0 = P.d_seg_off[s];
    const int ns = P.d_seg_off[s + 1] - g0;
    const double H = P.d_horizon_ms[s];
    const double slo = P.d_slo[s];
    int lanes_total = 0;
    for (int g = 0; g < ns; g++) lanes_total += P.d_seg_lanes[g0 + g];
    if (ns > kSimSegs || lanes_total > kSimLanes) {
      R.d_status[s] = PARVA_CAPACITY;
      continue;
    }
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
    bool wake = false;
    double wake_t = 0.0;
    uint32_t wake_q = 0;
    double* lat = R.d_latency + a0;

    auto schedule_wakeup = [&]() {
      if (wake || ptr >= na) return;
      wake = true;
      wake_t = arr[ptr];
      wake_q = seq++;
    };
    auto ingest = [&](double now) {
      while (ptr < na && arr[ptr] <= now) ptr++;
    };
    auto dispatch = [&](double now) {
      if (now >= H) return;
      while (qh < ptr && free_lanes > 0) {
        int g = 0;
        while (free_seg[g] == 0) g++;
        const double ms = P.d_seg_ms[g0 + g];
        const int64_t qn = ptr - qh;
        const int64_t b = P.d_seg_batch[g0 + g];
        const int64_t n = b < qn ? b : qn;
        const double first = arr[qh];
        qh += n;
        const double latency = __dadd_rn(__dsub_rn(now, first), ms);
        lat[batches++] = latency;
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
    for (;;) {
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
    R.d_served[s] = served;
    R.d_batches[s] = batches;
    R.d_violations[s] = violations;
    for (int g = 0; g < ns; g++) R.d_busy_ms[g0 + g] = busy[g];
    R.d_status[s] = PARVA_OK;
  }
}

}  // namespace parva

extern "C" int parva_simulate(const parva_sim_problem* p, const parva_sim_result* r, void* stream) {
  if (!p || !r || p->n_services < 0) return PARVA_BAD_INPUT;
  if (p->n_services == 0) return PARVA_OK;
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  // one thread per service; small blocks spread the (few, long) threads over every SM
  const int threads = 32;
  int blocks = (p->n_services + threads - 1) / threads;
  if (blocks > n_sm * 32) blocks = n_sm * 32;
  parva::simulate_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(*p, *r);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}
