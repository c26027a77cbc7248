// plan_general.cu — KG: relocate_segments / optimize_allocation on an
// arbitrary problem (any number of services and GPUs, arbitrary input
// DeploymentMap, GPU ids and ledger).  Used for the object API
// (relocate_segments, optimize_allocation) and for scenarios that overflow
// the fast path's 128-byte record (PARVA_CAPACITY).
//
// The allocator's optimize pass is a serial dependency chain (SURVEY.md
// §8e): one thread walks it.  First-fit is O(1) amortised through per-size
// "accepts" bitmaps with a lowest-nonzero-word hint instead of the
// reference's O(M) scans and O(M) _next_id (allocator.py:204-281), which is
// what makes the 10^5-segment case (C5) cheap.  Ledger rollback uses an undo
// log instead of the reference's whole-dict snapshot (allocator.py:387,418-419):
// same observable ledger, O(touched) instead of O(services) per GPU.
#include <cuda_runtime.h>

#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

struct GenWs {
  int64_t* id;
  uint8_t* mask;
  uint8_t* len;
  uint8_t* ngpc;
  int32_t* lcat;    // [cap*7]
  uint8_t* lslot;   // [cap*7]
  int64_t* b_id;    // backup (optimize input) for the regression fallback
  uint8_t* b_mask;
  uint8_t* b_len;
  uint8_t* b_ngpc;
  int32_t* b_lcat;
  uint8_t* b_lslot;
  uint64_t* acc;    // [5 * words]
  int32_t* q;       // proposal queue (size-2 part then size-1 part) [qcap]
  int32_t* q1;      // [qcap]
  int32_t* undo;    // [qcap]
  double* after;    // [n_services]
  uint8_t* seen;    // [n_services]
  int64_t* svc_pos; // [n_services + 1] relocation queue offsets of one size class
  int64_t* gpu_pos; // [cap + 1] cumulative capacity of one size class
  int64_t* hdr;     // [8]: G, max_id, status, next (ledger rank counter)
  int64_t words, qcap, cap;
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline size_t gen_layout(int64_t cap, int64_t qcap, int n_services, uint8_t* base,
                                             GenWs* w) {
  const int64_t words = (cap + 63) / 64;
  size_t off = 0;
  auto take = [&](size_t bytes) { uint8_t* p = base ? base + off : nullptr; off += align_up(bytes); return p; };
  GenWs t;
  t.id = (int64_t*)take(cap * 8); t.mask = take(cap); t.len = take(cap); t.ngpc = take(cap);
  t.lcat = (int32_t*)take(cap * 7 * 4); t.lslot = take(cap * 7);
  t.b_id = (int64_t*)take(cap * 8); t.b_mask = take(cap); t.b_len = take(cap); t.b_ngpc = take(cap);
  t.b_lcat = (int32_t*)take(cap * 7 * 4); t.b_lslot = take(cap * 7);
  t.acc = (uint64_t*)take(5 * words * 8);
  t.q = (int32_t*)take(qcap * 4); t.q1 = (int32_t*)take(qcap * 4); t.undo = (int32_t*)take(qcap * 4);
  t.after = (double*)take((size_t)(n_services + 1) * 8); t.seen = take(n_services + 1);
  t.svc_pos = (int64_t*)take((size_t)(n_services + 2) * 8); t.gpu_pos = (int64_t*)take((size_t)(cap + 2) * 8);
  t.hdr = (int64_t*)take(8 * 8);
  t.words = words; t.qcap = qcap; t.cap = cap;
  if (w) *w = t;
  return off;
}

struct Gen {
  const parva_general_problem P;
  GenWs w;
  int64_t G;
  int64_t max_id;
  int64_t hint[5];

  __device__ void set_acc(int64_t g) {
    const uint32_t m = w.mask[g];
    const int64_t word = g >> 6;
    const uint64_t bit = 1ull << (g & 63);
#pragma unroll
    for (int c = 0; c < 5; c++) {
      uint64_t* a = &w.acc[c * w.words + word];
      if (find_start(m, c) >= 0) {
        *a |= bit;
        if (word < hint[c]) hint[c] = word;
      } else {
        *a &= ~bit;
      }
    }
  }

  // first GPU (list order) accepting size class c, skipping `exclude`
  __device__ int64_t first_fit(int c, int64_t exclude) {
    const uint64_t* a = &w.acc[c * w.words];
    const int64_t nw = (G + 63) >> 6;
    int64_t k = hint[c];
    bool moving = true;
    for (; k < nw; k++) {
      uint64_t v = a[k];
      if (moving && v == 0) { hint[c] = k + 1; continue; }
      moving = false;
      if (exclude >= 0 && (exclude >> 6) == k) v &= ~(1ull << (exclude & 63));
      if (k == nw - 1 && (G & 63)) v &= (1ull << (G & 63)) - 1;
      if (v) return k * 64 + __ffsll((long long)v) - 1;
    }
    return -1;
  }

  __device__ void put(int64_t g, int cat) {
    const int c = class_of(cat);
    const int st = find_start(w.mask[g], c);
    w.mask[g] |= (uint8_t)footprint(c, st);
    w.ngpc[g] += (uint8_t)size_of_class(c);
    w.lcat[g * 7 + w.len[g]] = cat;
    w.lslot[g * 7 + w.len[g]] = (uint8_t)st;
    w.len[g]++;
    set_acc(g);
  }

  __device__ void pop(int64_t g) {
    const int k = --w.len[g];
    const int c = class_of(w.lcat[g * 7 + k]);
    w.mask[g] &= (uint8_t)~footprint(c, w.lslot[g * 7 + k]);
    w.ngpc[g] -= (uint8_t)size_of_class(c);
    set_acc(g);
  }

  __device__ int class_of(int cat) const {
    switch (P.d_cat_size[cat]) {
      case 1: return 0;
      case 2: return 1;
      case 3: return 2;
      case 4: return 3;
      default: return 4;
    }
  }

  // _FirstFit.place (allocator.py:194-251); returns GPU index, -1 no fit, -2 capacity
  __device__ int64_t place(int cat, int64_t exclude, bool allow_new) {
    int64_t g = first_fit(class_of(cat), exclude);
    if (g < 0) {
      if (!allow_new) return -1;
      if (G >= w.cap) return -2;
      g = G++;
      w.id[g] = ++max_id;  // _next_id: max(ids) + 1
      w.mask[g] = 0; w.len[g] = 0; w.ngpc[g] = 0;
      set_acc(g);
    }
    put(g, cat);
    return g;
  }
};

// ------------------------------------------------------------------ helpers
// successive greedy placements of size class c on a GPU with mask m
__device__ __forceinline__ int fill_cap(uint32_t m, int c) {
  int k = 0, st;
  while ((st = find_start(m, c)) >= 0) { m |= footprint(c, st); k++; }
  return k;
}
__device__ __forceinline__ int fill_start(uint32_t m, int c, int j) {
  for (int k = 0;; k++) {
    const int st = find_start(m, c);
    if (k == j) return st;
    m |= footprint(c, st);
  }
}
__device__ __forceinline__ uint32_t fill_mask(uint32_t m, int c, int used) {
  for (int k = 0; k < used; k++) m |= footprint(c, find_start(m, c));
  return m;
}

// exclusive block scan (1024 threads) of f(i), i < n, into out[0..n]; returns the total
template <class F>
__device__ int64_t block_scan(int64_t n, F f, int64_t* out, int64_t* sh /*[33]*/) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + tid;
    const int64_t v = i < n ? f(i) : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) sh[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0, wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += u;
      }
      sh[lane] = wi - w;        // exclusive warp offsets
      if (lane == 31) sh[32] = wi;
    }
    __syncthreads();
    if (i < n) out[i] = carry + sh[warp] + incl - v;
    carry += sh[32];
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
  __syncthreads();
  return carry;
}

__device__ __forceinline__ int64_t upper_bound64(const int64_t* a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;   // first index with a[idx] > x
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int class_of_size(int size) {
  return size == 7 ? 4 : size - 1;
}

// Initial map, ledger, and relocate_segments (allocator.py:292-316) in
// parallel.  Within one size class, first-fit fills GPUs strictly in list
// order -- a placement changes only the GPU it lands on, so every earlier
// GPU keeps rejecting the class -- and each GPU receives its greedy capacity
// for the class before the next one gets anything; GPUs appended when none
// accepts fill the same way.  So a class phase is: scan the per-service
// queue lengths, scan the per-GPU capacities, scatter queue entry i to the
// GPU whose capacity range holds i.
__global__ void __launch_bounds__(1024) gen_prepare_kernel(parva_general_problem P, parva_general_result R,
                                                            uint8_t* ws_base, int64_t cap, int64_t qcap) {
  GenWs w;
  gen_layout(cap, qcap, P.n_services, ws_base, &w);
  __shared__ int64_t sh[33];
  __shared__ unsigned long long s_max;
  __shared__ int s_next;
  const int tid = threadIdx.x;
  if (tid == 0) { s_max = 0; s_next = 0; }
  __syncthreads();
  for (int64_t g = tid; g < P.n_gpus; g += blockDim.x) {
    w.id[g] = P.d_gpu_id[g];
    atomicMax(&s_max, (unsigned long long)(P.d_gpu_id[g] + (1ll << 62)));
    uint32_t m = 0;
    int ng = 0, n = 0;
    for (int k = P.d_pl_off[g]; k < P.d_pl_off[g + 1]; k++, n++) {
      const int cat = P.d_pl_cat[k], c = class_of_size(P.d_cat_size[cat]);
      m |= footprint(c, P.d_pl_slot[k]);
      ng += size_of_class(c);
      w.lcat[g * 7 + n] = cat;
      w.lslot[g * 7 + n] = P.d_pl_slot[k];
    }
    w.mask[g] = (uint8_t)m; w.len[g] = (uint8_t)n; w.ngpc[g] = (uint8_t)ng;
  }
  for (int k = tid; k < P.n_names; k += blockDim.x) {
    R.d_ledger_val[k] = P.d_ledger_val[k];
    R.d_ledger_order[k] = P.d_ledger_order[k];
    atomicMax(&s_next, P.d_ledger_order[k]);
  }
  __syncthreads();
  int64_t G = P.n_gpus;
  int64_t max_id = P.n_gpus ? (int64_t)s_max - (1ll << 62) : -1;   // _next_id (allocator.py:280-281)
  int status = PARVA_OK;

  if (P.relocate) {
    for (int c = 4; c >= 0 && status == PARVA_OK; c--) {
      const int size = size_of_class(c);
      const int64_t L = block_scan(P.n_services, [&](int64_t s) -> int64_t {
        const int oc = P.d_svc_opt[s], lc = P.d_svc_last[s];
        return (oc >= 0 && class_of_size(P.d_cat_size[oc]) == c ? P.d_svc_count[s] : 0) +
               (lc >= 0 && class_of_size(P.d_cat_size[lc]) == c ? 1 : 0);
      }, w.svc_pos, sh);
      if (L == 0) continue;
      const int64_t S = block_scan(G, [&](int64_t g) -> int64_t { return fill_cap(w.mask[g], c); }, w.gpu_pos, sh);
      const int cap_e = fill_cap(0u, c);
      const int64_t rem = L > S ? L - S : 0;
      const int64_t n_new = (rem + cap_e - 1) / cap_e;
      if (G + n_new > w.cap) { status = PARVA_CAPACITY; break; }
      // scatter: thread t owns a contiguous run of queue entries
      const int64_t per = (L + blockDim.x - 1) / blockDim.x;
      const int64_t i0 = tid * per, i1 = min(L, i0 + per);
      if (i0 < i1) {
        int64_t s = upper_bound64(w.svc_pos, P.n_services + 1, i0) - 1;
        int64_t g = i0 < S ? upper_bound64(w.gpu_pos, G + 1, i0) - 1 : -1;
        for (int64_t i = i0; i < i1; i++) {
          while (w.svc_pos[s + 1] <= i) s++;
          const int oc = P.d_svc_opt[s];
          const int64_t r = i - w.svc_pos[s];
          const bool is_opt = oc >= 0 && class_of_size(P.d_cat_size[oc]) == c && r < P.d_svc_count[s];
          const int cat = is_opt ? oc : P.d_svc_last[s];
          if (i < S) {
            while (w.gpu_pos[g + 1] <= i) g++;
            const int j = (int)(i - w.gpu_pos[g]);
            w.lcat[g * 7 + w.len[g] + j] = cat;
            w.lslot[g * 7 + w.len[g] + j] = (uint8_t)fill_start(w.mask[g], c, j);
          } else {
            const int64_t k = i - S, gn = G + k / cap_e;
            const int j = (int)(k % cap_e);
            w.lcat[gn * 7 + j] = cat;
            w.lslot[gn * 7 + j] = (uint8_t)fill_start(0u, c, j);
          }
        }
      }
      __syncthreads();
      for (int64_t g = tid; g < G; g += blockDim.x) {
        const int64_t got = L - w.gpu_pos[g];
        const int capg = (int)(w.gpu_pos[g + 1] - w.gpu_pos[g]);
        const int used = got <= 0 ? 0 : (got < capg ? (int)got : capg);
        if (used) {
          w.mask[g] = (uint8_t)fill_mask(w.mask[g], c, used);
          w.len[g] += (uint8_t)used;
          w.ngpc[g] += (uint8_t)(used * size);
        }
      }
      for (int64_t k = tid; k < n_new; k += blockDim.x) {
        const int64_t g = G + k;
        const int used = (int)min((int64_t)cap_e, rem - k * cap_e);
        w.id[g] = max_id + 1 + k;
        w.mask[g] = (uint8_t)fill_mask(0u, c, used);
        w.len[g] = (uint8_t)used;
        w.ngpc[g] = (uint8_t)(used * size);
      }
      G += n_new;
      max_id += n_new;
      __syncthreads();
    }
  }
  if (tid == 0) {
    w.hdr[0] = G;
    w.hdr[1] = max_id;
    w.hdr[2] = status;
    w.hdr[3] = s_next;
  }
}

__device__ inline double unalloc_g(int64_t total, int64_t n) {
  if (n == 0) return 0.0;
  return __dsub_rn(1.0, __ddiv_rn((double)total, (double)(7 * n)));
}

__global__ void __launch_bounds__(1024) plan_general_kernel(parva_general_problem P, parva_general_result R,
                                                             uint8_t* ws_base, int64_t cap, int64_t qcap) {
  GenWs wsh;
  gen_layout(cap, qcap, P.n_services, ws_base, &wsh);
  const int64_t G0 = wsh.hdr[0];
  // accepts-bitmaps and the optimize-input backup, in parallel
  for (int64_t k = threadIdx.x; k < (G0 + 63) / 64; k += blockDim.x) {
    uint64_t b[5] = {0, 0, 0, 0, 0};
    for (int j = 0; j < 64 && k * 64 + j < G0; j++) {
      const uint32_t m = wsh.mask[k * 64 + j];
#pragma unroll
      for (int c = 0; c < 5; c++) if (find_start(m, c) >= 0) b[c] |= 1ull << j;
    }
#pragma unroll
    for (int c = 0; c < 5; c++) wsh.acc[c * wsh.words + k] = b[c];
  }
  if (P.optimize && wsh.hdr[2] == PARVA_OK)
    for (int64_t g = threadIdx.x; g < G0; g += blockDim.x) {
      wsh.b_id[g] = wsh.id[g]; wsh.b_mask[g] = wsh.mask[g]; wsh.b_len[g] = wsh.len[g]; wsh.b_ngpc[g] = wsh.ngpc[g];
      for (int k = 0; k < wsh.len[g]; k++) { wsh.b_lcat[g * 7 + k] = wsh.lcat[g * 7 + k]; wsh.b_lslot[g * 7 + k] = wsh.lslot[g * 7 + k]; }
    }
  __syncthreads();
  if (threadIdx.x != 0) return;
  Gen S{P, wsh, G0, wsh.hdr[1], {0, 0, 0, 0, 0}};
  GenWs& w = S.w;
  int status = (int)w.hdr[2];
  int32_t next = (int32_t)w.hdr[3];
  const int64_t n_before = S.G;
  int64_t total_before = 0;
  for (int64_t g = 0; g < S.G; g++) total_before += w.ngpc[g];
  R.d_counts[3] = (int32_t)n_before;
  int fallback = 0;
  int64_t nd = 0;

  if (status == PARVA_OK && P.optimize) {
    // ---- optimize_allocation (allocator.py:362-443)
    for (int64_t index = S.G - 1; index >= 0; index--) {
      const int nl = w.len[index];
      if (nl == 0 || (int)w.ngpc[index] > P.threshold) continue;
      int32_t lg_name[7];
      double lg_val[7];
      int32_t lg_ord[7];
      int nlog = 0;
      const int32_t sv_next = next;
      int64_t q2n = 0, q1n = 0;
      int fail = -1, rot = nl;
      int64_t fname = -1;
      bool qover = false;
      for (int k = 0; k < nl; k++) {
        const int cat = w.lcat[index * 7 + k];
        const int name = P.d_cat_name[cat];
        const int s = name < P.n_services ? name : -1;   // services_by_id.get
        if (s < 0) { fail = PARVA_DIAG_UNKNOWN_SERVICE; fname = name; rot = k; break; }
        lg_name[nlog] = s; lg_val[nlog] = R.d_ledger_val[s]; lg_ord[nlog] = R.d_ledger_order[s]; nlog++;
        const double tpp = P.d_cat_tp[cat];
        if (R.d_ledger_order[s] == 0) { R.d_ledger_order[s] = ++next; R.d_ledger_val[s] = __dadd_rn(0.0, tpp); }
        else R.d_ledger_val[s] = __dadd_rn(R.d_ledger_val[s], tpp);
        const int c1 = P.d_svc_t1[s], c2 = P.d_svc_t2[s];
        const double t1 = c1 >= 0 ? P.d_cat_tp[c1] : 0.0, t2 = c2 >= 0 ? P.d_cat_tp[c2] : 0.0;
        long long k2, k1;
        if (!propose_small(t1, t2, R.d_ledger_val[s], k2, k1)) {
          fail = PARVA_DIAG_SMALL_UNAVAILABLE; fname = s; rot = k + 1; break;
        }
        double v = R.d_ledger_val[s];
        for (long long j = 0; j < k2; j++) v = __dsub_rn(v, t2);
        for (long long j = 0; j < k1; j++) v = __dsub_rn(v, t1);
        R.d_ledger_val[s] = v;
        if (qover || q2n + k2 > w.qcap || q1n + k1 > w.qcap) qover = true;
        else {
          for (long long j = 0; j < k2; j++) w.q[q2n++] = c2;
          for (long long j = 0; j < k1; j++) w.q1[q1n++] = c1;
        }
      }
      if (fail < 0) {
        if (qover) fail = PARVA_DIAG_NEED_NEW_GPU;
        else {
          int64_t nu = 0;
          for (int64_t j = 0; j < q2n + q1n; j++) {
            const int cat = j < q2n ? w.q[j] : w.q1[j - q2n];
            const int64_t g = S.place(cat, index, false);
            if (g < 0) { fail = PARVA_DIAG_NEED_NEW_GPU; break; }
            w.undo[nu++] = (int32_t)g;
          }
          if (fail >= 0)
            for (int64_t j = nu - 1; j >= 0; j--) S.pop(w.undo[j]);
        }
      }
      if (fail >= 0) {
        if (rot != nl) {   // allocator.py:415-417: removed ones re-appended
          int32_t tc[7];
          uint8_t ts[7];
          for (int k = 0; k < nl; k++) { tc[k] = w.lcat[index * 7 + k]; ts[k] = w.lslot[index * 7 + k]; }
          for (int k = 0; k < nl; k++) {
            const int src = (k + rot) % nl;
            w.lcat[index * 7 + k] = tc[src];
            w.lslot[index * 7 + k] = ts[src];
          }
        }
        for (int k = nlog - 1; k >= 0; k--) {
          R.d_ledger_val[lg_name[k]] = lg_val[k];
          R.d_ledger_order[lg_name[k]] = lg_ord[k];
        }
        next = sv_next;
        if (nd < R.diag_cap) {
          R.d_diag[3 * nd] = fail;
          R.d_diag[3 * nd + 1] = w.id[index];
          R.d_diag[3 * nd + 2] = fname;
        }
        nd++;
      } else {
        w.len[index] = 0; w.mask[index] = 0; w.ngpc[index] = 0;
        S.set_acc(index);
      }
    }
    int64_t n_after = 0, total_after = 0;
    for (int64_t g = 0; g < S.G; g++) if (w.len[g]) { n_after++; total_after += w.ngpc[g]; }
    if (n_after > n_before ||
        unalloc_g(total_after, n_after) > __dadd_rn(unalloc_g(total_before, n_before), 1e-12)) {
      fallback = 1;
      for (int64_t g = 0; g < S.G; g++) {
        w.id[g] = w.b_id[g]; w.mask[g] = w.b_mask[g]; w.len[g] = w.b_len[g]; w.ngpc[g] = w.b_ngpc[g];
        for (int k = 0; k < w.len[g]; k++) { w.lcat[g * 7 + k] = w.b_lcat[g * 7 + k]; w.lslot[g * 7 + k] = w.b_lslot[g * 7 + k]; }
      }
      for (int k = 0; k < P.n_names; k++) { R.d_ledger_val[k] = P.d_ledger_val[k]; R.d_ledger_order[k] = P.d_ledger_order[k]; }
      nd = 1;
      if (R.diag_cap >= 1) { R.d_diag[0] = PARVA_DIAG_REGRESSED; R.d_diag[1] = -1; R.d_diag[2] = -1; }
    }
  }

  // ---- emit (compaction drops empty GPUs, ids kept; the fallback map is the
  // optimize input as is)
  int64_t ng = 0, np = 0;
  if (status == PARVA_OK) {
    const bool compact = P.optimize && !fallback;
    for (int64_t g = 0; g < S.G; g++) {
      if (compact && w.len[g] == 0) continue;
      if (ng >= R.gpu_cap || np + w.len[g] > R.place_cap) { status = PARVA_CAPACITY; break; }
      R.d_gpu_id[ng] = w.id[g];
      R.d_pl_off[ng] = (int32_t)np;
      for (int k = 0; k < w.len[g]; k++, np++) {
        R.d_pl_cat[np] = w.lcat[g * 7 + k];
        R.d_pl_slot[np] = w.lslot[g * 7 + k];
      }
      ng++;
    }
    R.d_pl_off[ng] = (int32_t)np;
    if (nd > R.diag_cap) status = PARVA_CAPACITY;
  }
  // ---- coverage assert (allocator.py:437-442), service_throughput in map order
  if (status == PARVA_OK && P.optimize && !fallback) {
    for (int s = 0; s < P.n_services; s++) { w.after[s] = 0.0; w.seen[s] = 0; }
    for (int64_t k = 0; k < np; k++) {
      const int name = P.d_cat_name[R.d_pl_cat[k]];
      if (name < P.n_services) { w.after[name] = __dadd_rn(w.after[name], P.d_cat_tp[R.d_pl_cat[k]]); w.seen[name] = 1; }
    }
    for (int s = 0; s < P.n_services; s++)
      if (P.d_svc_rate[s] > 0.0 && w.seen[s] && !(w.after[s] >= __dmul_rn(P.d_svc_rate[s], 1.0 - 1e-9)))
        status = PARVA_COVERAGE_ASSERT;
  }
  R.d_counts[0] = (int32_t)ng;
  R.d_counts[1] = (int32_t)np;
  R.d_counts[2] = (int32_t)nd;
  *R.d_fallback = fallback;
  *R.d_status = status;
}

size_t general_workspace(const parva_general_problem* p, int64_t cap) {
  return gen_layout(cap, cap * 7 + 8, p->n_services, nullptr, nullptr);
}

int launch_plan_general(const parva_general_problem* p, parva_general_result* r, void* ws, size_t ws_bytes,
                        cudaStream_t stream) {
  const int64_t cap = r->gpu_cap;
  if (general_workspace(p, cap) > ws_bytes) return PARVA_BAD_INPUT;
  gen_prepare_kernel<<<1, 1024, 0, stream>>>(*p, *r, (uint8_t*)ws, cap, cap * 7 + 8);
  plan_general_kernel<<<1, 1024, 0, stream>>>(*p, *r, (uint8_t*)ws, cap, cap * 7 + 8);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva
