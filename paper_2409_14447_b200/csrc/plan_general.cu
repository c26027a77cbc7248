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

__device__ inline double unalloc_g(int64_t total, int64_t n) {
  if (n == 0) return 0.0;
  return __dsub_rn(1.0, __ddiv_rn((double)total, (double)(7 * n)));
}

__global__ void plan_general_kernel(parva_general_problem P, parva_general_result R, uint8_t* ws_base,
                                    int64_t cap, int64_t qcap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Gen S{P, {}, 0, -1, {0, 0, 0, 0, 0}};
  gen_layout(cap, qcap, P.n_services, ws_base, &S.w);
  GenWs& w = S.w;
  int status = PARVA_OK;

  // ---- initial map
  for (int64_t k = 0; k < 5 * w.words; k++) w.acc[k] = 0;
  S.G = P.n_gpus;
  for (int64_t g = 0; g < P.n_gpus; g++) {
    w.id[g] = P.d_gpu_id[g];
    if (P.d_gpu_id[g] > S.max_id) S.max_id = P.d_gpu_id[g];
    uint32_t m = 0;
    int ng = 0, n = 0;
    for (int k = P.d_pl_off[g]; k < P.d_pl_off[g + 1]; k++, n++) {
      const int cat = P.d_pl_cat[k], c = S.class_of(cat);
      m |= footprint(c, P.d_pl_slot[k]);
      ng += size_of_class(c);
      w.lcat[g * 7 + n] = cat;
      w.lslot[g * 7 + n] = P.d_pl_slot[k];
    }
    w.mask[g] = (uint8_t)m; w.len[g] = (uint8_t)n; w.ngpc[g] = (uint8_t)ng;
    S.set_acc(g);
  }
  for (int c = 0; c < 5; c++) S.hint[c] = 0;
  int32_t next = 0;
  for (int k = 0; k < P.n_names; k++) {
    R.d_ledger_val[k] = P.d_ledger_val[k];
    R.d_ledger_order[k] = P.d_ledger_order[k];
    if (P.d_ledger_order[k] > next) next = P.d_ledger_order[k];
  }

  // ---- relocate_segments (allocator.py:292-316): sizes 7,4,3,2,1; FIFO by service
  if (P.relocate) {
    for (int c = 4; c >= 0 && status == PARVA_OK; c--) {
      for (int s = 0; s < P.n_services && status == PARVA_OK; s++) {
        const int oc = P.d_svc_opt[s], lc = P.d_svc_last[s];
        const long long reps = (oc >= 0 && S.class_of(oc) == c ? P.d_svc_count[s] : 0);
        for (long long r = 0; r < reps; r++)
          if (S.place(oc, -1, true) == -2) { status = PARVA_CAPACITY; break; }
        if (status == PARVA_OK && lc >= 0 && S.class_of(lc) == c)
          if (S.place(lc, -1, true) == -2) status = PARVA_CAPACITY;
      }
    }
  }
  const int64_t n_before = S.G;
  int64_t total_before = 0;
  for (int64_t g = 0; g < S.G; g++) total_before += w.ngpc[g];
  R.d_counts[3] = (int32_t)n_before;
  int fallback = 0;
  int64_t nd = 0;

  if (status == PARVA_OK && P.optimize) {
    for (int64_t g = 0; g < S.G; g++) {
      w.b_id[g] = w.id[g]; w.b_mask[g] = w.mask[g]; w.b_len[g] = w.len[g]; w.b_ngpc[g] = w.ngpc[g];
      for (int k = 0; k < w.len[g]; k++) { w.b_lcat[g * 7 + k] = w.lcat[g * 7 + k]; w.b_lslot[g * 7 + k] = w.lslot[g * 7 + k]; }
    }
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
  plan_general_kernel<<<1, 32, 0, stream>>>(*p, *r, (uint8_t*)ws, cap, cap * 7 + 8);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva
