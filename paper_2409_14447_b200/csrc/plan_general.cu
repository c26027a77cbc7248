// plan_general.cu — KG: relocate_segments / optimize_allocation on an
// arbitrary problem (any number of services and GPUs, arbitrary input
// DeploymentMap, GPU ids and ledger).  Used for the object API
// (relocate_segments, optimize_allocation) and for scenarios that overflow
// the fast path's 128-byte record (PARVA_CAPACITY).
//
// Relocation runs as parallel per-size-class phases (gen_prepare_kernel).  The
// optimize pass is a serial dependency chain walked by one
// warp; first-fit is an "accepts" bitmap search from a lazily advanced
// start word instead of the reference's O(M) scans and O(M) _next_id
// (allocator.py:204-281), which is what makes the 10^5-segment case (C5)
// cheap.  Ledger rollback uses an undo log instead of the reference's
// whole-dict snapshot (allocator.py:387,418-419): same observable ledger,
// O(touched) instead of O(services) per GPU.
#include <cuda_runtime.h>
#ifdef PARVA_KG_PROF
#include <cstdio>
#endif

#include "parva_common.cuh"
#include "parva_kernels.cuh"

namespace parva {

// Flattened catalogue entry: everything a drain needs about a placement kind
// in one 40-byte load (tp, the owning service's size-1/2 kinds and their tps).
struct CatExt {
  double tp, tp1, tp2;
  int32_t name, c1, c2, pad;
};

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
  int64_t* gpu_pos2;// [cap + 1] second scan buffer
  int64_t* hdr;     // [8]: G, max_id, status, next (ledger rank counter)
  CatExt* ext;      // [n_cat]
  int64_t words, qcap, cap;
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline size_t gen_layout(int64_t cap, int64_t qcap, int n_services, int n_cat, uint8_t* base,
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
  t.gpu_pos2 = (int64_t*)take((size_t)(cap + 2) * 8);
  t.hdr = (int64_t*)take(8 * 8);
  t.ext = (CatExt*)take((size_t)(n_cat + 1) * sizeof(CatExt));
  t.words = words; t.qcap = qcap; t.cap = cap;
  if (w) *w = t;
  return off;
}


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
// 8-bit GPU state: bits 0-6 occupied-or-blocked slots, bit 7 = a size-3
// segment sits at slot 0 (its blocked slot 3 is not a GPC), so
// num_gpcs = popc(bits 0-6) - bit 7.
constexpr uint32_t kFlag30 = 0x80u;
__device__ __forceinline__ uint32_t fill_mask8(uint32_t m8, int c, int used) {
  uint32_t m = m8 & 0x7Fu, f = m8 & kFlag30;
  for (int k = 0; k < used; k++) {
    const int st = find_start(m, c);
    m |= footprint(c, st);
    if (c == 2 && st == 0) f = kFlag30;
  }
  return m | f;
}
__device__ __forceinline__ int gpcs8(uint32_t m8) { return __popc(m8 & 0x7Fu) - (int)(m8 >> 7); }

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
  gen_layout(cap, qcap, P.n_services, P.n_cat, ws_base, &w);
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
      m |= footprint(c, P.d_pl_slot[k]) | (c == 2 && P.d_pl_slot[k] == 0 ? kFlag30 : 0u);
      ng += size_of_class(c);
      w.lcat[g * 7 + n] = cat;
      w.lslot[g * 7 + n] = P.d_pl_slot[k];
    }
    w.mask[g] = (uint8_t)m; w.len[g] = (uint8_t)n; w.ngpc[g] = (uint8_t)ng;
  }
  for (int k = tid; k < P.n_cat; k += blockDim.x) {
    CatExt e;
    e.tp = P.d_cat_tp[k];
    e.name = P.d_cat_name[k];
    const int sv = e.name < P.n_services ? e.name : -1;
    e.c1 = sv >= 0 ? P.d_svc_t1[sv] : -1;
    e.c2 = sv >= 0 ? P.d_svc_t2[sv] : -1;
    e.tp1 = e.c1 >= 0 ? P.d_cat_tp[e.c1] : 0.0;
    e.tp2 = e.c2 >= 0 ? P.d_cat_tp[e.c2] : 0.0;
    e.pad = 0;
    w.ext[k] = e;
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
      const int64_t S = block_scan(G, [&](int64_t g) -> int64_t { return fill_cap(w.mask[g] & 0x7Fu, c); }, w.gpu_pos, sh);
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
            w.lslot[g * 7 + w.len[g] + j] = (uint8_t)fill_start(w.mask[g] & 0x7Fu, c, j);
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
          w.mask[g] = (uint8_t)fill_mask8(w.mask[g], c, used);
          w.len[g] += (uint8_t)used;
          w.ngpc[g] += (uint8_t)(used * size);
        }
      }
      for (int64_t k = tid; k < n_new; k += blockDim.x) {
        const int64_t g = G + k;
        const int used = (int)min((int64_t)cap_e, rem - k * cap_e);
        w.id[g] = max_id + 1 + k;
        w.mask[g] = (uint8_t)fill_mask8(0u, c, used);
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

// Optimize (allocator.py:362-443) as a serial chain walked by warp 0 in
// lock step: every lane executes the same scalar chain on the same values
// (shared-memory reads are broadcasts, same-address stores coalesce), so the
// chain needs no shuffles and no divergence; a __syncwarp separates every
// read of shared state from the lanes' identical writes of it (the chain
// does not rely on lock-step execution: compute-sanitizer racecheck clean);
// the warp's lanes only split the loads of a drained list and the proposal
// search (propose_small_warp).  GPU state (8-bit mask + list length) and the
// accepts bitmaps of size classes 1 and 2 -- the only sizes a proposal has
// -- sit in shared memory when they fit (~110k GPUs), else in global memory.
// The next drain candidate (0 < num_gpcs <= threshold) is found 8 GPUs per
// load (SWAR per-byte popcount); first fit is the first nonzero accepts word
// at or after a per-class start word that moves past zero words once and
// back only when a GPU below it starts accepting (cursor-free first fit,
// same choice as a scan from GPU 0); undo entries carry (gpu, class, slot) so a rollback
// reads no lists; the freed_rate ledger rolls back from a log.
constexpr int OPT_THREADS = 512;
constexpr int kChainUndo = 256;   // undo entries kept in shared memory (the rest in w.undo)

struct OptState {
  uint8_t* M;        // mask | flag, per GPU
  uint8_t* Ln;       // list length, per GPU
  uint64_t* A;       // accepts bitmaps [2][words] (size classes 0, 1)
  int64_t words, G;
  int64_t lw[2];     // accepts words below lw[c] are zero (first-fit starts there)

  // GPU g's byte is now m: its accepts bits and the start words
  __device__ __forceinline__ void set_bits(int64_t g, uint32_t m) {
    m &= 0x7Fu;
    const int64_t k = g >> 6;
    const uint64_t bit = 1ull << (g & 63);
    const bool acc0 = m != 0x7Fu;                                                     // find_start(m, 0) >= 0
    const bool acc1 = (m & 0x03u) == 0 || (m & 0x0Cu) == 0 || (m & 0x30u) == 0;        // find_start(m, 1) >= 0
    const uint64_t a0 = A[k], a1 = A[words + k];
    __syncwarp();   // every lane has read the words before any lane writes them
    A[k] = acc0 ? (a0 | bit) : (a0 & ~bit);
    A[words + k] = acc1 ? (a1 | bit) : (a1 & ~bit);
    if (acc0 && k < lw[0]) lw[0] = k;
    if (acc1 && k < lw[1]) lw[1] = k;
    __syncwarp();   // the lanes wrote the same words: ordered before any lane reads them again
  }

  // first GPU in list order accepting class c (0 or 1), skipping `excl`:
  // the first nonzero accepts word at or after lw[c] (zero words are passed
  // once: lw only moves back when a GPU below it starts accepting)
  __device__ __forceinline__ int64_t first_fit(int c, int64_t excl) {
    const uint64_t* a = A + c * words;
    const int64_t ew = excl >> 6;
    const uint64_t ebit = 1ull << (excl & 63);
    for (int64_t k = lw[c]; k < words; k++) {
      const uint64_t word = a[k];
      const uint64_t v = k == ew ? word & ~ebit : word;
      if (v) return k * 64 + __ffsll((long long)v) - 1;
      if (!word && k == lw[c]) lw[c] = k + 1;
    }
    return -1;
  }

  // highest GPU <= idx with 0 < num_gpcs <= thr: 8 GPUs per load, tested
  // at once (per-byte popcount of the 7 slot bits minus the size-3@0 flag)
  __device__ __forceinline__ int64_t prev_candidate(int64_t idx, int thr) const {
    if (thr <= 0 || idx < 0) return -1;
    const uint64_t lo7 = 0x7F7F7F7F7F7F7F7Full, b1 = 0x0101010101010101ull;
    const uint64_t up = thr >= 7 ? 0ull : (uint64_t)(0x80 - thr - 1) * b1;   // + up sets bit 7 iff gpcs > thr
    uint64_t keep = (idx & 7) == 7 ? ~0ull : (1ull << (8 * ((idx & 7) + 1))) - 1;   // bytes <= idx
    for (int64_t w8 = idx >> 3; w8 >= 0; w8--, keep = ~0ull) {
      const uint64_t x = reinterpret_cast<const uint64_t*>(M)[w8];
      uint64_t v = x & lo7;
      v = v - ((v >> 1) & 0x5555555555555555ull);
      v = (v & 0x3333333333333333ull) + ((v >> 2) & 0x3333333333333333ull);
      v = (v + (v >> 4)) & 0x0F0F0F0F0F0F0F0Full;
      const uint64_t g = v - ((x >> 7) & b1);                   // gpcs per byte, 0..7 (the flag implies >= 4 cells)
      const uint64_t hit = (g + lo7) & ~(thr >= 7 ? 0ull : (g + up)) & (b1 << 7) & keep;
      if (hit) return w8 * 8 + ((63 - __clzll((long long)hit)) >> 3);
    }
    return -1;
  }
};

// the drained list and the chain's logs (shared memory, warp 0)
struct ChainSmem {
  CatExt ext[8];
  int32_t cat[8];
  uint8_t slot[8];
  long long k2[8], k1[8];
  int32_t lg_name[8], lg_ord[8];
  double lg_val[8];
  double lv[8];      // staged ledger entries of the drained services (lane k: entry k)
  int32_t lo[8];
  int32_t undo[kChainUndo];
};

// kSmem: GPU state and bitmaps in shared memory (dsm), so the
// compiler emits shared-memory accesses instead of generic ones
template <bool kSmem>
__device__ __forceinline__ int64_t opt_chain(const parva_general_problem& P, const parva_general_result& R,
                                             const GenWs& w, int64_t G0, int lane, ChainSmem& C, uint8_t* dsm) {
  OptState S;
  const int64_t gpad = (G0 + 15) & ~int64_t(15);
  S.words = (G0 + 63) / 64;
  S.G = G0;
  S.M = kSmem ? dsm : w.mask;
  S.Ln = kSmem ? dsm + gpad : w.len;
  S.A = kSmem ? reinterpret_cast<uint64_t*>(dsm + 2 * gpad) : w.acc;
  S.lw[0] = S.lw[1] = 0;
  int32_t next = (int32_t)w.hdr[3];
  int64_t nd = 0;
  int64_t idx = G0 - 1;
#ifdef PARVA_KG_PROF   // phase cycle counters of the serial chain (probe builds only)
  long long kp[6] = {0, 0, 0, 0, 0, 0}, kn_drain = 0, kn_place = 0, kt = clock64();
#define KG_MARK(i) do { const long long c_ = clock64(); kp[i] += c_ - kt; kt = c_; } while (0)
#else
#define KG_MARK(i) do { } while (0)
#endif
  while (true) {
    const int64_t index = S.prev_candidate(idx, P.threshold);
    if (index < 0) break;
    KG_MARK(0);
    idx = index - 1;
    const int nl = S.Ln[index];
    if (lane < nl) {            // lane k stages entry k of the drained list
      const int cat = w.lcat[index * 7 + lane];
      C.cat[lane] = cat;
      C.slot[lane] = w.lslot[index * 7 + lane];
      const CatExt X = w.ext[cat];
      C.ext[lane] = X;
      if (X.name < P.n_services) {   // the ledger entries, loaded in parallel
        C.lv[lane] = R.d_ledger_val[X.name];
        C.lo[lane] = R.d_ledger_order[X.name];
      }
    }
    __syncwarp();
    KG_MARK(1);
    const int32_t sv_next = next;
    int fail = -1, rot = nl, nlog = 0;
    int64_t fname = -1;
    for (int k = 0; k < nl; k++) {   // allocator.py:392-405, in order
      const CatExt X = C.ext[k];
      if (X.name >= P.n_services) { fail = PARVA_DIAG_UNKNOWN_SERVICE; fname = X.name; rot = k; break; }
      const int s = X.name;
      const double ov = C.lv[k];
      const int32_t oo = C.lo[k];
      const double f = oo == 0 ? __dadd_rn(0.0, X.tp) : __dadd_rn(ov, X.tp);
      const int32_t no = oo == 0 ? ++next : oo;
      if (oo == 0) R.d_ledger_order[s] = no;
      R.d_ledger_val[s] = f;
      C.lg_name[k] = s; C.lg_val[k] = ov; C.lg_ord[k] = oo;
      nlog = k + 1;
      long long k2, k1;
      if (!propose_small_warp(X.tp1, X.tp2, f, k2, k1, lane)) {
        fail = PARVA_DIAG_SMALL_UNAVAILABLE; fname = s; rot = k + 1; break;
      }
      double v = f;
      for (long long j = 0; j < k2; j++) v = __dsub_rn(v, X.tp2);
      for (long long j = 0; j < k1; j++) v = __dsub_rn(v, X.tp1);
      R.d_ledger_val[s] = v;
      C.k2[k] = k2; C.k1[k] = k1;
      for (int j = k + 1; j < nl; j++)   // a later entry of the same service sees this update
        if (C.ext[j].name == s) { C.lv[j] = v; C.lo[j] = no; }
      __syncwarp();
    }
    KG_MARK(2);
    int64_t nu = 0;
    if (fail < 0) {
      long long tot = 0;
      for (int k = 0; k < nl; k++) tot += C.k2[k] + C.k1[k];
      if (tot > w.qcap) fail = PARVA_DIAG_NEED_NEW_GPU;   // more GPCs than any map can free
      else {
        // proposals queue (allocator.py:403-405, drained by size): every size-2
        // kind in drain order, then every size-1 kind; first fit without new GPUs
        for (int c = 1; c >= 0 && fail < 0; c--) {
          for (int k = 0; k < nl && fail < 0; k++) {
            const long long cnt = c ? C.k2[k] : C.k1[k];
            const int cat = c ? C.ext[k].c2 : C.ext[k].c1;
            for (long long r = 0; r < cnt; r++) {
              KG_MARK(3);
              const int64_t g = S.first_fit(c, index);
              KG_MARK(5);
              if (g < 0) { fail = PARVA_DIAG_NEED_NEW_GPU; break; }
              const uint32_t m8 = S.M[g];
              const int st = find_start(m8 & 0x7Fu, c);
              const int ln = S.Ln[g];
              const uint32_t nm = m8 | footprint(c, st);
              __syncwarp();             // every lane has read the GPU's state before any lane updates it
              S.M[g] = (uint8_t)nm;
              S.Ln[g] = (uint8_t)(ln + 1);
              w.lcat[g * 7 + ln] = cat;
              w.lslot[g * 7 + ln] = (uint8_t)st;
              const int32_t u = (int32_t)(g << 4 | c << 3 | st);   // g < 2^27
              if (nu < kChainUndo) C.undo[nu] = u; else w.undo[nu] = u;
              nu++;
              __syncwarp();
              S.set_bits(g, nm);
            }
          }
        }
        if (fail >= 0) {  // all-or-nothing undo (allocator.py:272-277)
          for (int64_t j = nu - 1; j >= 0; j--) {
            const int32_t u = j < kChainUndo ? C.undo[j] : w.undo[j];
            const int64_t g = u >> 4;
            const int c = (u >> 3) & 1, st = u & 7;
            const uint32_t nm = S.M[g] & ~footprint(c, st);
            const int ln = S.Ln[g];
            __syncwarp();
            S.M[g] = (uint8_t)nm;
            S.Ln[g] = (uint8_t)(ln - 1);
            S.set_bits(g, nm);
          }
        }
      }
    }
    KG_MARK(3);
#ifdef PARVA_KG_PROF
    kn_drain++; kn_place += nu;
#endif
    if (fail >= 0) {
      if (rot != nl && lane < nl) {   // allocator.py:415-417: the removed ones are re-appended
        int src = lane + rot;
        if (src >= nl) src -= nl;
        w.lcat[index * 7 + lane] = C.cat[src];
        w.lslot[index * 7 + lane] = C.slot[src];
      }
      __syncwarp();                 // (the loop above may have left before its barrier)
      for (int k = nlog - 1; k >= 0; k--) {   // ledger rollback in reverse log order
        R.d_ledger_val[C.lg_name[k]] = C.lg_val[k];
        R.d_ledger_order[C.lg_name[k]] = C.lg_ord[k];
      }
      next = sv_next;
      if (nd < R.diag_cap) {
        R.d_diag[3 * nd] = fail;
        R.d_diag[3 * nd + 1] = w.id[index];
        R.d_diag[3 * nd + 2] = fname;
      }
      nd++;
    } else {
      S.M[index] = 0;
      S.Ln[index] = 0;
      S.set_bits(index, 0u);
    }
    __syncwarp();                 // C is restaged by the next drain
    KG_MARK(4);
  }
#ifdef PARVA_KG_PROF
  if (lane == 0)
    printf("KGPROF drains %lld placements %lld cycles: search %lld lists %lld ledger+propose %lld place %lld "
           "finish %lld (first_fit %lld)\n", kn_drain, kn_place, kp[0], kp[1], kp[2], kp[3], kp[4], kp[5]);
#endif
#undef KG_MARK
  return nd;
}

__global__ void __launch_bounds__(OPT_THREADS) plan_general_kernel(parva_general_problem P, parva_general_result R,
                                                                   uint8_t* ws_base, int64_t cap, int64_t qcap,
                                                                   int64_t smem_gpus) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ int64_t sh[33];
  __shared__ int s_fallback, s_status;
  __shared__ int64_t s_nd;
  __shared__ ChainSmem chain;
  GenWs w;
  gen_layout(cap, qcap, P.n_services, P.n_cat, ws_base, &w);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef PARVA_KG_PROF
  const long long kt0 = clock64();
#endif
  const int64_t G0 = w.hdr[0];
  int status = (int)w.hdr[2];
  const bool in_smem = G0 <= smem_gpus;
  const int64_t words = (G0 + 63) / 64;
  const int64_t gpad = (G0 + 15) & ~int64_t(15);
  OptState S;
  S.M = in_smem ? dsm : w.mask;
  S.Ln = in_smem ? dsm + gpad : w.len;
  S.A = in_smem ? reinterpret_cast<uint64_t*>(dsm + 2 * gpad) : w.acc;
  S.words = words;
  S.G = G0;
  S.lw[0] = S.lw[1] = 0;
  if (in_smem)
    for (int64_t g = tid; g < G0; g += blockDim.x) { S.M[g] = w.mask[g]; S.Ln[g] = w.len[g]; }
  __syncthreads();
  for (int64_t k = tid; k < words; k += blockDim.x) {
    uint64_t b[2] = {0, 0};
    for (int j = 0; j < 64 && k * 64 + j < G0; j++) {
      const uint32_t m = S.M[k * 64 + j] & 0x7Fu;
#pragma unroll
      for (int c = 0; c < 2; c++) if (find_start(m, c) >= 0) b[c] |= 1ull << j;
    }
#pragma unroll
    for (int c = 0; c < 2; c++) S.A[c * words + k] = b[c];
  }
  const bool run = P.optimize && status == PARVA_OK;
  if (run)
    for (int64_t g = tid; g < G0; g += blockDim.x) {
      w.b_mask[g] = w.mask[g]; w.b_len[g] = w.len[g];
      for (int k = 0; k < w.len[g]; k++) { w.b_lcat[g * 7 + k] = w.lcat[g * 7 + k]; w.b_lslot[g * 7 + k] = w.lslot[g * 7 + k]; }
    }
  if (tid == 0) { s_fallback = 0; s_status = status; s_nd = 0; }
  __syncthreads();

#ifdef PARVA_KG_PROF
  const long long kt1 = clock64();
#endif
  if (run && warp == 0) {
    const int64_t nd = in_smem ? opt_chain<true>(P, R, w, G0, lane, chain, dsm)
                               : opt_chain<false>(P, R, w, G0, lane, chain, dsm);
    if (lane == 0) s_nd = nd;
  }
  __syncthreads();

  // ---- compaction + regression check (allocator.py:423-435), parallel
#ifdef PARVA_KG_PROF
  const long long kt2 = clock64();
#endif
  int64_t nd = s_nd;
  if (run) {
    const int64_t n_after = block_scan(G0, [&](int64_t g) -> int64_t { return S.Ln[g] ? 1 : 0; }, w.gpu_pos, sh);
    const int64_t tot_after = block_scan(G0, [&](int64_t g) -> int64_t { return S.Ln[g] ? gpcs8(S.M[g]) : 0; },
                                         w.gpu_pos2, sh);
    const int64_t tot_before = block_scan(G0, [&](int64_t g) -> int64_t { return gpcs8(w.b_mask[g]); },
                                          w.gpu_pos2, sh);
    const double ua_b = unalloc_g(tot_before, G0), ua_a = unalloc_g(tot_after, n_after);
    if (tid == 0 && (n_after > G0 || ua_a > __dadd_rn(ua_b, 1e-12))) s_fallback = 1;
    __syncthreads();
    if (s_fallback) {
      for (int64_t g = tid; g < G0; g += blockDim.x) {
        S.M[g] = w.b_mask[g]; S.Ln[g] = w.b_len[g];
        for (int k = 0; k < w.b_len[g]; k++) { w.lcat[g * 7 + k] = w.b_lcat[g * 7 + k]; w.lslot[g * 7 + k] = w.b_lslot[g * 7 + k]; }
      }
      for (int k = tid; k < P.n_names; k += blockDim.x) { R.d_ledger_val[k] = P.d_ledger_val[k]; R.d_ledger_order[k] = P.d_ledger_order[k]; }
      nd = 1;
      if (tid == 0 && R.diag_cap >= 1) { R.d_diag[0] = PARVA_DIAG_REGRESSED; R.d_diag[1] = -1; R.d_diag[2] = -1; }
      __syncthreads();
    }
  }
  // ---- emit: GPUs in order (compacted unless fallback / no optimize), lists
  if (status == PARVA_OK) {
    const bool compact = run && !s_fallback;
    const int64_t ng = block_scan(G0, [&](int64_t g) -> int64_t { return !compact || S.Ln[g] ? 1 : 0; }, w.gpu_pos, sh);
    const int64_t np = block_scan(G0, [&](int64_t g) -> int64_t { return !compact || S.Ln[g] ? S.Ln[g] : 0; },
                                  w.gpu_pos2, sh);
    if (ng > R.gpu_cap || np > R.place_cap || nd > R.diag_cap) {
      status = PARVA_CAPACITY;
    } else {
      for (int64_t g = tid; g < G0; g += blockDim.x) {
        if (compact && !S.Ln[g]) continue;
        const int64_t o = w.gpu_pos[g], po = w.gpu_pos2[g];
        R.d_gpu_id[o] = w.id[g];
        R.d_pl_off[o] = (int32_t)po;
        for (int k = 0; k < S.Ln[g]; k++) { R.d_pl_cat[po + k] = w.lcat[g * 7 + k]; R.d_pl_slot[po + k] = w.lslot[g * 7 + k]; }
      }
      if (tid == 0) R.d_pl_off[ng] = (int32_t)np;
    }
    __syncthreads();
    // ---- coverage assert (allocator.py:437-442): service_throughput in map
    // order.  Parallel unordered sums first; any two summation orders of n
    // positive terms differ by at most 2n*2^-53*sum, so only a service within
    // that margin of its threshold is re-summed in map order (never seen).
    if (status == PARVA_OK && compact) {
      for (int s = tid; s < P.n_services; s += blockDim.x) { w.after[s] = 0.0; w.seen[s] = 0; w.svc_pos[s] = 0; }
      __syncthreads();
      for (int64_t k = tid; k < np; k += blockDim.x) {
        const CatExt X = w.ext[R.d_pl_cat[k]];
        if (X.name < P.n_services) {
          atomicAdd(&w.after[X.name], X.tp);
          atomicAdd(reinterpret_cast<unsigned long long*>(&w.svc_pos[X.name]), 1ull);
        }
      }
      __syncthreads();
      for (int s = tid; s < P.n_services; s += blockDim.x) {
        const int64_t cnt = w.svc_pos[s];
        if (!(P.d_svc_rate[s] > 0.0) || cnt == 0) continue;
        const double thr = __dmul_rn(P.d_svc_rate[s], 1.0 - 1e-9);
        const double sum = w.after[s];
        const double err = (double)(2 * cnt + 2) * 1.1102230246251565e-16 * sum;
        bool ok;
        if (sum - err >= thr) ok = true;
        else if (sum + err < thr) ok = false;
        else {   // exact: the reference's left-to-right sum in map order
          double e = 0.0;
          bool first = true;
          for (int64_t k = 0; k < np; k++) {
            const CatExt X = w.ext[R.d_pl_cat[k]];
            if (X.name == s) { e = first ? __dadd_rn(0.0, X.tp) : __dadd_rn(e, X.tp); first = false; }
          }
          ok = e >= thr;
        }
        if (!ok) atomicExch(&s_status, PARVA_COVERAGE_ASSERT);
      }
      __syncthreads();
      if (s_status == PARVA_COVERAGE_ASSERT) status = PARVA_COVERAGE_ASSERT;
    }
    if (tid == 0) { R.d_counts[0] = (int32_t)ng; R.d_counts[1] = (int32_t)np; }
  }
  if (tid == 0) {
    R.d_counts[2] = (int32_t)nd;
    R.d_counts[3] = (int32_t)G0;
    *R.d_fallback = s_fallback;
    *R.d_status = status;
#ifdef PARVA_KG_PROF
    printf("KGPROF kernel cycles: prologue %lld chain %lld epilogue %lld\n", kt1 - kt0, kt2 - kt1, clock64() - kt2);
#endif
  }
}

size_t general_workspace(const parva_general_problem* p, int64_t cap) {
  return gen_layout(cap, cap * 7 + 8, p->n_services, p->n_cat, nullptr, nullptr);
}

int launch_plan_general(const parva_general_problem* p, parva_general_result* r, void* ws, size_t ws_bytes,
                        cudaStream_t stream) {
  const int64_t cap = r->gpu_cap;
  if (general_workspace(p, cap) > ws_bytes) return PARVA_BAD_INPUT;
  gen_prepare_kernel<<<1, 1024, 0, stream>>>(*p, *r, (uint8_t*)ws, cap, cap * 7 + 8);
  // shared-memory state when it fits: 2 B per GPU + 2 bitmap bits per GPU
  static int s_smem[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  int& smem_max = s_smem[dev & (kMaxDevices - 1)];
  if (!smem_max) {
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, plan_general_kernel);
    smem_max -= (int)fa.sharedSizeBytes + 256;   // static shared memory of the kernel
    cudaFuncSetAttribute(plan_general_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
  }
  // largest G with 2 * pad16(G) + 16 * ceil(G / 64) <= smem_max
  int64_t smem_gpus = (int64_t)smem_max * 4 / 9;
  while (smem_gpus > 0 && 2 * ((smem_gpus + 15) & ~int64_t(15)) + 16 * ((smem_gpus + 63) / 64) > smem_max) smem_gpus--;
  const size_t smem = (size_t)smem_max;
  plan_general_kernel<<<1, OPT_THREADS, smem, stream>>>(*p, *r, (uint8_t*)ws, cap, cap * 7 + 8, smem_gpus);
  return cudaGetLastError() == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

}  // namespace parva
