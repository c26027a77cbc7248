// plan_thread.cuh — K2, thread-per-scenario form (included by plan_batch.cu).
//
// The same fused plan as the tile kernel -- configure_service for every
// service (configurator.py:189-191), relocate_segments (allocator.py:292-316)
// and optimize_allocation (allocator.py:362-443) per scenario -- with one
// THREAD per scenario instead of a lane group: the per-scenario allocator is
// a sequential chain, so a warp keeps 32 scenarios in flight with no
// collectives and no block barriers.  A warp owns 32 consecutive scenarios
// (a chunk):
//   * configure: the warp's lanes configure the chunk's services lane-
//     strided (coalesced inputs, config records stored as the tile kernel
//     stores them) through the prefix-argmax index read via L1; per service
//     the planner keeps a 4-byte meta word and the five best point positions
//     in shared memory;
//   * plan: thread j plans scenario k0 + j.  GPU state lives in registers:
//     one byte per GPU (7 slot bits + a size-3-at-slot-0 flag, so the GPC
//     count is popc - flag) packed into two u64 words, placement counts as
//     4-bit fields of a third; first-fit is a cursor over those bytes (cursor-
//     free first-fit).  Placements are a log in shared
//     memory (thread-minor): a GPU's list is its entries in log order, a
//     drained GPU's placements leave the log, a failed drain re-appends the
//     ones already removed (allocator.py:415-417).  A drain's ledger updates
//     are kept in registers and committed only when the drain succeeds, so a
//     failed drain needs no snapshot.
//   * emit: records are built in shared memory, then copied out by the warp
//     (coalesced).
// A scenario beyond the thread path's limits (more than kThS services, kThG
// GPUs, kThL placements, or services past the chunk's staging area) is
// re-planned by the whole warp with the warp planner (plan_scenario_warp<32>),
// whose own limits are the record's.

#ifndef PARVA_TH_WARPS
#define PARVA_TH_WARPS 1
#endif
#ifndef PARVA_TH_MINB
#define PARVA_TH_MINB 16
#endif
constexpr int TH_WARPS = PARVA_TH_WARPS;
constexpr int TH_THREADS = TH_WARPS * 32;
constexpr int kThS = 16;        // services per scenario on the thread path
constexpr int kThG = 16;        // GPUs
constexpr int kThL = 32;        // placement log entries
constexpr int kThSvc = 384;     // staged services per chunk (32 scenarios x 12)
constexpr int kThRow = 33;
constexpr int64_t kThPrefetch = 64 << 10;   // index bytes prefetched into L1 at kernel start      // staged record row, words (128-B record + pad: conflict-free)

struct alignas(16) ThWarp {
  union {
    struct {
      uint32_t meta[kThSvc];              // count (sat. 255) | opt << 8 | last << 12 | status << 16 (15 = none)
      uint16_t best[kThSvc][6];           // best point position per size class (0xFFFF = absent), table id
    } svc;
    uint32_t stage[32][kThRow];           // records being emitted
    struct {
      GScratch<32> g;
      GSvc<32> s;
    } w;                                  // warp planner of the deferred scenarios
  } u;
  uint16_t log[kThL][32];                 // placements: gpu << 11 | (service * 5 + class) << 3 | slot
};

// Per-thread ledger and diagnostics: touched only by drains and emission, so
// they live in (L1-cached) local memory rather than in the shared memory
// that bounds the warps per SM
struct ThLedger {
  double freed[kThS];                     // freed_rate ledger (allocator.py:396-404)
  uint8_t order[kThS];                    // ledger insertion rank, 0 = absent
  uint16_t diag[kThG];                    // optimize diagnostics
};

// GPU state of one scenario, in registers
struct ThGpus {
  uint64_t lo, hi;   // GPU g's byte: bits 0-6 occupied-or-blocked slots, bit 7 = size 3 at slot 0
  uint64_t len;      // placements per GPU, 4 bits each
  uint64_t acc;      // bit 16 c + g: GPU g accepts a segment of size class c (c = 0..3)
  uint32_t acc4;     // bit g: GPU g is empty (accepts size 7)
};

__device__ __forceinline__ uint32_t th_byte(const ThGpus& G, int g) {
  return (uint32_t)((g < 8 ? G.lo : G.hi) >> ((g & 7) << 3)) & 0xFFu;
}
__device__ __forceinline__ int th_len(const ThGpus& G, int g) { return (int)(G.len >> (4 * g)) & 15; }
__device__ __forceinline__ int th_gpc(uint32_t b) { return __popc(b & 0x7Fu) - (int)(b >> 7); }
// GPUs (bit g) that accept size class c (cursor-free first-fit = lowest bit;
// GPUs past the map are empty and accept anything)
__device__ __forceinline__ uint32_t th_acc(const ThGpus& G, int c) {
  return c == 4 ? G.acc4 : (uint32_t)(G.acc >> (16 * c)) & 0xFFFFu;
}
constexpr uint64_t kThSpread = 0x0001000100010001ull;
__device__ __forceinline__ void th_init(ThGpus& G) {
  G.lo = G.hi = G.len = 0;
  G.acc = ~0ull;
  G.acc4 = 0xFFFFu;
}
// GPU g's byte changed to b: its acceptance bits from the table (bit c of
// tbl[b & 0x7F] = find_start(b, c) >= 0, mig.py:114-122)
__device__ __forceinline__ void th_set_acc(ThGpus& G, int g, uint32_t b, const uint8_t* tbl) {
  const uint32_t v = tbl[b & 0x7Fu];
  const uint64_t four = ((uint64_t)(v & 15u) * 0x0000200040008001ull) & kThSpread;   // bit c -> bit 16 c
  G.acc = (G.acc & ~(kThSpread << g)) | (four << g);
  G.acc4 = (G.acc4 & ~(1u << g)) | ((v >> 4 & 1u) << g);
}

// the footprint option of class c that GPU byte b takes first (mig.py:41-54:
// size 7 {7F}, 4 {0F}, 3 {70 = @4, 0F = @0}, 2 {03, 0C, 30}, 1: the lowest
// free slot); the option's cells are its footprint, its lowest bit the start
__device__ __forceinline__ uint32_t th_option(uint32_t b, int c) {
  b &= 0x7Fu;
  const uint32_t f = ~b & 0x7Fu;
  const uint32_t k1 = (b & 0x03u) == 0 ? 0x03u : (b & 0x0Cu) == 0 ? 0x0Cu : 0x30u;
  const uint32_t k2 = (b & 0x70u) == 0 ? 0x70u : 0x0Fu;
  return c == 4 ? 0x7Fu : c == 3 ? 0x0Fu : c == 2 ? k2 : c == 1 ? k1 : f & (0u - f);   // (selects: no divergence)
}

// place a segment of class c on GPU g (the first-fit choice); false: log full
__device__ __forceinline__ bool th_place(ThWarp& P, int t, ThGpus& G, int& L, int g, int c, int s,
                                         const uint8_t* tbl) {
  if (L >= kThL) return false;
  const uint32_t b = th_byte(G, g);
  const uint32_t k = th_option(b, c);
  const uint32_t nb = b | k | (c == 2 && k == 0x0Fu ? 0x80u : 0u);   // size 3 at slot 0 uses 3 of its 4 cells
  const int sh = (g & 7) << 3;
  if (g < 8) G.lo = (G.lo & ~(0xFFull << sh)) | (uint64_t)nb << sh;
  else G.hi = (G.hi & ~(0xFFull << sh)) | (uint64_t)nb << sh;
  th_set_acc(G, g, nb, tbl);
  G.len += 1ull << (4 * g);
  P.log[L++][t] = (uint16_t)(g << 11 | (s * 5 + c) << 3 | (__ffs(k) - 1));
  return true;
}

__device__ __forceinline__ int th_reps(uint32_t mt, int c) {
  return ((int)(mt >> 8 & 15) == c ? (int)(mt & 255) : 0) + ((int)(mt >> 12 & 15) == c ? 1 : 0);
}

// relocate_segments from an empty map (allocator.py:292-316): the queue is
// size 7, 4, 3, 2, 1 (allocator.py:46-51), services in input order, opt
// copies then last (:284-289); first-fit over the GPUs, new GPUs appended
// (:280-281) -- the first GPU past the map accepts anything.  One flat loop
// over the thread's queue items, so the warp's threads stay converged;
// cmA = classes 4..1 x 16 service bits, cm0 = class 0.  ok = false: defer
// (more than kThG GPUs or a full log).
__device__ __forceinline__ void th_relocate(ThWarp& P, int t, const uint32_t* meta, uint64_t cmA, uint32_t cm0,
                                            int segs, ThGpus& G, int& L, int& ngpus, bool& ok, const uint8_t* tbl) {
  th_init(G);
  L = 0;
  ngpus = 0;
  const int items = ok ? segs : 0;
  const int maxit = __reduce_max_sync(0xffffffffu, items);
  int c = 4, nexts = 0, s = 0, left = 0;
  for (int it = 0; it < maxit; it++) {
    if (it < items && ok) {
      while (left == 0) {                      // the next service with segments of class c
        const uint32_t cm = c > 0 ? (uint32_t)(cmA >> (16 * (4 - c))) & 0xFFFFu : cm0;
        const uint32_t m = cm >> nexts << nexts;
        if (m) { s = __ffs(m) - 1; nexts = s + 1; left = th_reps(meta[s], c); }
        else { c--; nexts = 0; }
      }
      const int g = __ffs(th_acc(G, c)) - 1;
      if (g < 0 || !th_place(P, t, G, L, g, c, s, tbl)) ok = false;
      else { ngpus = max(ngpus, g + 1); left--; }
    }
  }
  __syncwarp();
}
// best throughput of (service li of the chunk, size class c); 0 = absent
__device__ __forceinline__ double th_tp(const ThWarp& P, const IndexView& V, const int64_t* seg_start, int li, int c) {
  const int b = P.u.svc.best[li][c];
  if (b == 0xFFFF) return 0.0;
  const int tb = P.u.svc.best[li][5];
  return V.tp[(seg_start[tb * 5 + c] + b) * V.tp_stride];
}

// Plan outcome of one thread's scenario, carried from planning to emission
// (the staging rows alias the service area, so emission starts only after
// the whole warp has planned)
enum { TH_OK = 0, TH_ERROR = 1, TH_CAPACITY = 2, TH_DEFER = 3 };
struct ThState {
  ThGpus G;
  int kind, L, ngpus, n_before, nd, n, err;   // err = status | service << 8 (TH_ERROR)
  bool fallback;
};

// One drain attempt of optimize_allocation (allocator.py:386-419) on GPU
// `index` (nl placements): remove each placement, credit the freed_rate
// ledger, propose replacement small segments (allocator.py:319-359), refill
// them onto the other GPUs (size 2 first, then size 1; no new GPU), all or
// nothing; a failure restores the drained placements and the ledger and
// records a diagnostic.  The ledger changes stay in registers until the
// drain succeeds.  ok = false: defer (the placement log is full).
__device__ __forceinline__ void th_drain(const PlanArgs& A, const IndexView& V, ThWarp& P, ThLedger& Q, int t, int i0,
                                         int index,
                                         int nl, ThGpus& G, int& L, int ngpus, int& next, int& nd, bool& ok,
                                         const uint8_t* tbl) {
  const int64_t* seg_start = A.seg_start;
  // the drained GPU's placements, in list order (log positions)
  uint64_t pos = 0;
  {
    int q = 0;
    for (int j = 0; j < L && q < nl; j++)
      if ((P.log[j][t] >> 11) == index) { pos |= (uint64_t)j << (8 * q); q++; }
  }
  const int sv_next = next;
  int fail = -1, fsvc = 0, rot = nl, tot2 = 0, tot1 = 0;
  uint32_t wsp = 0;              // service of entry kk (4 bits each)
  uint64_t r2p = 0, r1p = 0;     // proposed size-2 / size-1 counts of entry kk (bytes)
  int wo[7];
  double wf[7];
  uint16_t ev[7];
#pragma unroll
  for (int kk = 0; kk < 7; kk++) { wo[kk] = 0; wf[kk] = 0.0; ev[kk] = 0; }
#pragma unroll
  for (int kk = 0; kk < 7; kk++) {
    if (kk < nl && fail < 0) {
      const uint16_t v = P.log[(pos >> (8 * kk)) & 0xFF][t];
      ev[kk] = v;
      const int cat = (v >> 3) & 0xFF;
      const int s = cat / 5, c = cat % 5;
      wsp |= (uint32_t)s << (4 * kk);
      const double tpp = th_tp(P, V, seg_start, i0 + s, c);
      // the ledger entry of s as this drain has left it so far
      bool seen = false;
      double cur = 0.0;
      int ord = 0;
#pragma unroll
      for (int jj = 0; jj < kk; jj++)
        if ((int)(wsp >> (4 * jj) & 15u) == s) { seen = true; cur = wf[jj]; ord = wo[jj]; }
      if (!seen) { ord = Q.order[s]; cur = Q.freed[s]; }
      double f;
      if (ord == 0) { ord = ++next; f = __dadd_rn(0.0, tpp); }
      else f = __dadd_rn(cur, tpp);
      wo[kk] = ord;
      const double t1 = th_tp(P, V, seg_start, i0 + s, 0), t2 = th_tp(P, V, seg_start, i0 + s, 1);
      long long k2, k1;
      if (!propose_small(t1, t2, f, k2, k1)) {
        wf[kk] = f;
        fail = PARVA_DIAG_SMALL_UNAVAILABLE; fsvc = s; rot = kk + 1;
      } else {
        for (long long j = 0; j < k2; j++) f = __dsub_rn(f, t2);
        for (long long j = 0; j < k1; j++) f = __dsub_rn(f, t1);
        wf[kk] = f;
        // more small segments than the other GPUs' slots cannot fit: the
        // refill would need a new GPU (any bound >= 7 (ngpus - 1) is exact)
        if (tot2 > kThG * 7 || tot2 + k2 > kThG * 7 || tot1 + k1 > kThG * 7) tot2 = kThG * 7 + 1;
        else { tot2 += (int)k2; tot1 += (int)k1; }
        r2p |= (uint64_t)min(k2, (long long)kThG * 7) << (8 * kk);
        r1p |= (uint64_t)min(k1, (long long)kThG * 7) << (8 * kk);
      }
    }
  }
  if (fail < 0) {
    if (tot2 > kThG * 7) fail = PARVA_DIAG_NEED_NEW_GPU;
    else {
      // allocate(exclude=index, allow_new=False) (allocator.py:255-277):
      // every size-2 segment in drain order, then every size-1 segment
      const ThGpus Gs = G;
      const int Ls = L;
      const uint32_t allowed = ((1u << ngpus) - 1u) & ~(1u << index);
      int cc = 1, kk = -1, left = 0;
      const int total = tot2 + tot1;
      for (int it = 0; it < total; it++) {
        while (left == 0) {
          if (++kk >= nl) { cc = 0; kk = 0; }
          left = (int)(((cc ? r2p : r1p) >> (8 * kk)) & 0xFFu);
        }
        const uint32_t acc = th_acc(G, cc) & allowed;
        if (!acc) { fail = PARVA_DIAG_NEED_NEW_GPU; break; }
        if (!th_place(P, t, G, L, __ffs(acc) - 1, cc, (int)(wsp >> (4 * kk) & 15u), tbl)) { ok = false; break; }
        left--;
      }
      if (fail >= 0) { G = Gs; L = Ls; }         // all or nothing (allocator.py:272-277)
    }
  }
  if (!ok) return;
  if (fail >= 0) {
    // restore (allocator.py:415-417): the drained placements not yet
    // removed keep their order, the removed ones are re-appended
    if (rot != nl) {
      int w = 0, dropped = 0;
      for (int j = 0; j < L; j++) {
        const uint16_t v = P.log[j][t];
        if ((v >> 11) == index && dropped < rot) { dropped++; continue; }
        P.log[w++][t] = v;
      }
#pragma unroll
      for (int kk = 0; kk < 7; kk++)
        if (kk < rot) P.log[w++][t] = ev[kk];
    }
    next = sv_next;
    if (nd < kThG)
      Q.diag[nd] = (uint16_t)(index << 7 | fail << 5 | (fail == PARVA_DIAG_SMALL_UNAVAILABLE ? fsvc : 0));
    nd++;
  } else {
    // committed: the ledger, and the drained GPU leaves the map
#pragma unroll
    for (int kk = 0; kk < 7; kk++)
      if (kk < nl) {
        const int s = (int)(wsp >> (4 * kk) & 15u);
        Q.freed[s] = wf[kk];
        Q.order[s] = (uint8_t)wo[kk];
      }
    int w = 0;
    for (int j = 0; j < L; j++) {
      const uint16_t v = P.log[j][t];
      if ((v >> 11) != index) P.log[w++][t] = v;
    }
    L = w;
    const uint64_t keep = ~(0xFFull << ((index & 7) << 3));
    if (index < 8) G.lo &= keep; else G.hi &= keep;
    G.len &= ~(15ull << (4 * index));
    G.acc |= kThSpread << index;
    G.acc4 |= 1u << index;
  }
}

// Plan the scenario of thread t (chunk-local services [i0, i0 + n); valid:
// the thread has one).  Every lane of the warp calls it: the loops are
// warp-uniform or per-thread with short bodies, so the threads reconverge.
__device__ __forceinline__ void th_plan(const PlanArgs& A, const IndexView& V, ThWarp& P, ThLedger& Q, int t,
                                        bool valid, int i0, int n, ThState& R, const uint8_t* tbl) {
  R.kind = TH_DEFER;
  R.n = n;
  R.nd = 0;
  R.L = 0;
  R.ngpus = 0;
  R.n_before = 0;
  R.fallback = false;
  bool ok = valid && n >= 0 && n <= kThS && i0 + n <= kThSvc;
  const uint32_t* meta = P.u.svc.meta + (ok ? i0 : 0);
  // services: first failure (input order), segment total, per-class queues
  uint64_t cmA = 0;
  uint32_t cm0 = 0;
  int segs = 0;
  if (ok) {
    for (int s = 0; s < n; s++) {
      const uint32_t mt = meta[s];
      const int st = (int)(mt >> 16 & 0xFF);
      if (st != PARVA_OK) {           // plan_scenario_warp: the first failing service's status
        R.kind = TH_ERROR;
        R.err = st | s << 8;
        ok = false;
        break;
      }
      const int cnt = (int)(mt & 255), opt = (int)(mt >> 8 & 15), last = (int)(mt >> 12 & 15);
      segs += cnt + (last != 15);
      if (cnt > 0) {
        if (opt > 0) cmA |= 1ull << (16 * (4 - opt) + s); else cm0 |= 1u << s;
      }
      if (last != 15) {
        if (last > 0) cmA |= 1ull << (16 * (4 - last) + s); else cm0 |= 1u << s;
      }
    }
    if (ok && segs > kThG * 7) ok = false;
  }
  ThGpus& G = R.G;
  int L, ngpus;
  th_relocate(P, t, meta, cmA, cm0, segs, G, L, ngpus, ok, tbl);
  const int n_before = ngpus;
  int total_before = 0;
  if (ok) {
    for (int g = 0; g < ngpus; g++) total_before += th_gpc(th_byte(G, g));
    for (int s = 0; s < n; s++) Q.order[s] = 0;
  }
  int nd = 0;
  bool fallback = false;
  if (A.optimize) {
    // GPUs last -> first (allocator.py:382); each round every thread drains
    // its next candidate (condition checked when it is visited)
    int next = 0, idx = ok ? ngpus : 0;
    for (;;) {
      bool have = false;
      int nl = 0;
      if (ok)
        while (idx > 0) {
          idx--;
          nl = th_len(G, idx);
          if (nl > 0 && th_gpc(th_byte(G, idx)) <= A.threshold) { have = true; break; }
        }
      if (!__any_sync(0xffffffffu, have)) break;
      if (have) th_drain(A, V, P, Q, t, i0, idx, nl, G, L, ngpus, next, nd, ok, tbl);
      __syncwarp();
    }
    // compaction + regression check (allocator.py:423-435), in integers as
    // in the warp planner (exact for <= 32 GPUs)
    bool redo = false;
    if (ok) {
      int n_after = 0, total_after = 0;
      for (int g = 0; g < ngpus; g++)
        if (th_len(G, g) > 0) { n_after++; total_after += th_gpc(th_byte(G, g)); }
      redo = n_after > n_before ||
             (n_after > 0 && n_before > 0 && total_after * n_before < total_before * n_after);
    }
    if (__any_sync(0xffffffffu, redo)) {
      // the relocation result again (deterministic), empty ledger
      ThGpus G2;
      int L2, ng2;
      bool ok2 = redo;
      th_relocate(P, t, meta, cmA, cm0, segs, G2, L2, ng2, ok2, tbl);
      if (redo) {
        fallback = true;
        G = G2; L = L2; ngpus = ng2;
        for (int s = 0; s < n; s++) Q.order[s] = 0;
        nd = 0;
      }
    }
  }
  if (!ok) return;
  R.kind = nd > kThG ? TH_DEFER : TH_OK;
  R.L = L;
  R.ngpus = ngpus;
  R.n_before = n_before;
  R.nd = nd;
  R.fallback = fallback;
}

// Build thread t's record into its staging row (reads the log, diagnostics
// and ledger, never the service area the row aliases).  Returns 1 when a
// 64-byte record spills (the row holds the full 128-byte record).
__device__ __forceinline__ int th_emit(const PlanArgs& A, ThWarp& P, const ThLedger& Q, int t, ThState& R) {
  uint32_t* row = P.u.stage[t];
#pragma unroll
  for (int w = 0; w < 32; w++) row[w] = 0u;
  if (R.kind == TH_ERROR) {
    row[0] = (uint32_t)(R.err & 0xFF) | (uint32_t)(R.err >> 8 & 0xFF) << 8;
    return 0;
  }
  if (R.kind == TH_CAPACITY) {
    row[0] = PARVA_CAPACITY;
    return 0;
  }
  const ThGpus& G = R.G;
  int n_final = 0, n_led = 0;
  for (int g = 0; g < R.ngpus; g++) n_final += th_len(G, g) > 0;
  for (int s = 0; s < R.n; s++) n_led += Q.order[s] > 0;
  const int n_place = R.L;
  const int led_off = (2 * (n_place + R.nd) + 7) & ~7;
  const int need = led_off + 10 * n_led;
  if (need > PARVA_PLAN_PAYLOAD) {
    R.kind = TH_CAPACITY;
    row[0] = PARVA_CAPACITY;
    return 0;
  }
  row[0] = (uint32_t)n_final << 16 | (uint32_t)R.n_before << 24;
  row[1] = (uint32_t)n_place | (uint32_t)R.nd << 8 | (uint32_t)n_led << 16 |
           (uint32_t)(R.fallback ? PARVA_FLAG_FALLBACK : 0) << 24;
  uint16_t* pay = reinterpret_cast<uint16_t*>(row + 2);
  // placements GPU by GPU, each GPU's in list (= log) order: per-GPU write
  // positions as bytes of two words
  uint64_t plo = 0, phi = 0;
  {
    int acc = 0;
    for (int g = 0; g < R.ngpus; g++) {
      const uint64_t v = (uint64_t)acc << ((g & 7) << 3);
      if (g < 8) plo |= v; else phi |= v;
      acc += th_len(G, g);
    }
  }
  for (int j = 0; j < n_place; j++) {
    const uint16_t v = P.log[j][t];
    const int g = v >> 11, sh = (g & 7) << 3;
    const int p = (int)(((g < 8 ? plo : phi) >> sh) & 0xFF);
    if (g < 8) plo += 1ull << sh; else phi += 1ull << sh;
    pay[p] = v;
  }
  for (int d = 0; d < R.nd; d++) pay[n_place + d] = Q.diag[d];
  if (n_led) {
    uint32_t* val = row + 2 + led_off / 4;                 // 8-B values in insertion order
    uint16_t* key = pay + (led_off + 8 * n_led) / 2;       // u16 service | rank << 8
    for (int s = 0; s < R.n; s++) {
      const int o = Q.order[s];
      if (!o) continue;
      const unsigned long long b = (unsigned long long)__double_as_longlong(Q.freed[s]);
      val[2 * (o - 1)] = (uint32_t)b;
      val[2 * (o - 1) + 1] = (uint32_t)(b >> 32);
      key[o - 1] = (uint16_t)(s | o << 8);
    }
  }
  return A.plan_bytes == 64 && need > 64 - 8;
}

// configure K services at once through the global index (segment starts
// as i64): the 5 K binary searches advance in lockstep, so a lane keeps 5 K
// independent loads in flight per step (configurator.py:93-124 via the
// prefix-argmax index, then select_optimal_segment + match_demand); stores
// each config record at its index.  valid[j] = false: service j is absent.
template <int K>
__device__ __forceinline__ void th_configure_k(const PlanArgs& A, const double* tp, int tp_stride, const int t[K],
                                               const double rate[K], const double bound[K], const int64_t i[K],
                                               const bool valid[K], parva_config_record r[K]) {
  int s0[K * 5], n[K * 5], lo[K * 5];
  int nmax = 0;
#pragma unroll
  for (int j = 0; j < K; j++) {
    const bool ok = valid[j] && t[j] >= 0 && t[j] < A.n_tables;
#pragma unroll
    for (int c = 0; c < 5; c++) {
      s0[j * 5 + c] = ok ? (int)A.seg_start[t[j] * 5 + c] : 0;
      n[j * 5 + c] = ok ? A.seg_count[t[j] * 5 + c] : 0;
      lo[j * 5 + c] = 0;
      nmax = max(nmax, n[j * 5 + c]);
    }
  }
  for (int step = nmax ? 1 << (31 - __clz(nmax)) : 0; step > 0; step >>= 1) {
#pragma unroll
    for (int q = 0; q < K * 5; q++) {
      const int probe = lo[q] + step;
      if (probe <= n[q] && A.idx_lat[s0[q] + probe - 1] < bound[q / 5]) lo[q] = probe;
    }
  }
#pragma unroll
  for (int j = 0; j < K; j++) {
    if (!valid[j]) continue;
    double tpc[5];
    r[j] = parva_config_record{};
    if (t[j] < 0 || t[j] >= A.n_tables) {
#pragma unroll
      for (int c = 0; c < 5; c++) r[j].best[c] = -1;
      r[j].opt_sc = -1; r[j].last_sc = -1; r[j].status = PARVA_BAD_INPUT;
    } else {
#pragma unroll
      for (int c = 0; c < 5; c++) {
        const int q = j * 5 + c;
        const int b = lo[q] ? (int)A.idx_best[s0[q] + lo[q] - 1] : -1;
        r[j].best[c] = (int16_t)b;
        tpc[c] = b >= 0 ? tp[(s0[q] + b) * tp_stride] : 0.0;
      }
      match_demand(tpc, rate[j], r[j], A.cfg_format == PARVA_CFG_FULL);
      if (r[j].status == PARVA_INFEASIBLE_SLO) r[j].opt_sc = -1;
    }
    store_config(A, i[j], r[j]);
  }
}

__device__ __forceinline__ int th_table(const PlanArgs& A, int64_t i) {
  return A.svc_table16 ? (int)A.svc_table16[i] : A.svc_table[i];
}

// the planner's view of a configured service (chunk-local index li)
__device__ __forceinline__ void th_stage(ThWarp& P, int li, int t, const parva_config_record& r) {
  if (li >= kThSvc) return;
  const long long cn = r.count < 0 ? 0 : r.count > 255 ? 255 : r.count;
  P.u.svc.meta[li] = (uint32_t)cn | (uint32_t)(r.opt_sc < 0 ? 15 : r.opt_sc) << 8 |
                     (uint32_t)(r.last_sc < 0 ? 15 : r.last_sc) << 12 | (uint32_t)(r.status & 0xFF) << 16;
  uint16_t* b = P.u.svc.best[li];
#pragma unroll
  for (int c = 0; c < 5; c++) b[c] = (uint16_t)r.best[c];
  b[5] = (uint16_t)t;
}

// K2, thread-per-scenario form.  kMirror: the fused all-gather (each chunk's
// records also go to this rank's part of the slot on every rank).
template <bool kMirror>
__global__ void __launch_bounds__(TH_THREADS, PARVA_TH_MINB) plan_thread_kernel(PlanArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ int go;
  __shared__ uint8_t s_acc[128];   // bit c: a GPU with these occupied cells accepts size class c
  // an overlapped successor may take SM space as this grid's CTAs retire;
  // the slot ticket keeps it from storing into a slot still being written
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ThWarp& P = reinterpret_cast<ThWarp*>(smem_raw)[warp];
  const double* tp = A.idx_tp ? A.idx_tp : A.pts;
  const int tp_stride = A.idx_tp ? 1 : 2;
  const IndexView V{nullptr, nullptr, A.idx_lat, A.idx_best, tp, tp_stride};
  for (int m = threadIdx.x; m < 128; m += TH_THREADS) {
    uint32_t v = 0;
#pragma unroll
    for (int c = 0; c < 5; c++) v |= (uint32_t)(find_start((uint32_t)m, c) >= 0) << c;
    s_acc[m] = (uint8_t)v;
  }
  if (threadIdx.x == 0) {
    go = 1;
#if !defined(PARVA_AB_NO_TICKET) && !defined(PARVA_AB_NO_WAIT)
    if (A.slot_count)
      go = ticket_wait(A.slot_count, A.slot_wait, A.ack_row, A.n_mirror, A.ack_prev, A.ticket_timeout_ns, A.err_word);
#endif
  }
  // warm this SM's L1 with the index (a small one: every lookup of the
  // binary searches would otherwise start as a dependent chain of L2 misses)
  if (A.n_points * 18 <= kThPrefetch) {
    const int64_t np = A.n_points, nseg = (int64_t)A.n_tables * 5;
    const char* rg[5] = {(const char*)A.idx_lat, (const char*)A.idx_best, (const char*)tp, (const char*)A.seg_start,
                         (const char*)A.seg_count};
    const int64_t nb[5] = {np * 8, np * 2, np * 8 * tp_stride, nseg * 8, nseg * 4};
#pragma unroll
    for (int r = 0; r < 5; r++)
      for (int64_t o = (int64_t)threadIdx.x * 128; o < nb[r]; o += TH_THREADS * 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(rg[r] + o));
  }
  __syncthreads();
  if (A.slot_count && !go) return;            // timed out: store nothing
  const int n_chunks = (A.n_scen + 31) / 32;
  const int stride = gridDim.x * TH_WARPS;
  for (int ch = blockIdx.x * TH_WARPS + warp; ch < n_chunks; ch += stride) {
    const int k0 = ch * 32, k1 = min(A.n_scen, k0 + 32), cnt = k1 - k0;
    const int a_base = A.scen_off[k0], a_end = A.scen_off[k1];
    // the chunk's inputs (~7 KB for C2) into L1 at once: the configure
    // rounds below then wait on L1 instead of one HBM latency each
    {
      const int64_t nsv = a_end - a_base;
      const char* rg[3] = {A.svc_table16 ? (const char*)(A.svc_table16 + a_base) : (const char*)(A.svc_table + a_base),
                           (const char*)(A.svc_rate + a_base), (const char*)(A.svc_bound + a_base)};
      const int64_t nb[3] = {nsv * (A.svc_table16 ? 2 : 4), nsv * 8, nsv * 8};
#pragma unroll
      for (int r = 0; r < 3; r++)
        for (int64_t o = (int64_t)lane * 128; o < nb[r] + 128; o += 32 * 128)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(rg[r] + o));
    }
    // ---- configure the chunk's services (lane-strided, coalesced; two
    // services per lane at a time)
    for (int i = a_base + lane; i < a_end; i += 64) {
      const int64_t ii[2] = {i, i + 32};
      const bool v[2] = {true, i + 32 < a_end};
      const int tt[2] = {th_table(A, i), v[1] ? th_table(A, i + 32) : 0};
      const double rr[2] = {A.svc_rate[i], v[1] ? A.svc_rate[i + 32] : 0.0};
      const double bb[2] = {A.svc_bound[i], v[1] ? A.svc_bound[i + 32] : 0.0};
      parva_config_record r[2];
      th_configure_k<2>(A, tp, tp_stride, tt, rr, bb, ii, v, r);
      th_stage(P, i - a_base, tt[0], r[0]);
      if (v[1]) th_stage(P, i + 32 - a_base, tt[1], r[1]);
    }
    __syncwarp();
    // ---- plan: thread j takes scenario k0 + j
    ThState R;
    ThLedger Q;
    {
      int a = a_base, n = 0;
      if (lane < cnt) { a = A.scen_off[k0 + lane]; n = A.scen_off[k0 + lane + 1] - a; }
      th_plan(A, V, P, Q, lane, lane < cnt && a >= a_base, a - a_base, n, R, s_acc);
    }
    __syncwarp();
    // ---- emit into the staging rows (they alias the service area)
    int sp = 0;
    if (lane < cnt && R.kind != TH_DEFER) sp = th_emit(A, P, Q, lane, R);
    if (sp) {
      // 64-byte records: the full record goes to the overflow area (direct:
      // the scenario's slot; else the spill list), the 64-byte slot says so
      const int k = k0 + lane;
      uint32_t* row = P.u.stage[lane];
      uint32_t* dst = nullptr;
      uint32_t head = PARVA_SPILLED;
      if (A.spill_direct) {
        dst = reinterpret_cast<uint32_t*>(A.spill + (size_t)k * 128);
      } else {
        const int slot = atomicAdd(A.spill_count, 1);
        if (slot < A.spill_cap) {
          uint8_t* e = A.spill + (size_t)slot * kSpillEntry;
          *reinterpret_cast<int4*>(e) = make_int4(k, 0, 0, 0);
          dst = reinterpret_cast<uint32_t*>(e + 16);
        } else {
          head = PARVA_CAPACITY;
        }
      }
      if (dst)
        for (int w = 0; w < 32; w++) dst[w] = row[w];
      row[0] = head;
      for (int w = 1; w < 16; w++) row[w] = 0u;
    }
    __syncwarp();
    const unsigned defer = __ballot_sync(0xffffffffu, lane < cnt && R.kind == TH_DEFER);
    {
      const int lg = A.plan_bytes == 64 ? 4 : 5;       // words per record: 16 or 32
      uint32_t* dst = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(A.plan) + (size_t)k0 * A.plan_bytes);
      for (int w = lane; w < cnt << lg; w += 32) {
        const int r = w >> lg;
        if (!(defer >> r & 1u)) dst[w] = P.u.stage[r][w & ((1 << lg) - 1)];
      }
    }
    __syncwarp();
    // ---- deferred scenarios: the whole warp (lane = service, then GPU)
    for (unsigned m = defer; m; m &= m - 1) {
      const int j = __ffs(m) - 1, k = k0 + j;
      const int a = A.scen_off[k], n = A.scen_off[k + 1] - a;
      if (n > 0 && n <= PARVA_PLAN_MAX_SERVICES && lane < n) {
        const int64_t ii[1] = {a + lane};
        const bool v[1] = {true};
        const int tt[1] = {th_table(A, a + lane)};
        const double rr[1] = {A.svc_rate[a + lane]}, bb[1] = {A.svc_bound[a + lane]};
        parva_config_record r[1];
        th_configure_k<1>(A, tp, tp_stride, tt, rr, bb, ii, v, r);
        double tpc[5];
#pragma unroll
        for (int c = 0; c < 5; c++) {
          const int b = r[0].best[c];
          tpc[c] = (b >= 0 && r[0].status != PARVA_BAD_INPUT) ? tp[(A.seg_start[tt[0] * 5 + c] + b) * tp_stride] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 5; c++) P.u.w.s.tp[lane * 5 + c] = tpc[c];
        P.u.w.s.meta[lane] = pack_meta(r[0].opt_sc, r[0].last_sc, r[0].status, r[0].count);
      }
      __syncwarp();
      plan_scenario_warp<32>(A, P.u.w.g, k, n, P.u.w.s.tp, P.u.w.s.meta, n >= 0, lane, Grp<32>{0xffffffffu, 0});
      __syncwarp();
    }
    if (kMirror) {
      // fused all-gather: the chunk's plan and config records go to this
      // rank's part of the slot on every rank (coalesced peer stores)
      __syncwarp();
      const int cfg_b = A.cfg_format == PARVA_CFG_TINY ? 8 : A.cfg_format == PARVA_CFG_COMPACT ? 16 : 32;
      const size_t p0 = (size_t)k0 * A.plan_bytes, pn = (size_t)cnt * A.plan_bytes / 16;
      const size_t c0 = (size_t)a_base * cfg_b, cn = (size_t)(a_end - a_base) * cfg_b / 8;
      const uint4* ps = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(A.plan) + p0);
      const uint2* cs = reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(A.cfg) + c0);
      for (int mm = 0; mm < A.n_mirror; mm++) {
        uint4* pd = reinterpret_cast<uint4*>(A.mirror_plan[mm] + p0);
        uint2* cd = reinterpret_cast<uint2*>(A.mirror_cfg[mm] + c0);
        if (pd == ps) continue;
        for (size_t x = lane; x < pn; x += 32) pd[x] = ps[x];
        for (size_t x = lane; x < cn; x += 32) cd[x] = cs[x];
      }
      if (A.plan_bytes == 64) {
        for (int j = 0; j < cnt; j++) {
          const size_t kk = (size_t)(k0 + j);
          if (reinterpret_cast<const uint8_t*>(A.plan)[kk * 64] == PARVA_SPILLED && lane < 8) {
            const uint4 v = reinterpret_cast<const uint4*>(A.spill + kk * 128)[lane];
            for (int mm = 0; mm < A.n_mirror; mm++)
              if (A.mirror_spill[mm] != A.spill) reinterpret_cast<uint4*>(A.mirror_spill[mm] + kk * 128)[lane] = v;
          }
        }
      }
    }
  }
#if !defined(PARVA_AB_NO_TICKET) && !defined(PARVA_AB_NO_DONE)
  if (A.slot_count) {
    // completion, as in the tile kernel: one release reduction per CTA
    // after a barrier; fused: the last CTA publishes the epoch on every rank
    if (kMirror) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      if (kMirror && atomicAdd(A.done_ctas, 1u) == gridDim.x - 1) {
        atomicExch(A.done_ctas, 0u);
        __threadfence_system();
        for (int mm = 0; mm < A.n_mirror; mm++)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.peer_flag[mm]), "r"(A.flag_epoch) : "memory");
      }
      unsigned long long mine = 0;
      for (int w = 0; w < TH_WARPS; w++)
        for (int ch = blockIdx.x * TH_WARPS + w; ch < n_chunks; ch += stride)
          mine += (unsigned long long)(min(A.n_scen, ch * 32 + 32) - ch * 32);
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(A.slot_count), "l"(mine) : "memory");
    }
  }
#endif
}
