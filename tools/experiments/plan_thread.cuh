// plan_thread.cuh — K2 planner, thread-per-scenario form (sm_100a).
// EXPERIMENT (not built): thread-per-scenario planner. Exact (passed every GPU parity
// test when wired into the tile kernel) and 2.8x fewer warp instructions than the
// warp planner on C2 (7.8 M vs 22 M), but latency-bound at C2 scale: 68 scenarios
// per SM leave 2-3 warps whose divergent chains take ~43 us, so the kernel went
// from 36 us to 60 us (C4: 2.3 ms -> 3.7 ms with 1 CTA/SM). Kept for reference.
//
// relocate_segments (allocator.py:292-316) + optimize_allocation
// (allocator.py:362-443) for one scenario per THREAD, on the configured
// services a tile left in shared memory.  This is the common case of the
// batched planner (<= kTS services, <= kTG GPUs per scenario): the per-
// scenario algorithm is sequential anyway, so one thread per scenario keeps
// 32 scenarios in flight per warp instead of one, at the same exact
// semantics as the warp planner (plan_batch.cu), which remains the path for
// scenarios beyond these limits.
//
// State lives in shared memory in thread-minor arrays (x[i][kTP]), so any
// per-thread index is bank-conflict free.  A GPU is a byte: bits 0-6 are the
// occupied-or-blocked slots, bit 7 marks a size-3 segment at slot 0 (which
// blocks slot 3 without occupying it), so its GPC count is
// popc(mask & 0x7F) - (mask >> 7).
#pragma once

#include "parva_common.cuh"

namespace parva {

constexpr int kTP = 128;   // planner threads (tile scenarios) per CTA
constexpr int kTG = 16;    // GPUs per scenario on the thread path
constexpr int kTS = 16;    // services per scenario on the thread path
constexpr int kTD = 7;     // placements per GPU (7 slots)
constexpr int kRecStride = 132;   // staged record stride (bytes): 33 words, conflict-free

struct alignas(16) ThreadState {
  double freed[kTS][kTP];          // freed_rate ledger (allocator.py:396-404)
  double lfreed[kTD][kTP];         // ledger log of the drain in progress (rollback)
  uint8_t r2[kTD][kTP];            // proposal runs of the drain in progress: k2, k1 (saturated:
  uint8_t r1[kTD][kTP];            //   more than kTG*kTD of either cannot fit anyway)
  uint16_t list[kTG * kTD][kTP];   // per-GPU placement lists: (service*5 + class) << 3 | slot
  uint16_t diag[kTG][kTP];         // optimize diagnostics, gpu << 7 | reason << 5 | service
  uint8_t mask[kTG][kTP];
  uint8_t len[kTG][kTP];
  uint8_t smask[kTG][kTP];         // refill snapshot (all-or-nothing undo, allocator.py:272-277)
  uint8_t slen[kTG][kTP];
  uint8_t order[kTS][kTP];         // ledger insertion rank, 0 = absent
  uint8_t lorder[kTD][kTP];
  uint8_t ls[kTD][kTP];            // service of each log entry / run
};

__device__ __forceinline__ int tgpc(uint32_t m) { return __popc(m & 0x7Fu) - (int)(m >> 7); }

__device__ __forceinline__ uint32_t tfoot(int c, int st) {
  return footprint(c, st) | (c == 2 && st == 0 ? 0x80u : 0u);
}

// first-fit of one segment of class c onto GPUs [*cur, ngpus) skipping
// `skip`; *cur only advances (GPUs before it refuse class c, and placements
// never make a GPU accept more).  Returns the GPU or -1.
__device__ __forceinline__ int tfirst_fit(ThreadState& S, int t, int c, int ngpus, int skip, int& cur, int& st) {
  for (int g = cur; g < ngpus; g++) {
    if (g == skip) continue;
    const int s = find_start(S.mask[g][t] & 0x7Fu, c);
    if (s >= 0) { cur = g; st = s; return g; }
  }
  cur = ngpus;
  return -1;
}

__device__ __forceinline__ void tplace(ThreadState& S, int t, int g, int c, int st, int svc) {
  S.mask[g][t] = (uint8_t)(S.mask[g][t] | tfoot(c, st));
  const int l = S.len[g][t];
  S.list[g * kTD + l][t] = (uint16_t)(((svc * 5 + c) << 3) | st);
  S.len[g][t] = (uint8_t)(l + 1);
}

// relocate_segments: queue order size 7,4,3,2,1 (allocator.py:46-51),
// services in input order, opt copies then last (:284-289); first-fit with
// new GPUs appended (:280-281).  Returns the GPU count, or -1 if it would
// exceed kTG (the warp path takes the scenario).
__device__ __forceinline__ int trelocate(ThreadState& S, int t, int n, const uint64_t* meta) {
  int ngpus = 0;
  for (int c = 4; c >= 0; c--) {
    int cur = 0;
    for (int s = 0; s < n; s++) {
      const uint64_t m = meta[s];
      const int opt = (int)(m >> 48 & 15), last = (int)(m >> 52 & 15);
      const int reps = (opt == c ? (int)(m & ((1ull << 48) - 1)) : 0) + (last == c ? 1 : 0);
      for (int r = 0; r < reps; r++) {
        int st = 0;
        int g = tfirst_fit(S, t, c, ngpus, -1, cur, st);
        if (g < 0) {
          if (ngpus == kTG) return -1;
          g = ngpus++;
          S.mask[g][t] = 0;
          S.len[g][t] = 0;
          st = find_start(0u, c);
          cur = g;
        }
        tplace(S, t, g, c, st, s);
      }
    }
  }
  return ngpus;
}

__device__ __forceinline__ double tunallocated(int total, int n) {
  if (n == 0) return 0.0;
  return __dsub_rn(1.0, __ddiv_rn((double)total, (double)(7 * n)));
}

// Plan scenario k (n services, configured at cat_tp / meta) into the staged
// record `rec` (plan_bytes wide).  Returns false if the scenario exceeds the
// thread path's limits (the caller hands it to the warp planner).
__device__ bool plan_scenario_thread(const PlanArgs& A, ThreadState& S, int t, int k, int n, const double* cat_tp,
                                     const uint64_t* meta, uint8_t* rec) {
  if (n < 0 || n > kTS) return false;
  // ------------------------------------------------ configured services
  int status = PARVA_OK, err_svc = 0;
  long long segs = 0;
  for (int s = 0; s < n; s++) {
    const uint64_t m = meta[s];
    const int st = (int)(m >> 56);
    if (st != PARVA_OK) { status = st; err_svc = s; break; }
    segs += (long long)(m & ((1ull << 48) - 1)) + (((m >> 52) & 15) != 15 ? 1 : 0);
  }
  uint32_t* rec32 = reinterpret_cast<uint32_t*>(rec);
  if (status != PARVA_OK) {
    for (int w = 0; w < A.plan_bytes / 4; w++) rec32[w] = 0u;
    rec[0] = (uint8_t)status;
    rec[1] = (uint8_t)err_svc;
    return true;
  }
  if (segs > kTG * kTD) return false;

  // --------------------------------------------------- relocate_segments
  const int ngpus = trelocate(S, t, n, meta);
  if (ngpus < 0) return false;
  int total_before = 0;
  for (int g = 0; g < ngpus; g++) total_before += tgpc(S.mask[g][t]);
  for (int s = 0; s < n; s++) S.order[s][t] = 0;

  // -------------------------------------------------- optimize_allocation
  int nd = 0, next = 0;
  bool changed = false, fallback = false;
  if (A.optimize) {
    for (int index = ngpus - 1; index >= 0; index--) {
      const int nl = S.len[index][t];
      if (nl == 0 || tgpc(S.mask[index][t]) > A.threshold) continue;
      const int sv_next = next;
      int fail = -1, fsvc = 0, rot = nl, nlog = 0;
      int tot2 = 0, tot1 = 0;
      for (int kk = 0; kk < nl; kk++) {
        const int cat = S.list[index * kTD + kk][t] >> 3;
        const int s = cat / 5;
        const double tpp = cat_tp[cat];
        // ledger log entry before the change (whole-ledger restore = replaying it backwards)
        S.ls[nlog][t] = (uint8_t)s;
        S.lfreed[nlog][t] = S.freed[s][t];
        S.lorder[nlog][t] = S.order[s][t];
        nlog++;
        double f;
        if (S.order[s][t] == 0) { next++; S.order[s][t] = (uint8_t)next; f = __dadd_rn(0.0, tpp); }
        else f = __dadd_rn(S.freed[s][t], tpp);
        const double t1 = cat_tp[s * 5 + 0], t2 = cat_tp[s * 5 + 1];
        long long k2, k1;
        if (!propose_small(t1, t2, f, k2, k1)) { S.freed[s][t] = f; fail = PARVA_DIAG_SMALL_UNAVAILABLE; fsvc = s; rot = kk + 1; break; }
        for (long long j = 0; j < k2; j++) f = __dsub_rn(f, t2);
        for (long long j = 0; j < k1; j++) f = __dsub_rn(f, t1);
        S.freed[s][t] = f;
        // more small segments than the other GPUs' slots cannot fit: needs a new GPU
        if (tot2 + k2 > kTG * kTD || tot1 + k1 > kTG * kTD) { tot2 = tot1 = kTG * kTD + 1; }
        else { tot2 += (int)k2; tot1 += (int)k1; }
        S.r2[kk][t] = (uint8_t)(k2 > 255 ? 255 : k2);
        S.r1[kk][t] = (uint8_t)(k1 > 255 ? 255 : k1);
      }
      if (fail < 0) {
        if (tot2 > kTG * kTD || tot1 > kTG * kTD) fail = PARVA_DIAG_NEED_NEW_GPU;
        else {
          // allocate(exclude=index, allow_new=False): every size-2 segment in
          // drain order, then every size-1 segment (the queues drain by size)
          for (int g = 0; g < ngpus; g++) { S.smask[g][t] = S.mask[g][t]; S.slen[g][t] = S.len[g][t]; }
          for (int c = 1; c >= 0 && fail < 0; c--) {
            int cur = 0;
            for (int kk = 0; kk < nl && fail < 0; kk++) {
              const int s = (S.list[index * kTD + kk][t] >> 3) / 5;
              const int reps = c == 1 ? S.r2[kk][t] : S.r1[kk][t];
              for (int r = 0; r < reps; r++) {
                int st = 0;
                const int g = tfirst_fit(S, t, c, ngpus, index, cur, st);
                if (g < 0) { fail = PARVA_DIAG_NEED_NEW_GPU; break; }
                tplace(S, t, g, c, st, s);
              }
            }
          }
          if (fail >= 0)
            for (int g = 0; g < ngpus; g++) { S.mask[g][t] = S.smask[g][t]; S.len[g][t] = S.slen[g][t]; }
        }
      }
      if (fail >= 0) {
        // restore: drained placements not yet removed keep their order, the
        // removed ones are re-appended (allocator.py:415-417)
        if (rot != nl) {
          uint16_t e[kTD];
          for (int j = 0; j < nl; j++) e[j] = S.list[index * kTD + j][t];
          for (int j = 0; j < nl; j++) {
            int src = j + rot;
            if (src >= nl) src -= nl;
            S.list[index * kTD + j][t] = e[src];
          }
        }
        for (int q = nlog - 1; q >= 0; q--) {
          const int s = S.ls[q][t];
          S.freed[s][t] = S.lfreed[q][t];
          S.order[s][t] = S.lorder[q][t];
        }
        next = sv_next;
        S.diag[nd][t] = (uint16_t)(index << 7 | fail << 5 | (fail == PARVA_DIAG_SMALL_UNAVAILABLE ? fsvc : 0));
        nd++;
      } else {
        S.len[index][t] = 0;
        S.mask[index][t] = 0;
        changed = true;
      }
    }
    if (changed) {
      // compaction + regression check (allocator.py:423-435)
      int n_after = 0, total_after = 0;
      for (int g = 0; g < ngpus; g++)
        if (S.len[g][t] > 0) { n_after++; total_after += tgpc(S.mask[g][t]); }
      const double ua_before = tunallocated(total_before, ngpus);
      const double ua_after = tunallocated(total_after, n_after);
      if (n_after > ngpus || ua_after > __dadd_rn(ua_before, 1e-12)) {
        // fall back to the relocation result: re-derive it (deterministic)
        fallback = true;
        trelocate(S, t, n, meta);
        for (int s = 0; s < n; s++) S.order[s][t] = 0;
        nd = 0;
      }
    }
  }

  // ------------------------------------------------------- emit record
  int n_place = 0, n_final = 0;
  for (int g = 0; g < ngpus; g++) {
    const int l = S.len[g][t];
    n_place += l;
    n_final += l > 0;
  }
  int n_led = 0;
  for (int s = 0; s < n; s++) n_led += S.order[s][t] > 0;
  const int led_off = (2 * (n_place + nd) + 7) & ~7;
  const int need = led_off + 10 * n_led;
  for (int w = 0; w < A.plan_bytes / 4; w++) rec32[w] = 0u;
  if (need > PARVA_PLAN_PAYLOAD) {
    rec[0] = PARVA_CAPACITY;
    return true;
  }
  const bool spill = A.plan_bytes == 64 && need > 64 - 8;
  // the full 128-byte record goes to global directly when it spills; the
  // staged record is built for the (first) plan_bytes
  uint8_t full[128];
  uint8_t* R = spill ? full : rec;
  const int lim = spill ? 128 : A.plan_bytes;
  if (spill) for (int w = 0; w < 32; w++) reinterpret_cast<uint32_t*>(full)[w] = 0u;
  R[0] = PARVA_OK;
  R[2] = (uint8_t)n_final;
  R[3] = (uint8_t)ngpus;
  R[4] = (uint8_t)n_place;
  R[5] = (uint8_t)nd;
  R[6] = (uint8_t)n_led;
  R[7] = fallback ? PARVA_FLAG_FALLBACK : 0;
  uint8_t* pay = R + 8;
  int p = 0;
  for (int g = 0; g < ngpus; g++) {
    const int l = S.len[g][t];
    for (int j = 0; j < l; j++, p++) {
      const uint16_t v = (uint16_t)(g << 11 | S.list[g * kTD + j][t]);
      if (8 + 2 * p + 1 < lim) { pay[2 * p] = (uint8_t)v; pay[2 * p + 1] = (uint8_t)(v >> 8); }
    }
  }
  for (int d = 0; d < nd; d++, p++) {
    const uint16_t v = S.diag[d][t];
    if (8 + 2 * p + 1 < lim) { pay[2 * p] = (uint8_t)v; pay[2 * p + 1] = (uint8_t)(v >> 8); }
  }
  for (int s = 0; s < n; s++) {
    const int o = S.order[s][t];
    if (o == 0) continue;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(S.freed[s][t]);
    const int vo = led_off + 8 * (o - 1);
    for (int b = 0; b < 8; b++) pay[vo + b] = (uint8_t)(bits >> (8 * b));
    const uint16_t key = (uint16_t)(s | o << 8);
    const int ko = led_off + 8 * n_led + 2 * (o - 1);
    pay[ko] = (uint8_t)key;
    pay[ko + 1] = (uint8_t)(key >> 8);
  }
  if (spill) {
    for (int w = 0; w < 16; w++) rec32[w] = 0u;
    uint8_t* dst = nullptr;
    if (A.spill_direct) {
      dst = A.spill + (size_t)k * 128;
      rec[0] = PARVA_SPILLED;
    } else {
      const int slot = atomicAdd(A.spill_count, 1);
      if (slot < A.spill_cap) {
        uint8_t* e = A.spill + (size_t)slot * kSpillEntry;
        *reinterpret_cast<int4*>(e) = make_int4(k, 0, 0, 0);
        dst = e + 16;
        rec[0] = PARVA_SPILLED;
      } else {
        rec[0] = PARVA_CAPACITY;
      }
    }
    if (dst)
      for (int w = 0; w < 8; w++) reinterpret_cast<uint4*>(dst)[w] = reinterpret_cast<const uint4*>(full)[w];
  }
  return true;
}

}  // namespace parva
