/*
 * migplan_oracle.c — plain-C restatement of the reference planner hot path.
 *
 * TEST INFRASTRUCTURE (see migplan_oracle.h).  Compiled with
 * -ffp-contract=off and without -ffast-math so every double operation rounds
 * exactly like CPython's float arithmetic.  Citations are file:line into
 * /root/reference/pkg/src/migplan/.
 */
#include "migplan_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const int SIZES[5] = {1, 2, 3, 4, 7};

static int size_class(int s) {
  switch (s) {
    case 1: return 0;
    case 2: return 1;
    case 3: return 2;
    case 4: return 3;
    case 7: return 4;
  }
  return -1;
}

/* ======================================================= configurator.py */

/* Python 3.12 builtin sum() of floats with int start 0: result = 0 + x0,
 * then Neumaier compensation over the rest (bltinmodule.c builtin_sum_impl). */
double oracle_pysum(const double* x, int64_t n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0;
  for (int64_t i = 1; i < n; i++) {
    double v = x[i], t = f + v;
    if (fabs(f) >= fabs(v)) c += (f - t) + v;
    else c += (v - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* Service.coverage (configurator.py:60-62) = sum(opt.tp x count, last.tp). */
static double coverage(double topt, int64_t count, int has_last, double tlast) {
  if (count == 0 && !has_last) return 0.0;
  double f, c = 0.0;
  int64_t i0;
  if (count > 0) { f = 0.0 + topt; i0 = 1; } else { f = 0.0 + tlast; i0 = 0; has_last = 0; }
  for (int64_t i = i0; i < count + (has_last ? 1 : 0); i++) {
    double v = i < count ? topt : tlast, t = f + v;
    if (fabs(f) >= fabs(v)) c += (f - t) + v;
    else c += (v - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* _better_triplet (configurator.py:116-124): tuple
 * (tp, -lat, -batch, -procs) > ...; first unequal element decides. */
static int better(double tpa, double lata, int ba, int pa, double tpb, double latb, int bb,
                  int pb) {
  if (tpa != tpb) return tpa > tpb;
  if (-lata != -latb) return -lata > -latb;
  if (ba != bb) return -ba > -bb;
  return -pa > -pb;
}

/* select_optimal_segment (configurator.py:127-139): left fold in caller order. */
int oracle_select_optimal(const otrip* t, int32_t n) {
  if (n <= 0) return -1;
  int best = 0;
  for (int i = 1; i < n; i++) {
    double lhs = t[i].tp * (double)t[best].size;
    double rhs = t[best].tp * (double)t[i].size;
    if (lhs > rhs || (lhs == rhs && t[i].size > t[best].size)) best = i;
  }
  return best;
}

#define COUNT_LIMIT 1099511627776.0 /* 2^40: counts beyond this are refused */

int oracle_configure(const double* tp, const double* lat, const int32_t* batch,
                     const int32_t* procs, const int64_t* seg_start,
                     const int32_t* seg_count, double bound, double rate,
                     parva_config_record* out) {
  memset(out, 0, sizeof(*out));
  for (int c = 0; c < 5; c++) out->best[c] = -1;
  out->opt_sc = -1;
  out->last_sc = -1;
  /* decide_best_triplets (configurator.py:93-113): every point in key order,
   * strict `<` against the internal latency bound, per-size argmax. */
  int any = 0;
  for (int c = 0; c < 5; c++) {
    int64_t s0 = seg_start[c];
    int bj = -1;
    for (int j = 0; j < seg_count[c]; j++) {
      int64_t i = s0 + j;
      if (!(lat[i] < bound)) continue;
      if (bj < 0) { bj = j; continue; }
      int64_t b = s0 + bj;
      if (better(tp[i], lat[i], batch[i], procs[i], tp[b], lat[b], batch[b], procs[b])) bj = j;
    }
    out->best[c] = (int16_t)bj;
    if (bj >= 0) any = 1;
  }
  if (!any) { out->status = PARVA_INFEASIBLE_SLO; return 0; }
  /* best_triplets sorted by size (:112); select_optimal_segment fold (:127-139) */
  otrip trips[5];
  int tc[5], n = 0;
  for (int c = 0; c < 5; c++) {
    if (out->best[c] < 0) continue;
    int64_t i = seg_start[c] + out->best[c];
    trips[n].size = SIZES[c]; trips[n].tp = tp[i]; tc[n] = c; n++;
  }
  int o = tc[oracle_select_optimal(trips, n)];
  double topt = tp[seg_start[o] + out->best[o]];
  /* match_demand (configurator.py:142-186) */
  int64_t count = 0;
  if (rate > 0) {
    double q = floor(rate / topt);
    if (!(q <= COUNT_LIMIT)) { out->status = PARVA_COUNT_OVERFLOW; out->opt_sc = (int8_t)o; return 0; }
    count = (int64_t)q;
  }
  double remaining = rate - (double)count * topt;
  double m = (1.0 > rate) ? 1.0 : rate; /* max(rate, 1.0) */
  if (remaining <= 1e-9 * m) remaining = 0.0;
  int last = -1;
  if (remaining > 0) {
    for (int k = 0; k < n; k++) {
      if (trips[k].tp >= remaining) { last = tc[k]; break; }
    }
    if (last < 0) { /* :166-176 fallback: first max-throughput triplet */
      int fb = 0;
      for (int k = 1; k < n; k++) if (trips[k].tp > trips[fb].tp) fb = k;
      if (trips[fb].tp >= remaining) last = tc[fb];
      else { out->status = PARVA_RESIDUAL_UNCOVERABLE; out->opt_sc = (int8_t)o; return 0; }
    }
  }
  out->opt_sc = (int8_t)o;
  out->last_sc = (int8_t)last;
  out->count = count;
  out->coverage = coverage(topt, count, last >= 0, last >= 0 ? tp[seg_start[last] + out->best[last]] : 0.0);
  return 0;
}

/* ========================================================== mig.py model */

typedef struct {
  int32_t name;
  otrip t;       /* size, batch, procs, tp */
  int32_t slot;
} Pl;

typedef struct {
  int64_t id;
  int32_t n;
  Pl p[8];
} Gpu;

typedef struct {
  Gpu* g;
  int32_t n, cap;
  int64_t max_id;      /* running max of ids: _next_id (allocator.py:280-281) */
} Map;

/* _START_OPTIONS (mig.py:41-54) as (start, occupied mask, blocked mask). */
typedef struct { int start, occ, blk; } Opt;
static const Opt OPT7[] = {{0, 0x7F, 0}};
static const Opt OPT4[] = {{0, 0x0F, 0}};
static const Opt OPT3[] = {{4, 0x70, 0}, {0, 0x07, 0x08}};
static const Opt OPT2[] = {{0, 0x03, 0}, {2, 0x0C, 0}, {4, 0x30, 0}};
static const Opt OPT1[] = {{0, 1, 0}, {1, 2, 0}, {2, 4, 0}, {3, 8, 0}, {4, 16, 0}, {5, 32, 0}, {6, 64, 0}};

static const Opt* options(int size, int* n) {
  switch (size) {
    case 7: *n = 1; return OPT7;
    case 4: *n = 1; return OPT4;
    case 3: *n = 2; return OPT3;
    case 2: *n = 3; return OPT2;
    case 1: *n = 7; return OPT1;
  }
  *n = 0;
  return NULL;
}

static const Opt* option_of(const Pl* p) {
  int n;
  const Opt* o = options(p->t.size, &n);
  for (int k = 0; k < n; k++) if (o[k].start == p->slot) return &o[k];
  return NULL;
}

static int num_gpcs(const Gpu* g) {
  int s = 0;
  for (int k = 0; k < g->n; k++) s += g->p[k].t.size;
  return s;
}

/* GpuState.slot_map (mig.py:100-109): -1 free, -2 blocked, else occupant. */
static void slot_map(const Gpu* g, int cells[7]) {
  for (int c = 0; c < 7; c++) cells[c] = -1;
  for (int k = 0; k < g->n; k++) {
    const Opt* o = option_of(&g->p[k]);
    for (int c = 0; c < 7; c++) {
      if (o->occ >> c & 1) cells[c] = k;
      if (o->blk >> c & 1) cells[c] = -2;
    }
  }
}

/* GpuState.find_start (mig.py:114-122). Returns start slot or -1. */
static int find_start(const Gpu* g, int size) {
  if (num_gpcs(g) + size > 7) return -1;
  int cells[7];
  slot_map(g, cells);
  int n;
  const Opt* o = options(size, &n);
  for (int k = 0; k < n; k++) {
    int fp = o[k].occ | o[k].blk, ok = 1;
    for (int c = 0; c < 7; c++) if ((fp >> c & 1) && cells[c] != -1) ok = 0;
    if (ok) return o[k].start;
  }
  return -1;
}

static int pl_eq(const Pl* a, const Pl* b) {
  return a->name == b->name && a->t.size == b->t.size && a->t.batch == b->t.batch &&
         a->t.procs == b->t.procs && a->t.tp == b->t.tp && a->slot == b->slot;
}

/* GpuState.remove (mig.py:151-158): list.remove -> first equal element. */
static int gpu_remove(Gpu* g, const Pl* p) {
  for (int k = 0; k < g->n; k++) {
    if (pl_eq(&g->p[k], p)) {
      memmove(&g->p[k], &g->p[k + 1], sizeof(Pl) * (size_t)(g->n - k - 1));
      g->n--;
      return 0;
    }
  }
  return -1;
}

static int gpu_contains(const Gpu* g, const Pl* p) {
  for (int k = 0; k < g->n; k++) if (pl_eq(&g->p[k], p)) return 1;
  return 0;
}

static void map_push(Map* m, int64_t id) {
  if (m->n == m->cap) {
    m->cap = m->cap ? m->cap * 2 : 16;
    m->g = (Gpu*)realloc(m->g, sizeof(Gpu) * (size_t)m->cap);
  }
  m->g[m->n].id = id;
  m->g[m->n].n = 0;
  m->n++;
  if (id > m->max_id) m->max_id = id;
}

/* ===================================================== allocator.py model */

/* SegmentQueues (allocator.py:32-51): FIFO per size, drained 7,4,3,2,1. */
typedef struct { int32_t name; otrip t; } QEnt;
typedef struct {
  QEnt* q[5];
  int64_t n[5], cap[5];
} Queues;

static void q_push(Queues* Q, int32_t name, const otrip* t) {
  int c = size_class(t->size);
  if (Q->n[c] == Q->cap[c]) {
    Q->cap[c] = Q->cap[c] ? Q->cap[c] * 2 : 16;
    Q->q[c] = (QEnt*)realloc(Q->q[c], sizeof(QEnt) * (size_t)Q->cap[c]);
  }
  Q->q[c][Q->n[c]].name = name;
  Q->q[c][Q->n[c]].t = *t;
  Q->n[c]++;
}

static void q_clear(Queues* Q) { for (int c = 0; c < 5; c++) Q->n[c] = 0; }
static void q_free(Queues* Q) { for (int c = 0; c < 5; c++) free(Q->q[c]); }

/* _FirstFit (allocator.py:168-281) with per-size cursors. */
typedef struct {
  Map* m;
  int32_t cursors[5];
} FirstFit;

static void note_removal(FirstFit* ff, int index) {
  for (int c = 0; c < 5; c++) if (ff->cursors[c] > index) ff->cursors[c] = index;
}

/* _FirstFit.place (:194-251).  Returns GPU index or -1; *out = placement. */
static int ff_place(FirstFit* ff, int32_t name, const otrip* t, int exclude, int allow_new, Pl* out) {
  int c = size_class(t->size);
  int i = ff->cursors[c];
  int advanced = 1;
  Map* m = ff->m;
  while (i < m->n) {
    if (i == exclude) { advanced = 0; i++; continue; }
    int st = find_start(&m->g[i], t->size);
    if (st >= 0) {
      Gpu* g = &m->g[i];
      g->p[g->n].name = name; g->p[g->n].t = *t; g->p[g->n].slot = st;
      *out = g->p[g->n];
      g->n++;
      return i;
    }
    i++;
    if (advanced) ff->cursors[c] = i;
  }
  if (!allow_new) return -1;
  map_push(m, m->max_id + 1);
  Gpu* g = &m->g[m->n - 1];
  int st = find_start(g, t->size);
  g->p[0].name = name; g->p[0].t = *t; g->p[0].slot = st;
  g->n = 1;
  *out = g->p[0];
  return m->n - 1;
}

/* _FirstFit.allocate (:253-278): all-or-nothing.  Returns #unplaced. */
static int64_t ff_allocate(FirstFit* ff, Queues* Q, int exclude, int allow_new) {
  int64_t total = 0, unplaced = 0;
  for (int c = 0; c < 5; c++) total += Q->n[c];
  int* idx = (int*)malloc(sizeof(int) * (size_t)(total + 1));
  Pl* pl = (Pl*)malloc(sizeof(Pl) * (size_t)(total + 1));
  int64_t np = 0;
  for (int c = 4; c >= 0; c--) {
    for (int64_t k = 0; k < Q->n[c]; k++) {
      Pl p;
      int r = ff_place(ff, Q->q[c][k].name, &Q->q[c][k].t, exclude, allow_new, &p);
      if (r < 0) unplaced++;
      else { idx[np] = r; pl[np] = p; np++; }
    }
  }
  q_clear(Q);
  if (unplaced) {
    for (int64_t k = np - 1; k >= 0; k--) {
      gpu_remove(&ff->m->g[idx[k]], &pl[k]);
      note_removal(ff, idx[k]);
    }
  }
  free(idx);
  free(pl);
  return unplaced;
}

/* propose_small_segments (:319-359) */
int oracle_propose(const otrip* t1, const otrip* t2, double freed, int64_t* k2out, int64_t* k1out) {
  *k2out = 0; *k1out = 0;
  if (freed <= 0) return 0;
  if (!t1 && !t2) return 1;
  int64_t max_k2 = 0;
  if (t2) max_k2 = (int64_t)ceil(freed / t2->tp - 1e-12);
  int have = 0;
  int64_t bg = 0, bc = 0, bn = 0;
  double m = (1.0 > freed) ? 1.0 : freed;
  for (int64_t k2 = 0; k2 <= max_k2; k2++) {
    double covered = t2 ? (double)k2 * t2->tp : 0.0;
    double shortv = freed - covered;
    int64_t k1;
    if (shortv <= 1e-12 * m) k1 = 0;
    else if (t1) {
      k1 = (int64_t)ceil(shortv / t1->tp - 1e-12);
      if (k1 < 1) k1 = 1;
    } else continue;
    int64_t g = 2 * k2 + k1, cn = k2 + k1, nk = -k2;
    if (!have || g < bg || (g == bg && (cn < bc || (cn == bc && nk < bn)))) {
      have = 1; bg = g; bc = cn; bn = nk;
    }
  }
  if (!have) return 1;
  *k2out = -bn;
  *k1out = bc - (-bn);
  return 0;
}

static double unallocated(const Map* m) {
  if (m->n == 0) return 0.0;
  int64_t tot = 0;
  for (int i = 0; i < m->n; i++) tot += num_gpcs(&m->g[i]);
  return 1.0 - (double)tot / (double)(7 * (int64_t)m->n);
}

static void map_clone(Map* dst, const Map* src) {
  dst->n = src->n;
  dst->cap = src->n ? src->n : 1;
  dst->g = (Gpu*)malloc(sizeof(Gpu) * (size_t)dst->cap);
  memcpy(dst->g, src->g, sizeof(Gpu) * (size_t)src->n);
  dst->max_id = src->max_id;
}

typedef struct { int64_t reason, gpu, name; } Diag;

typedef struct {
  double* val;
  int32_t* order;
  int32_t next;
  int32_t k;
} Ledger;

static int emit(const Map* m, oresult* r) {
  int64_t np = 0;
  for (int i = 0; i < m->n; i++) np += m->g[i].n;
  r->n_gpus = m->n;
  r->n_place = (int32_t)np;
  if (m->n > r->gpu_cap || np > r->place_cap) return PARVA_CAPACITY;
  int64_t k = 0;
  for (int i = 0; i < m->n; i++) {
    r->gpu_id[i] = m->g[i].id;
    r->pl_off[i] = (int32_t)k;
    for (int j = 0; j < m->g[i].n; j++, k++) {
      r->pl_name[k] = m->g[i].p[j].name;
      r->pl_trip[k] = m->g[i].p[j].t;
      r->pl_slot[k] = m->g[i].p[j].slot;
    }
  }
  r->pl_off[m->n] = (int32_t)k;
  return PARVA_OK;
}

int oracle_plan_general(const oproblem* P, oresult* r) {
  Map in = {0};
  in.max_id = -1;
  for (int g = 0; g < P->n_gpus; g++) {
    map_push(&in, P->gpu_id[g]);
    Gpu* G = &in.g[g];
    for (int k = P->pl_off[g]; k < P->pl_off[g + 1]; k++) {
      G->p[G->n].name = P->pl_name[k];
      G->p[G->n].t = P->pl_trip[k];
      G->p[G->n].slot = P->pl_slot[k];
      G->n++;
    }
  }
  r->status = PARVA_OK;
  r->fallback = 0;
  r->n_diag = 0;
  for (int k = 0; k < P->n_names; k++) {
    r->ledger_val[k] = P->ledger_val ? P->ledger_val[k] : 0.0;
    r->ledger_order[k] = P->ledger_order ? P->ledger_order[k] : 0;
  }
  Queues Q;
  memset(&Q, 0, sizeof(Q));
  /* relocate_segments (:292-316) into the given map with fresh cursors */
  if (P->relocate) {
    for (int s = 0; s < P->n_services; s++) {
      if (P->svc_opt[s].valid) for (int64_t k = 0; k < P->svc_count[s]; k++) q_push(&Q, s, &P->svc_opt[s]);
      if (P->svc_last[s].valid) q_push(&Q, s, &P->svc_last[s]);
    }
    FirstFit ff = {&in, {0, 0, 0, 0, 0}};
    ff_allocate(&ff, &Q, -1, 1);
  }
  r->n_gpus_unopt = in.n;
  int64_t unopt_place = 0;
  for (int i = 0; i < in.n; i++) unopt_place += in.g[i].n;
  r->unopt_place = (int32_t)unopt_place;
  if (!P->optimize) {
    int st = emit(&in, r);
    free(in.g);
    q_free(&Q);
    r->status = st;
    return st;
  }

  /* optimize_allocation (:362-443) */
  Map res;
  map_clone(&res, &in);
  Ledger L = {r->ledger_val, r->ledger_order, 0, P->n_names};
  for (int k = 0; k < P->n_names; k++) if (L.order[k] > L.next) L.next = L.order[k];
  double* saved_val = (double*)malloc(sizeof(double) * (size_t)(P->n_names + 1));
  int32_t* saved_ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)(P->n_names + 1));
  Diag* diags = (Diag*)malloc(sizeof(Diag) * (size_t)(res.n + 2));
  int nd = 0;
  FirstFit ff = {&res, {0, 0, 0, 0, 0}};
  for (int index = res.n - 1; index >= 0; index--) {
    Gpu* gpu = &res.g[index];
    if (gpu->n == 0 || num_gpcs(gpu) > P->threshold) continue;
    Pl drained[8];
    int nd_pl = gpu->n;
    memcpy(drained, gpu->p, sizeof(Pl) * (size_t)nd_pl);
    memcpy(saved_val, L.val, sizeof(double) * (size_t)P->n_names);
    memcpy(saved_ord, L.order, sizeof(int32_t) * (size_t)P->n_names);
    int32_t saved_next = L.next;
    int32_t saved_cur[5];
    memcpy(saved_cur, ff.cursors, sizeof(saved_cur));
    q_clear(&Q);
    int failure = -1;
    int64_t fname = -1;
    for (int k = 0; k < nd_pl; k++) {
      const Pl* pl = &drained[k];
      int s = pl->name < P->n_services ? pl->name : -1; /* services_by_id.get */
      if (s < 0) { failure = PARVA_DIAG_UNKNOWN_SERVICE; fname = pl->name; break; }
      if (L.order[s] == 0) { L.order[s] = ++L.next; L.val[s] = 0.0 + pl->t.tp; }
      else L.val[s] = L.val[s] + pl->t.tp;
      gpu_remove(gpu, pl);
      const otrip* t1 = P->svc_best[s * 5 + 0].valid ? &P->svc_best[s * 5 + 0] : NULL;
      const otrip* t2 = P->svc_best[s * 5 + 1].valid ? &P->svc_best[s * 5 + 1] : NULL;
      int64_t k2, k1;
      if (oracle_propose(t1, t2, L.val[s], &k2, &k1)) {
        failure = PARVA_DIAG_SMALL_UNAVAILABLE; fname = s; break;
      }
      for (int64_t j = 0; j < k2; j++) { L.val[s] -= t2->tp; q_push(&Q, s, t2); }
      for (int64_t j = 0; j < k1; j++) { L.val[s] -= t1->tp; q_push(&Q, s, t1); }
    }
    if (failure < 0) {
      note_removal(&ff, index);
      if (ff_allocate(&ff, &Q, index, 0)) { failure = PARVA_DIAG_NEED_NEW_GPU; fname = -1; }
    }
    if (failure >= 0) {
      for (int k = 0; k < nd_pl; k++)
        if (!gpu_contains(gpu, &drained[k])) gpu->p[gpu->n++] = drained[k];
      memcpy(L.val, saved_val, sizeof(double) * (size_t)P->n_names);
      memcpy(L.order, saved_ord, sizeof(int32_t) * (size_t)P->n_names);
      L.next = saved_next;
      memcpy(ff.cursors, saved_cur, sizeof(saved_cur));
      diags[nd].reason = failure; diags[nd].gpu = gpu->id; diags[nd].name = fname; nd++;
    }
  }
  /* compaction (:423): drop empty GPUs, ids kept */
  int w = 0;
  for (int i = 0; i < res.n; i++) if (res.g[i].n) res.g[w++] = res.g[i];
  res.n = w;
  int st = PARVA_OK;
  if (res.n > in.n || unallocated(&res) > unallocated(&in) + 1e-12) {
    /* regression fallback (:428-435): input map, input ledger, one diagnostic */
    r->fallback = 1;
    for (int k = 0; k < P->n_names; k++) {
      r->ledger_val[k] = P->ledger_val ? P->ledger_val[k] : 0.0;
      r->ledger_order[k] = P->ledger_order ? P->ledger_order[k] : 0;
    }
    st = emit(&in, r);
    if (r->diag_cap < 1) st = PARVA_CAPACITY;
    else { r->diag[0] = PARVA_DIAG_REGRESSED; r->diag[1] = -1; r->diag[2] = -1; r->n_diag = 1; }
  } else {
    st = emit(&res, r);
    r->n_diag = nd;
    if (nd > r->diag_cap) st = PARVA_CAPACITY;
    else for (int k = 0; k < nd; k++) {
      r->diag[3 * k] = diags[k].reason; r->diag[3 * k + 1] = diags[k].gpu; r->diag[3 * k + 2] = diags[k].name;
    }
    /* coverage assert (:437-442): service_throughput in map order */
    if (st == PARVA_OK) {
      double* after = (double*)calloc((size_t)P->n_services + 1, sizeof(double));
      char* seen = (char*)calloc((size_t)P->n_services + 1, 1);
      for (int i = 0; i < res.n; i++)
        for (int j = 0; j < res.g[i].n; j++) {
          int s = res.g[i].p[j].name;
          if (s < P->n_services) { after[s] = (seen[s] ? after[s] : 0.0) + res.g[i].p[j].t.tp; seen[s] = 1; }
        }
      for (int s = 0; s < P->n_services; s++)
        if (P->svc_rate[s] > 0 && seen[s] && !(after[s] >= P->svc_rate[s] * (1 - 1e-9))) st = PARVA_COVERAGE_ASSERT;
      free(after);
      free(seen);
    }
  }
  r->status = st;
  free(saved_val);
  free(saved_ord);
  free(diags);
  free(in.g);
  free(res.g);
  q_free(&Q);
  return st;
}

/* ======================================================== pipeline.py */

static int tab_args(const int64_t* seg_start, int t, int64_t ss[5]) {
  for (int c = 0; c < 5; c++) ss[c] = seg_start[t * 5 + c];
  return 0;
}

static otrip trip_of(const double* tp, const double* lat, const int32_t* batch, const int32_t* procs,
                     int64_t i, int c) {
  otrip t;
  t.size = SIZES[c]; t.batch = batch[i]; t.procs = procs[i]; t.tp = tp[i]; t.lat = lat[i]; t.valid = 1;
  return t;
}

int oracle_plan_scenario(const double* tp, const double* lat, const int32_t* batch,
                         const int32_t* procs, const int64_t* seg_start,
                         const int32_t* seg_count, int32_t n_svc,
                         const int32_t* svc_table, const double* svc_rate,
                         const double* svc_bound, int32_t optimize, int32_t threshold,
                         parva_config_record* cfg, oresult* r) {
  /* configure_service x N in input order (pipeline.py:96) */
  int first_err = -1, err_status = 0;
  for (int s = 0; s < n_svc; s++) {
    int64_t ss[5];
    tab_args(seg_start, svc_table[s], ss);
    oracle_configure(tp, lat, batch, procs, ss, seg_count + svc_table[s] * 5, svc_bound[s], svc_rate[s], &cfg[s]);
    if (cfg[s].status != PARVA_OK && first_err < 0) { first_err = s; err_status = cfg[s].status; }
  }
  r->n_gpus = r->n_place = r->n_diag = r->n_gpus_unopt = r->fallback = 0;
  if (first_err >= 0) { r->status = err_status; return err_status; }
  otrip* best = (otrip*)calloc((size_t)n_svc * 5 + 1, sizeof(otrip));
  otrip* opt = (otrip*)calloc((size_t)n_svc + 1, sizeof(otrip));
  otrip* last = (otrip*)calloc((size_t)n_svc + 1, sizeof(otrip));
  int64_t* count = (int64_t*)calloc((size_t)n_svc + 1, sizeof(int64_t));
  for (int s = 0; s < n_svc; s++) {
    int t = svc_table[s];
    for (int c = 0; c < 5; c++)
      if (cfg[s].best[c] >= 0) best[s * 5 + c] = trip_of(tp, lat, batch, procs, seg_start[t * 5 + c] + cfg[s].best[c], c);
    opt[s] = best[s * 5 + cfg[s].opt_sc];
    if (cfg[s].last_sc >= 0) last[s] = best[s * 5 + cfg[s].last_sc];
    count[s] = cfg[s].count;
  }
  oproblem P;
  memset(&P, 0, sizeof(P));
  P.n_names = n_svc; P.n_services = n_svc;
  P.svc_best = best; P.svc_opt = opt; P.svc_count = count; P.svc_last = last; P.svc_rate = svc_rate;
  int32_t zero = 0;
  P.n_gpus = 0; P.pl_off = &zero;
  P.relocate = 1; P.optimize = optimize; P.threshold = threshold;
  int st = oracle_plan_general(&P, r);
  free(best); free(opt); free(last); free(count);
  return st;
}

/* Encode a general result into the fast-path record (parva_b200.h). */
static void encode_record(const oresult* r, int n_svc, int cfg_err, int err_svc, parva_plan_record* rec) {
  memset(rec, 0, sizeof(*rec));
  if (n_svc > PARVA_PLAN_MAX_SERVICES) { rec->status = PARVA_CAPACITY; return; }
  if (cfg_err) { rec->status = (uint8_t)cfg_err; rec->err_service = (uint8_t)err_svc; return; }
  if (r->n_gpus_unopt > PARVA_PLAN_MAX_GPUS || r->status == PARVA_CAPACITY) { rec->status = PARVA_CAPACITY; return; }
  if (r->status != PARVA_OK) { rec->status = (uint8_t)r->status; return; }
  int nd = r->fallback ? 0 : r->n_diag;
  int nl = 0;
  if (!r->fallback)
    for (int s = 0; s < n_svc; s++) if (r->ledger_order[s]) nl++;
  int np = r->n_place;
  int led_off = (2 * (np + nd) + 7) & ~7;
  if (led_off + 10 * nl > PARVA_PLAN_PAYLOAD) { rec->status = PARVA_CAPACITY; return; }
  rec->n_gpus = (uint8_t)r->n_gpus;
  rec->n_gpus_unopt = (uint8_t)r->n_gpus_unopt;
  rec->n_place = (uint8_t)np;
  rec->n_diag = (uint8_t)nd;
  rec->n_ledger = (uint8_t)nl;
  rec->flags = r->fallback ? PARVA_FLAG_FALLBACK : 0;
  uint16_t u;
  for (int g = 0; g < r->n_gpus; g++)
    for (int k = r->pl_off[g]; k < r->pl_off[g + 1]; k++) {
      int cat = r->pl_name[k] * 5 + size_class(r->pl_trip[k].size);
      u = (uint16_t)(r->gpu_id[g] << 11 | cat << 3 | r->pl_slot[k]);
      memcpy(rec->payload + 2 * k, &u, 2);
    }
  for (int k = 0; k < nd; k++) {
    u = (uint16_t)(r->diag[3 * k + 1] << 7 | r->diag[3 * k] << 5 | (r->diag[3 * k + 2] < 0 ? 0 : r->diag[3 * k + 2]));
    memcpy(rec->payload + 2 * (np + k), &u, 2);
  }
  if (!r->fallback)
    for (int s = 0; s < n_svc; s++) {
      int o = r->ledger_order[s];
      if (!o) continue;
      memcpy(rec->payload + led_off + 8 * (o - 1), &r->ledger_val[s], 8);
      u = (uint16_t)(s | o << 8);
      memcpy(rec->payload + led_off + 8 * nl + 2 * (o - 1), &u, 2);
    }
}

int oracle_plan_batch_records(const double* tp, const double* lat, const int32_t* batch,
                              const int32_t* procs, const int64_t* seg_start,
                              const int32_t* seg_count, int32_t n_scen,
                              const int32_t* scen_off, const int32_t* svc_table,
                              const double* svc_rate, const double* svc_bound,
                              int32_t optimize, int32_t threshold,
                              parva_config_record* cfg, parva_plan_record* plan, int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel
#endif
  {
    enum { GCAP = 4096, PCAP = 4096 * 7, DCAP = 4096 };
    oresult r;
    memset(&r, 0, sizeof(r));
    r.gpu_cap = GCAP; r.place_cap = PCAP; r.diag_cap = DCAP;
    r.gpu_id = (int64_t*)malloc(sizeof(int64_t) * GCAP);
    r.pl_off = (int32_t*)malloc(sizeof(int32_t) * (GCAP + 1));
    r.pl_name = (int32_t*)malloc(sizeof(int32_t) * PCAP);
    r.pl_trip = (otrip*)malloc(sizeof(otrip) * PCAP);
    r.pl_slot = (int32_t*)malloc(sizeof(int32_t) * PCAP);
    r.diag = (int64_t*)malloc(sizeof(int64_t) * 3 * DCAP);
    int maxs = 1;
    for (int k = 0; k < n_scen; k++) if (scen_off[k + 1] - scen_off[k] > maxs) maxs = scen_off[k + 1] - scen_off[k];
    r.ledger_val = (double*)malloc(sizeof(double) * (size_t)maxs);
    r.ledger_order = (int32_t*)malloc(sizeof(int32_t) * (size_t)maxs);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
    for (int k = 0; k < n_scen; k++) {
      int a = scen_off[k], n = scen_off[k + 1] - a;
      oracle_plan_scenario(tp, lat, batch, procs, seg_start, seg_count, n, svc_table + a,
                           svc_rate + a, svc_bound + a, optimize, threshold, cfg + a, &r);
      int cfg_err = 0, err_svc = 0;
      for (int s = 0; s < n; s++) if (cfg[a + s].status) { cfg_err = cfg[a + s].status; err_svc = s; break; }
      encode_record(&r, n, cfg_err, err_svc, &plan[k]);
    }
    free(r.gpu_id); free(r.pl_off); free(r.pl_name); free(r.pl_trip); free(r.pl_slot); free(r.diag);
    free(r.ledger_val); free(r.ledger_order);
  }
  return 0;
}

int oracle_configure_batch(const double* tp, const double* lat, const int32_t* batch,
                           const int32_t* procs, const int64_t* seg_start,
                           const int32_t* seg_count, int32_t n_q, const int32_t* q_table,
                           const double* q_rate, const double* q_bound,
                           parva_config_record* out, int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int q = 0; q < n_q; q++) {
    int t = q_table[q];
    oracle_configure(tp, lat, batch, procs, seg_start + t * 5, seg_count + t * 5, q_bound[q], q_rate[q], &out[q]);
  }
  return 0;
}

/* ------------------------------------------------------------ simulator */
/* One service of run_simulation's event loop (evaluation.py:337-416),
 * restated with a binary heap of (time, seq, kind, payload) as in the
 * reference (heapq, evaluation.py:341-349).  Arrivals in ms, sorted. */
typedef struct { double t; int64_t seq; int kind; int payload; } sim_ev;

static int ev_less(const sim_ev* a, const sim_ev* b) {
  if (a->t != b->t) return a->t < b->t;
  return a->seq < b->seq;
}

static void heap_push(sim_ev* h, int* n, sim_ev e) {
  int i = (*n)++;
  h[i] = e;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!ev_less(&h[i], &h[p])) break;
    sim_ev tmp = h[i]; h[i] = h[p]; h[p] = tmp; i = p;
  }
}

static sim_ev heap_pop(sim_ev* h, int* n) {
  sim_ev top = h[0];
  h[0] = h[--(*n)];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < *n && ev_less(&h[l], &h[m])) m = l;
    if (r < *n && ev_less(&h[r], &h[m])) m = r;
    if (m == i) break;
    sim_ev tmp = h[i]; h[i] = h[m]; h[m] = tmp; i = m;
  }
  return top;
}

typedef struct {
  const double* arr; int64_t na; const double* seg_ms; const int32_t* seg_batch; double slo, horizon;
  sim_ev* heap; int nh; int* free_seg; int free_lanes, wake;
  int64_t seq, ptr, qh, served, batches, viol;
  double* lat; double* busy;
} sim_state;

/* schedule_wakeup (evaluation.py:362-366) */
static void sim_wakeup(sim_state* S) {
  if (S->wake || S->ptr >= S->na) return;
  S->wake = 1;
  sim_ev e = {S->arr[S->ptr], S->seq++, 1, 0};
  heap_push(S->heap, &S->nh, e);
}

/* ingest (evaluation.py:353-360): searchsorted(side="right") on a monotone clock */
static void sim_ingest(sim_state* S, double now) {
  while (S->ptr < S->na && S->arr[S->ptr] <= now) S->ptr++;
}

/* dispatch (evaluation.py:368-388) */
static void sim_dispatch(sim_state* S, double now) {
  if (now >= S->horizon) return;
  while (S->qh < S->ptr && S->free_lanes > 0) {
    int g = 0;
    while (S->free_seg[g] == 0) g++;
    int64_t n = S->ptr - S->qh < S->seg_batch[g] ? S->ptr - S->qh : S->seg_batch[g];
    double first = S->arr[S->qh];
    S->qh += n;
    double wait = now - first;
    double latency = wait + S->seg_ms[g];
    S->lat[S->batches++] = latency;
    S->served += n;
    if (latency > S->slo) S->viol++;
    S->free_seg[g]--;
    S->free_lanes--;
    double rem = S->horizon - now;
    double m = S->seg_ms[g] <= rem ? S->seg_ms[g] : rem;
    S->busy[g] += m > 0.0 ? m : 0.0;
    sim_ev c = {now + S->seg_ms[g], S->seq++, 0, g};
    heap_push(S->heap, &S->nh, c);
  }
}

int oracle_simulate_service(int64_t na, const double* arr, int32_t ns, const double* seg_ms,
                            const int32_t* seg_batch, const int32_t* seg_lanes, double slo, double horizon_ms,
                            int64_t* served_o, int64_t* batches_o, int64_t* viol_o, double* lat, double* busy) {
  int cap = 1;
  for (int g = 0; g < ns; g++) cap += seg_lanes[g];
  sim_state S = {0};
  S.arr = arr; S.na = na; S.seg_ms = seg_ms; S.seg_batch = seg_batch; S.slo = slo; S.horizon = horizon_ms;
  S.heap = (sim_ev*)malloc(sizeof(sim_ev) * (size_t)(cap + 1));
  S.free_seg = (int*)malloc(sizeof(int) * (size_t)(ns + 1));
  S.lat = lat; S.busy = busy;
  for (int g = 0; g < ns; g++) { S.free_seg[g] = seg_lanes[g]; S.free_lanes += seg_lanes[g]; busy[g] = 0.0; }
  if (ns > 0) sim_wakeup(&S);
  /* main loop (evaluation.py:395-416) */
  while (S.nh > 0) {
    sim_ev e = heap_pop(S.heap, &S.nh);
    if (e.kind == 0) {
      S.free_seg[e.payload]++;
      S.free_lanes++;
      if (e.t < horizon_ms) {
        sim_ingest(&S, e.t);
        sim_dispatch(&S, e.t);
        if (S.qh == S.ptr) sim_wakeup(&S);
      }
    } else {
      S.wake = 0;
      sim_ingest(&S, e.t);
      sim_dispatch(&S, e.t);
      if (S.free_lanes > 0) sim_wakeup(&S);
    }
  }
  free(S.heap);
  free(S.free_seg);
  *served_o = S.served; *batches_o = S.batches; *viol_o = S.viol;
  return 0;
}
