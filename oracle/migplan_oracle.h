/*
 * migplan_oracle.h — CPU restatement of the reference planner's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2409_14447_b200/ links, loads
 * or calls this; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, as the checker.  Parity of this
 * oracle is pinned against golden vectors rendered from the reference itself
 * (tests/golden/make_golden.py -> tests/test_oracle_golden.py).
 *
 * Every function restates a reference function (file:line into
 * /root/reference/pkg/src/migplan/), following its control flow, including
 * the first-fit cursors, list-equality removal and the restore-by-append of
 * drained placements.
 */
#ifndef MIGPLAN_ORACLE_H
#define MIGPLAN_ORACLE_H
#include <stdint.h>
#include "../include/parva_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t size, batch, procs;
  double tp, lat;
  int32_t valid;
} otrip;

/* A general planning problem (host arrays). */
typedef struct {
  int32_t n_names, n_services;
  const otrip* svc_best;      /* [n_services*5] by size class; valid=0 if absent */
  const otrip* svc_opt;       /* [n_services] valid=0 -> None                   */
  const int64_t* svc_count;   /* [n_services]                                   */
  const otrip* svc_last;      /* [n_services]                                   */
  const double* svc_rate;     /* [n_services]                                   */
  int32_t n_gpus;             /* initial map                                    */
  const int64_t* gpu_id;
  const int32_t* pl_off;      /* [n_gpus+1]                                     */
  const int32_t* pl_name;
  const otrip* pl_trip;       /* size, batch, procs, tp (lat ignored)           */
  const int32_t* pl_slot;
  const double* ledger_val;   /* [n_names]                                      */
  const int32_t* ledger_order;
  int32_t relocate, optimize, threshold;
} oproblem;

typedef struct {
  int32_t status, n_gpus, n_gpus_unopt, n_place, n_diag, fallback;
  int32_t gpu_cap, place_cap, diag_cap;
  int64_t* gpu_id;
  int32_t* pl_off;
  int32_t* pl_name;
  otrip* pl_trip;
  int32_t* pl_slot;
  int64_t* diag;              /* [diag_cap*3] reason, gpu id, name */
  double* ledger_val;         /* [n_names] */
  int32_t* ledger_order;
  /* unoptimized map (relocation result) */
  int32_t unopt_place;
} oresult;

/* configure_service (configurator.py:189-191) over one prepared table given
 * as 5 size-class segments of key-ordered points. */
int oracle_configure(const double* tp, const double* lat, const int32_t* batch,
                     const int32_t* procs, const int64_t* seg_start,
                     const int32_t* seg_count, double bound, double rate,
                     parva_config_record* out);

/* select_optimal_segment (configurator.py:127-139): index of the chosen triplet. */
int oracle_select_optimal(const otrip* t, int32_t n);

/* propose_small_segments (allocator.py:319-359): returns 0 ok (k2,k1 set),
 * 1 SmallSegmentsUnavailableError. */
int oracle_propose(const otrip* t1, const otrip* t2, double freed, int64_t* k2, int64_t* k1);

/* Python 3.12 builtin sum() over floats (start 0). */
double oracle_pysum(const double* x, int64_t n);

/* relocate_segments / optimize_allocation on a general problem. */
int oracle_plan_general(const oproblem* p, oresult* r);

/* plan_services over prepared tables for one scenario.  Writes n_svc config
 * records; runs the allocator only if every service configured. */
int oracle_plan_scenario(const double* tp, const double* lat, const int32_t* batch,
                         const int32_t* procs, const int64_t* seg_start,
                         const int32_t* seg_count, int32_t n_svc,
                         const int32_t* svc_table, const double* svc_rate,
                         const double* svc_bound, int32_t optimize, int32_t threshold,
                         parva_config_record* cfg, oresult* r);

/* Batched plan_services in the parva record format (same encoding as the
 * CUDA fast path, including PARVA_CAPACITY), OpenMP over scenarios. */
int oracle_plan_batch_records(const double* tp, const double* lat, const int32_t* batch,
                              const int32_t* procs, const int64_t* seg_start,
                              const int32_t* seg_count, int32_t n_scen,
                              const int32_t* scen_off, const int32_t* svc_table,
                              const double* svc_rate, const double* svc_bound,
                              int32_t optimize, int32_t threshold,
                              parva_config_record* cfg, parva_plan_record* plan, int32_t n_threads);

/* configure_service for many (table, rate, bound) queries, OpenMP. */
int oracle_configure_batch(const double* tp, const double* lat, const int32_t* batch,
                           const int32_t* procs, const int64_t* seg_start,
                           const int32_t* seg_count, int32_t n_q, const int32_t* q_table,
                           const double* q_rate, const double* q_bound,
                           parva_config_record* out, int32_t n_threads);

/* run_simulation event loop for one service (evaluation.py:337-416) */
int oracle_simulate_service(int64_t na, const double* arr, int32_t ns, const double* seg_ms,
                            const int32_t* seg_batch, const int32_t* seg_lanes, double slo, double horizon_ms,
                            int64_t* served_o, int64_t* batches_o, int64_t* viol_o, double* lat, double* busy);

#ifdef __cplusplus
}
#endif

#endif
