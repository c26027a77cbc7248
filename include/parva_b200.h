/*
 * parva_b200.h — C ABI of the B200-native ParvaGPU scheduling hot path.
 *
 * The reference (arXiv 2409.14447's `migplan`, pure Python) has no FFI; its
 * drop-in boundary is the Python API in pkg/src/migplan/__init__.py:12-74.
 * Each entry point below replaces a batch of calls to that API:
 *
 *   parva_configure_sweep  <- configure_service(service, table) per query
 *                             (configurator.py:189-191 = decide_best_triplets
 *                             :93-124 + select_optimal_segment :127-139 +
 *                             match_demand :142-186)
 *   parva_build_index      <- (no reference equivalent) latency-sorted
 *                             prefix-argmax index of prepared tables, so
 *                             many queries per table cost O(log n)
 *   parva_plan_batch       <- plan_services(services, tables, options) per
 *                             scenario, timed region pipeline.py:95-103:
 *                             configure -> relocate_segments
 *                             (allocator.py:292-316) -> optimize_allocation
 *                             (allocator.py:362-443)
 *   parva_plan_general     <- relocate_segments / optimize_allocation on
 *                             arbitrary service sets and DeploymentMaps
 *                             (no size limits; also the overflow path of
 *                             parva_plan_batch)
 *
 * All pointers named d_* are device pointers; `stream` is a cudaStream_t
 * (void* here so the header needs no CUDA include).  Calls are
 * stream-ordered and asynchronous; they return a parva_status for argument
 * errors and launch failures only — per-row results are in the records.
 * parva_plan_host is the host-buffer convenience entry (copies inside).
 * No entry allocates device memory except through the caller's workspace.
 */
#ifndef PARVA_B200_H
#define PARVA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARVA_ABI_VERSION 1

/* instance sizes by size class c: 1, 2, 3, 4, 7 GPCs (mig.py:19) */
#define PARVA_NUM_SIZES 5

/* per-row status codes */
enum parva_status {
  PARVA_OK = 0,
  PARVA_INFEASIBLE_SLO = 1,        /* InfeasibleSLOError (configurator.py:110-111)   */
  PARVA_RESIDUAL_UNCOVERABLE = 2,  /* ResidualUncoverableError (configurator.py:173)  */
  PARVA_COUNT_OVERFLOW = 3,        /* rate/throughput not a finite int64 (math.floor)   */
  PARVA_CAPACITY = 4,              /* fast-path record limits exceeded: re-plan general */
  PARVA_BAD_INPUT = 5,
  PARVA_COVERAGE_ASSERT = 6,       /* optimize coverage assert (allocator.py:437-442)   */
  PARVA_LAUNCH_ERROR = 7,
  PARVA_SPILLED = 8                /* 64-byte record: full record is in the spill list */
};

/* diagnostic reasons (allocator.py:394,401,410-412,432-434) */
enum parva_diag_reason {
  PARVA_DIAG_SMALL_UNAVAILABLE = 0, /* "service 'x' has no size-1 or size-2 triplet"      */
  PARVA_DIAG_NEED_NEW_GPU = 1,      /* "replacements for GPU g would need a new GPU; ..." */
  PARVA_DIAG_UNKNOWN_SERVICE = 2,   /* "unknown service 'x'"                               */
  PARVA_DIAG_REGRESSED = 3          /* "optimization regressed GPU count or ..."          */
};

/* Prepared profile tables (filter_feasible + optional restrict applied,
 * pipeline.py:70-80), structure of arrays grouped by (table, size class):
 * segment s = t*5 + c holds points [seg_start[s], seg_start[s] + seg_count[s])
 * in key order (batch asc, procs asc; profiles.py:98-100).  Within a segment
 * the point's position is its tie-break rank, so no key array is read.  A
 * point is 16 bytes: (throughput rps, latency ms) interleaved, so every point
 * starts 16-byte aligned and a segment streams as one contiguous range.
 * d_pts must hold 2 extra doubles of padding. */
typedef struct {
  const double*  d_pts;       /* (tp, lat) pairs        [2 * n_points] */
  const int64_t* d_seg_start; /* [n_tables * 5]                    */
  const int32_t* d_seg_count; /* [n_tables * 5]                    */
  int32_t n_tables;
  int64_t n_points;
  int32_t max_seg_points;     /* max of seg_count (PARVA_CFG_TINY needs <= 254) */
} parva_tables;

/* Raw (unprepared) tables, same grouping: every point of the source
 * ProfileTable, with the fields the preparation predicates read. */
typedef struct {
  const double*  d_tp;
  const double*  d_lat;
  const double*  d_mem;       /* memory_required, GB   [n_points] */
  const int32_t* d_procs;     /* process_count         [n_points] */
  const int64_t* d_seg_start; /* [n_tables * 5]                    */
  const int32_t* d_seg_count; /* [n_tables * 5]                    */
  int32_t n_tables;
  int64_t n_points;
} parva_raw_tables;

/* Latency-sorted prefix-argmax index over the same segments (same offsets).
 * lat_sorted[seg_start[s] + j] ascending; best[seg_start[s] + j] is the
 * within-segment position of the argmax of the first j+1 sorted points under
 * (tp desc, lat asc, position asc). */
typedef struct {
  double*   d_lat_sorted;     /* [n_points + 2]                  */
  uint16_t* d_best;           /* [n_points + 8]                  */
  double*   d_tp;             /* [n_points + 2] tp in key order  */
} parva_index;

/* 32-byte per-service configuration record (a Service after match_demand). */
typedef struct {
  int16_t best[PARVA_NUM_SIZES]; /* within-segment point position, -1 = size absent */
  int8_t  opt_sc;                /* optimal_segment size class, -1 = none           */
  int8_t  last_sc;               /* last_segment size class, -1 = none              */
  uint8_t status;                /* parva_status                                    */
  uint8_t flags;
  int16_t reserved;
  int64_t count;                 /* optimal_segment_count                           */
  double  coverage;              /* Service.coverage (Python 3.12 sum, Neumaier)    */
} parva_config_record;

/* 16-byte compact config record (host transfers; parva_plan_host).  count
 * saturates at 65535 with flags bit0 set (such a service cannot fit the fast
 * path's record anyway).  Coverage is not carried: Service.coverage is a
 * property of the decoded segments (configurator.py:60-62). */
typedef struct {
  int16_t  best[PARVA_NUM_SIZES];
  int8_t   opt_sc;
  int8_t   last_sc;
  uint8_t  status;
  uint8_t  flags;               /* bit0: count saturated */
  uint16_t count;
} parva_config_compact;

/* 8-byte tiny config record, for tables with at most 254 points per
 * (table, size) -- every entry rejects PARVA_CFG_TINY with PARVA_BAD_INPUT
 * when tables->max_seg_points > 254: best[c] = 255 if absent; opt_last = opt | last << 4 (15 =
 * none); status_flags = status | 0x80 if count > 255 (count saturates at
 * 255 -- more than 224 segments cannot fit the fast path anyway). */
typedef struct {
  uint8_t best[PARVA_NUM_SIZES];
  uint8_t opt_last;
  uint8_t status_flags;
  uint8_t count;
} parva_config_tiny;

#define PARVA_CFG_FULL 0
#define PARVA_CFG_COMPACT 1
#define PARVA_CFG_TINY 2

/* 128-byte per-scenario plan record (fast path: <=32 services, <=32 GPUs).
 * Header (8 B), then a packed 120-byte payload:
 *   u16 place[n_place]   gpu << 11 | cat << 3 | slot, cat = service*5 + size class
 *   u16 diag[n_diag]     gpu << 7 | reason << 5 | service
 *   (pad to 8 B)  f64 ledger_val[n_ledger]  u16 ledger_key[n_ledger]
 *                 ledger_key = service | rank << 8; entry i has rank i+1
 *                 (freed_rate insertion order, allocator.py:396)
 * Anything that does not fit 120 B reports PARVA_CAPACITY and is re-planned
 * by the general kernel.  GPU ids equal relocation indices
 * (allocator.py:280-281 on a fresh map); placements are listed GPU by GPU
 * in final-map order, each GPU's list in list order. */
#define PARVA_PLAN_PAYLOAD 120
#define PARVA_PLAN_MAX_GPUS 32
#define PARVA_PLAN_MAX_SERVICES 32
#define PARVA_FLAG_FALLBACK 1u   /* regression fallback: map = relocation result */

typedef struct {
  uint8_t  status;
  uint8_t  err_service;   /* scenario-local index of the first failing service */
  uint8_t  n_gpus;        /* final map                                         */
  uint8_t  n_gpus_unopt;  /* PlanResult.unoptimized_gpu_count (pipeline.py:98) */
  uint8_t  n_place;
  uint8_t  n_diag;
  uint8_t  n_ledger;
  uint8_t  flags;
  uint8_t  payload[PARVA_PLAN_PAYLOAD];
} parva_plan_record;

/* ---------------------------------------------------------------- entries */

int parva_abi_version(void);

/* Device bytes of workspace parva_plan_batch needs (0 today; reserved). */
size_t parva_plan_batch_workspace(int32_t n_scenarios, int32_t n_services);

/* prepare_tables (pipeline.py:70-80) on the device: filter_feasible
 * (profiles.py:260-271, memory_required <= h_memcap5[size class]) and, if
 * single_process, restrict(process_counts=(1,)) (profiles.py:115-129).
 * Writes the prepared layout into caller-allocated device arrays (capacity
 * raw->n_points; d_pts 2*n_points + 2 doubles), d_src = raw index of each
 * kept point; *h_n_points = prepared count (synchronizes `stream`). */
int parva_prepare_tables(const parva_raw_tables* raw, const double* h_memcap5,
                         int32_t single_process, double* d_pts, int64_t* d_seg_start,
                         int32_t* d_seg_count, int32_t* d_src, int64_t* h_n_points,
                         void* stream);

/* Build the prefix-argmax index of `tables` into `index` (both device). */
int parva_build_index(const parva_tables* tables, parva_index* index, void* stream);

/* One query per row: table id, request rate, internal latency bound
 * (Service.internal_latency = slo / 2 by default, configurator.py:87-89).
 * Streams each queried table once from HBM; HBM-bound. */
int parva_configure_sweep(const parva_tables* tables, int32_t n_queries,
                          const int32_t* d_q_table, const double* d_q_rate,
                          const double* d_q_bound, parva_config_record* d_out,
                          void* stream);

/* Plan n_scenarios independent scenarios.  Scenario k owns services
 * [d_scen_off[k], d_scen_off[k+1]); service i queries table d_svc_table[i];
 * n_services = d_scen_off[n_scenarios] - d_scen_off[0].  Two launches: every
 * service is configured by one thread, then one warp plans each scenario.
 * Writes one config record per service (parva_config_record, or
 * parva_config_compact when cfg_format == PARVA_CFG_COMPACT) and one plan
 * record per scenario.  index must have been built from tables. */
int parva_plan_batch(const parva_tables* tables, const parva_index* index,
                     int32_t n_scenarios, int32_t n_services, const int32_t* d_scen_off,
                     const int32_t* d_svc_table, const double* d_svc_rate,
                     const double* d_svc_bound, int32_t optimize, int32_t threshold,
                     void* d_cfg, int32_t cfg_format, parva_plan_record* d_plan,
                     void* stream);

/* Output-slot ticket of an overlapped launch.  A caller that keeps several
 * launches in flight rotates their outputs over slots; each slot owns a u64
 * completion counter in device memory (zeroed before first use) to which
 * every CTA of a launch into the slot adds its scenario count after its last
 * store (one release reduction).  Before its first store every CTA waits
 * until the counter has reached wait_count -- the scenarios of all earlier
 * launches into the slot -- so launches into one slot never overlap, however
 * many grids are in flight, while consecutive slots still overlap freely.  A
 * wait longer than 60 s (environment PARVA_TICKET_TIMEOUT_MS overrides)
 * stores PARVA_LAUNCH_ERROR into *d_err (if non-NULL) and the CTA stores
 * nothing (no hang). */
typedef struct {
  unsigned long long* d_count;     /* the slot's completion counter (device)         */
  unsigned long long wait_count;   /* scenarios of the earlier launches into the slot */
  int32_t* d_err;                  /* optional error word (device)                   */
} parva_slot_ticket;

/* parva_plan_batch as a programmatic dependent launch: it may start while
 * the previous call on `stream` is still planning its last scenarios (its
 * CTAs take SM slots as the predecessor's retire), so back-to-back batches
 * leave no idle tail.  `ticket` (required) serializes launches that share
 * an output slot: d_cfg / d_plan belong to the ticket's slot.  Inputs must
 * stay unmodified until the launch completes. */
int parva_plan_batch_overlapped(const parva_tables* tables, const parva_index* index,
                                int32_t n_scenarios, int32_t n_services, const int32_t* d_scen_off,
                                const int32_t* d_svc_table, const double* d_svc_rate,
                                const double* d_svc_bound, int32_t optimize, int32_t threshold,
                                void* d_cfg, int32_t cfg_format, parva_plan_record* d_plan,
                                const parva_slot_ticket* ticket, void* stream);

/* Fused all-gather for the sharded device path (one process per GPU,
 * SURVEY §8e; replaces plan_services per scenario plus the NCCL all-gather
 * of the per-scenario plans).  Every rank owns one gathered buffer with
 * n_slots slots; slot s holds every rank's [plan | config | overflow]
 * sections and, in a header, a flag row (rank r's last landed epoch of the
 * slot) and an ack row (rank r's last released epoch of the slot).
 * parva_plan_batch_fused plans this rank's shard and, tile by tile while the
 * other CTAs keep planning, stores the tile's records into this rank's
 * sections of the slot on every rank (NVLink P2P stores into buffers mapped
 * by CUDA IPC).  With plan_bytes == 64 the records are 64-byte plan records
 * (the 128-byte record truncated to 56 payload bytes; a scenario whose
 * payload does not fit has status PARVA_SPILLED and its full record at the
 * same index of the overflow section) -- 152 B per C2 scenario on the wire
 * instead of 216.  Before its first store every CTA waits for the slot's
 * ticket (this rank's earlier launches into the slot have completed) and for
 * every rank's release of the slot's previous epoch (d_acks[m] >=
 * prev_epoch); after a system-scope fence the last CTA (d_done) stores the
 * epoch into this rank's flag word of the slot on every rank.  The call is
 * rejected (PARVA_BAD_INPUT) when the records would not fit the sections
 * (n_scenarios * plan_bytes > plan_capacity, n_services * config record
 * bytes > cfg_capacity, or n_scenarios * 128 > spill_capacity). */
typedef struct {
  int32_t n;               /* ranks, 1..8                                      */
  int32_t overlap;         /* launch as a programmatic dependent launch        */
  void* plan[8];           /* this rank's plan section of the slot on rank m  */
  void* cfg[8];            /* its config section                               */
  void* spill[8];          /* its overflow section (plan_bytes == 64)          */
  uint32_t* flag[8];       /* this rank's flag word of the slot on rank m      */
  const uint32_t* d_acks;  /* the slot's ack row in this rank's buffer [n]     */
  uint32_t* d_done;        /* the slot's CTA counter (device, zeroed; self-resetting) */
  void* d_spill;           /* local overflow records (plan_bytes == 64)        */
  int64_t plan_capacity;   /* bytes of one rank's plan section                 */
  int64_t cfg_capacity;    /* bytes of one rank's config section               */
  int64_t spill_capacity;  /* bytes of one rank's overflow section             */
  int32_t plan_bytes;      /* 128, or 64 (overflow section used)               */
  uint32_t epoch;          /* this launch's epoch (nonzero), published in the flags */
  uint32_t prev_epoch;     /* the slot's previous epoch (0: first use)         */
  int32_t reserved;
  parva_slot_ticket ticket;/* this rank's launches into the slot              */
} parva_mirror;
int parva_plan_batch_fused(const parva_tables* tables, const parva_index* index,
                           int32_t n_scenarios, int32_t n_services, const int32_t* d_scen_off,
                           const int32_t* d_svc_table, const double* d_svc_rate,
                           const double* d_svc_bound, int32_t optimize, int32_t threshold,
                           void* d_cfg, int32_t cfg_format, parva_plan_record* d_plan,
                           const parva_mirror* mirror, void* stream);

/* Consumer side of one slot: make `stream` wait until every rank's flag word
 * in d_flags equals `epoch` exactly (an epoch that was already overwritten
 * is an error, never stale data), then, if `release`, store `epoch` into
 * this rank's ack word of the slot on every rank (ack[m]) so producers may
 * reuse the slot -- release only when nothing later on the stream reads the
 * slot, else call parva_gather_release after the last reader.  A wait
 * longer than timeout_ns stores PARVA_LAUNCH_ERROR into *d_status and
 * releases nothing (producers then time out too: no hang).  pdl: launch as
 * a programmatic dependent launch (it may start while the previous kernel
 * on the stream runs; a later launch still waits for it to finish). */
typedef struct {
  int32_t n;               /* ranks, 1..8                                      */
  int32_t pdl;
  const uint32_t* d_flags; /* the slot's flag row in this rank's buffer [n]   */
  uint32_t* ack[8];        /* this rank's ack word of the slot on rank m      */
} parva_gather_slot;
int parva_gather_wait(const parva_gather_slot* slot, uint32_t epoch, int32_t release, int64_t timeout_ns,
                      int32_t* d_status, void* stream);
int parva_gather_release(const parva_gather_slot* slot, uint32_t epoch, void* stream);

/* Benchmark gate: one thread of `stream` waits until the pinned host word
 * *h_flag equals `value` (PARVA_LAUNCH_ERROR into *d_status after
 * timeout_ns).  Queue the work of a timed region behind it, then open it:
 * the region then measures device execution without host launch gaps. */
int parva_host_gate(const uint32_t* h_flag, uint32_t value, int64_t timeout_ns, int32_t* d_status,
                    void* stream);
/* CUDA IPC plumbing for the gathered blocks: an exportable zeroed device
 * allocation, its handle (parva_ipc_handle_bytes() bytes), and the mapping
 * of a peer's handle into this process (peer access enabled lazily). */
int parva_ipc_alloc(size_t bytes, void** d_ptr);
int parva_ipc_free(void* d_ptr);
int parva_ipc_handle_bytes(void);
int parva_ipc_handle(void* d_ptr, void* handle);
int parva_ipc_open(const void* handle, void** d_ptr);
int parva_ipc_close(void* d_ptr);

/* parva_plan_batch for tables too large for the shared-memory index: the
 * config records in d_cfg were produced by parva_configure_sweep. */
int parva_plan_batch_preconfigured(const parva_tables* tables, int32_t n_scenarios,
                                   int32_t n_services, const int32_t* d_scen_off, const int32_t* d_svc_table,
                                   int32_t optimize, int32_t threshold,
                                   parva_config_record* d_cfg, parva_plan_record* d_plan,
                                   void* stream);

/* Host-buffer entry for one batch: copies inputs to the device, plans, and
 * copies records back, then synchronizes `stream`.  The batch is cut into
 * chunks whose H2D copy, plan launch and D2H copy are pipelined on internal
 * streams (ordered after and before `stream`).  h_cfg receives config records
 * in cfg_format.  Tables and index are device-resident (built once).  Device
 * scratch comes from `d_scratch` (parva_plan_host_scratch bytes). */
size_t parva_plan_host_scratch(int32_t n_scenarios, int32_t n_services);
int parva_plan_host(const parva_tables* tables, const parva_index* index,
                    int32_t n_scenarios, const int32_t* h_scen_off,
                    const int32_t* h_svc_table, const double* h_svc_rate,
                    const double* h_svc_bound, int32_t optimize, int32_t threshold,
                    void* h_cfg, int32_t cfg_format, parva_plan_record* h_plan,
                    void* d_scratch, size_t scratch_bytes, void* stream);

/* Packed host batches: one contiguous input block and one output block per
 * chunk, so each chunk costs one H2D and one D2H copy.  A chunk of k
 * scenarios and m services is laid out (offsets from parva_packed_layout):
 *   input : int32 scen_off[k+1] (chunk-local, scen_off[0] = 0), f64 rate[m],
 *           f64 bound[m], uint16 table[m]
 *   output: plan records[k] (plan_bytes = 128, or 64 with a spill list),
 *           config records[m] (cfg_format), then for 64-byte records
 *           int32 spill_count (+pad to 16 B) and spill_cap entries of
 *           {int32 scenario (chunk-local), int32 pad, parva_plan_record}.
 * A 64-byte plan record is the 128-byte record truncated to 56 payload bytes;
 * a scenario whose payload does not fit has status PARVA_SPILLED and its full
 * record in the spill list (PARVA_CAPACITY if the list is full).  Blocks are
 * padded to 256 bytes. */
typedef struct {
  int64_t in_scen_off, in_rate, in_bound, in_table, in_bytes;
  int64_t out_plan, out_cfg, out_spill, out_bytes;
  int32_t plan_bytes, spill_cap;
} parva_chunk_layout;

int parva_packed_layout(int32_t k, int32_t m, int32_t cfg_format, int32_t plan_bytes,
                        parva_chunk_layout* out);

/* Plan a packed batch: chunk c has h_chunk_scen[c] scenarios and
 * h_chunk_svc[c] services, input block h_in[c], output block h_out[c] (host
 * memory, pinned for full speed).  H2D(c+1) / plan(c) / D2H(c-1) overlap in a
 * cached CUDA graph; returns after `stream` has synchronized.  Scratch:
 * parva_plan_host_packed_scratch bytes of device memory. */
size_t parva_plan_host_packed_scratch(int32_t n_chunks, const int32_t* h_chunk_scen,
                                      const int32_t* h_chunk_svc, int32_t cfg_format,
                                      int32_t plan_bytes);
int parva_plan_host_packed(const parva_tables* tables, const parva_index* index,
                           int32_t n_chunks, const int32_t* h_chunk_scen,
                           const int32_t* h_chunk_svc, const void* const* h_in,
                           void* const* h_out, int32_t optimize, int32_t threshold,
                           int32_t cfg_format, int32_t plan_bytes, void* d_scratch,
                           size_t scratch_bytes, void* stream);

/* Streamed input block (parva_plan_host_mapped): a header, then one packed
 * chunk block (parva_packed_layout of the chunk, chunk-local offsets) per
 * chunk of consecutive scenarios, so the data of the first scenarios arrives
 * first.  Header: int32 n_chunks, int32 chunk_scen (scenarios per chunk, the
 * last chunk may hold fewer), int32 pad[2], parva_stream_chunk[n_chunks];
 * padded to 256 bytes.  A chunk whose scenarios all list the same table ids
 * (same count, same order -- e.g. every scenario over one model set) stores
 * that sequence once (tmpl = its length) instead of one id per service, and
 * no offsets (rates at the block start; scenario k owns services
 * [k tmpl, (k+1) tmpl)).  Chunk blocks are 16-byte aligned. */
typedef struct {
  int32_t scen_lo;      /* first scenario of the chunk          */
  int32_t svc_lo;       /* first service of the chunk           */
  int32_t k, m;         /* scenarios, services                  */
  int64_t offset;       /* byte offset of the chunk block       */
  int32_t tmpl;         /* > 0: table ids stored once per chunk  */
  int32_t reserved;
} parva_stream_chunk;

#define parva_stream_header_bytes(n_chunks) ((((int64_t)(n_chunks) * 32 + 16) + 255) & ~(int64_t)255)

/* Bytes of the streamed input block for a batch: an upper bound for these
 * offsets (exact when no chunk repeats one table-id sequence). */
int64_t parva_stream_bytes(int32_t n_scenarios, const int32_t* h_scen_off, int32_t chunk_scen);
/* Pack a batch (services of scenario k: [h_scen_off[k], h_scen_off[k+1]),
 * h_scen_off[0] = 0) into a streamed input block of `capacity` bytes;
 * returns the bytes written (pass that as in_bytes), or -1. */
int64_t parva_stream_pack(int32_t n_scenarios, const int32_t* h_scen_off, const uint16_t* h_table,
                          const double* h_rate, const double* h_bound, int32_t chunk_scen,
                          void* h_block, int64_t capacity);

/* parva_stream_pack from the plain arrays a caller of parva_plan_host holds
 * (int32 table ids; ids outside [0, 65535) become 0xFFFF, i.e. no table:
 * PARVA_BAD_INPUT for that service), on up to n_threads host threads (0 =
 * all; PARVA_PACK_THREADS caps the pool).  Returns the bytes written, or -1
 * (bad offsets, capacity too small). */
int64_t parva_stream_pack_arrays(int32_t n_scenarios, const int32_t* h_scen_off, const int32_t* h_table,
                                 const double* h_rate, const double* h_bound, int32_t chunk_scen,
                                 void* h_block, int64_t capacity, int32_t n_threads);

/* Zero-copy host entry (the end-to-end path; one batch, one launch).  The
 * input block (streamed layout, parva_stream_pack) and the output block
 * (parva_mapped_layout: plan records[k], config records[m], and for 64-byte
 * plan records an overflow area of k full 128-byte records -- a scenario
 * with status PARVA_SPILLED has its full record at index k) live in pinned,
 * mapped host memory.  Inside the one kernel loader warps copy the input
 * block over PCIe in 8 KB slices, in order, into a device staging area and
 * publish each slice with a flag; every half warp then takes the next
 * scenario, waits for its chunk's slices, configures and plans it (full
 * warps re-plan the few that need more than 16 services or GPUs), and
 * writes its records straight into the host output block.  So the H2D
 * stream, the planning and the D2H writes overlap.  Scratch:
 * parva_plan_host_mapped_scratch bytes of device memory (initialised by the
 * first call with it; one call at a time per scratch).  Synchronizes
 * `stream` before returning.  The device address of the last few blocks is
 * cached and a scratch keeps its flag epoch: call parva_forget_block before
 * freeing a block or a scratch. */
void parva_forget_block(const void* h_block);
int parva_mapped_layout(int32_t k, int32_t m, int32_t cfg_format, int32_t plan_bytes,
                        parva_chunk_layout* out);
size_t parva_plan_host_mapped_scratch(int64_t in_bytes);
int parva_plan_host_mapped(const parva_tables* tables, const parva_index* index,
                           int32_t n_scenarios, int32_t n_services, const void* h_in,
                           int64_t in_bytes, void* h_out, int32_t optimize, int32_t threshold,
                           int32_t cfg_format, int32_t plan_bytes, void* d_scratch,
                           size_t scratch_bytes, void* stream);

/* Asynchronous form: enqueue the same call and return at once with a ticket
 * for parva_plan_host_mapped_wait, which spins on a completion word the
 * kernel writes into pinned host memory after a system-scope fence (no
 * stream synchronize).  Consecutive calls on one stream overlap: each is a
 * programmatic dependent launch, so the next call's loaders start streaming
 * its input while the previous call plans its last scenarios.  Overlap is
 * bounded by construction on the host: a call on a scratch, or into an
 * output block, that an unfinished call still uses first waits for that call
 * (so give each call in flight its own scratch and output block to keep
 * them overlapping).  The input block must stay unmodified until the call
 * completes.  Replaces a sequence of plan_services calls (pipeline.py:83-111)
 * over successive scenario batches. */
int parva_plan_host_mapped_submit(const parva_tables* tables, const parva_index* index,
                                  int32_t n_scenarios, int32_t n_services, const void* h_in,
                                  int64_t in_bytes, void* h_out, int32_t optimize,
                                  int32_t threshold, int32_t cfg_format, int32_t plan_bytes,
                                  void* d_scratch, size_t scratch_bytes, void* stream,
                                  uint64_t* ticket);
int parva_plan_host_mapped_wait(uint64_t ticket);

/* The end-to-end step in one call, from the plain arrays a caller of
 * parva_plan_host holds (any host memory): wait for any unfinished call
 * still reading the pinned input block h_in (capacity in_capacity,
 * parva_stream_bytes), pack the arrays into it (parva_stream_pack_arrays, on
 * the library's host threads), then parva_plan_host_mapped_submit.  The
 * records of the call are in h_out after parva_plan_host_mapped_wait(*ticket). */
int parva_plan_host_arrays_submit(const parva_tables* tables, const parva_index* index,
                                  int32_t n_scenarios, const int32_t* h_scen_off,
                                  const int32_t* h_table, const double* h_rate,
                                  const double* h_bound, int32_t chunk_scen, void* h_in,
                                  int64_t in_capacity, void* h_out, int32_t optimize,
                                  int32_t threshold, int32_t cfg_format, int32_t plan_bytes,
                                  void* d_scratch, size_t scratch_bytes, void* stream,
                                  uint64_t* ticket);

/* ------------------------------------------------------ general problems */
/* One problem = a catalogue of segment kinds, a service list, an optional
 * initial DeploymentMap and ledger.  Names (service ids) are indices
 * 0..n_names-1; services are names 0..n_services-1, other names only occur
 * in placements or the initial ledger (unknown services).  All arrays are
 * device arrays. */
typedef struct {
  /* catalogue of segment kinds: instance size (1,2,3,4,7), throughput, name */
  int32_t n_cat;
  const uint8_t* d_cat_size;
  const double*  d_cat_tp;
  const int32_t* d_cat_name;
  /* services: small-segment kinds for propose_small_segments (cat or -1),
   * and the relocation queue input: opt kind x count, then last kind */
  int32_t n_services;
  int32_t n_names;
  const int32_t* d_svc_t1;
  const int32_t* d_svc_t2;
  const int32_t* d_svc_opt;
  const int64_t* d_svc_count;
  const int32_t* d_svc_last;
  const double*  d_svc_rate;     /* for the optimize coverage assert          */
  /* initial map: n_gpus GPUs with ids; placements [pl_off[g], pl_off[g+1]) */
  int32_t n_gpus;
  const int64_t* d_gpu_id;
  const int32_t* d_pl_off;
  const int32_t* d_pl_cat;
  const uint8_t* d_pl_slot;
  /* initial ledger over names (order 0 = absent) */
  const double*  d_ledger_val;
  const int32_t* d_ledger_order;
  int32_t relocate;              /* run relocate_segments into the map       */
  int32_t optimize;              /* run optimize_allocation afterwards        */
  int32_t threshold;
} parva_general_problem;

typedef struct {
  int32_t gpu_cap;               /* capacity of the GPU arrays                */
  int32_t place_cap;             /* capacity of the placement arrays          */
  int32_t diag_cap;
  int32_t* d_status;             /* [1] parva_status                          */
  int32_t* d_counts;             /* [4] n_gpus, n_place, n_diag, n_gpus_unopt */
  int64_t* d_gpu_id;             /* [gpu_cap]                                 */
  int32_t* d_pl_off;             /* [gpu_cap + 1]                             */
  int32_t* d_pl_cat;             /* [place_cap]                               */
  uint8_t* d_pl_slot;            /* [place_cap]                               */
  int64_t* d_diag;               /* [diag_cap*3]: reason, gpu id, name        */
  double*  d_ledger_val;         /* [n_names]                                 */
  int32_t* d_ledger_order;       /* [n_names]                                 */
  int32_t* d_fallback;           /* [1]                                       */
} parva_general_result;

/* Device workspace for parva_plan_general (GPU state + lists + queues). */
size_t parva_plan_general_workspace(const parva_general_problem* p, int32_t gpu_cap);
int parva_plan_general(const parva_general_problem* p, parva_general_result* r,
                       void* d_workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------- simulator */
/* Batched run_simulation (evaluation.py:207-226, 327-416):
 * one independent simulation per service, for any number of runs at once.
 * Service s: arrival process d_kind[s] (0 none, 1 poisson, 2 deterministic)
 * from its numpy PCG64 state d_pcg[4s..4s+3] (state hi, lo, increment hi,
 * lo -- SeedSequence(seed).spawn(n)[i] seeded on the host), d_scale[s]
 * (poisson: 1/rate; deterministic: step = 1/rate), d_count[s] (poisson: the
 * chunk size max(int(rate*horizon*1.2)+16, 64); deterministic: floor(
 * horizon/step)); a buffer [d_buf_off[s], d_buf_off[s+1]) for its arrivals
 * (ms), which afterwards holds its batch latencies; segments [d_seg_off[s],
 * d_seg_off[s+1]) in dispatch (deployment-map) order.  Device arrays. */
typedef struct {
  int32_t n_services;
  const int32_t*  d_kind;
  const uint64_t* d_pcg;         /* [4 n_services]                           */
  const double*   d_scale;
  const int64_t*  d_count;
  const double*   d_horizon_s;
  const int64_t*  d_buf_off;     /* [n_services + 1]                         */
  const int32_t*  d_seg_off;     /* [n_services + 1]                         */
  const double*   d_seg_ms;      /* segment service time (profiled latency)  */
  const int32_t*  d_seg_batch;
  const int32_t*  d_seg_lanes;   /* process count                            */
  const double*   d_slo;         /* client-facing SLO (ms)                   */
  const double*   d_horizon_ms;
} parva_sim_problem;

typedef struct {
  int64_t* d_arrived;            /* [n_services]                             */
  int64_t* d_served;
  int64_t* d_batches;
  int64_t* d_violations;
  double*  d_buf;                /* batch b of service s at d_buf_off[s] + b  */
  double*  d_busy_ms;            /* per segment                              */
  int32_t* d_status;             /* per service: PARVA_OK, or PARVA_CAPACITY
                                    (buffer, > 32 segments or > 64 lanes)   */
} parva_sim_result;

int parva_simulate(const parva_sim_problem* problem, const parva_sim_result* result, void* stream);
/* Host-side seeding: the PCG64 states (state hi, lo, inc hi, lo per child)
 * of np.random.default_rng(SeedSequence(seed).spawn(...)[first_child + c])
 * for c < n_children, the seed given as little-endian uint32 words
 * (evaluation.py:308-315 seeding; numpy SeedSequence + PCG64 seeding restated). */
int parva_sim_seed_states(const uint32_t* seed_words, int32_t n_seed_words, int64_t first_child,
                          int64_t n_children, uint64_t* out);
/* Test hooks: glibc log1p on (-1, 0] as the simulator computes it, and numpy
 * Generator.exponential(scale) draws from a PCG64 state. */
int parva_sim_log1p(const double* d_x, double* d_out, int64_t n, void* stream);
int parva_sim_exponential(const uint64_t* d_pcg, double scale, int64_t n, double* d_out, void* stream);

/* ------------------------------------------------ fine-grained API kernels */
/* Lists k = [d_off[k], d_off[k+1]) of (instance size, throughput) triplets in
 * caller order (one thread per list). */

/* select_optimal_segment (configurator.py:127-139): absolute index of the
 * chosen triplet, -1 for an empty list. */
int parva_select_optimal_lists(int32_t n_lists, const int32_t* d_off, const int32_t* d_size,
                               const double* d_tp, int32_t* d_out, void* stream);

/* match_demand (configurator.py:142-186) on best_triplets lists: absolute
 * indices of optimal/last triplet (-1 none), count, coverage, status. */
int parva_match_demand_lists(int32_t n_lists, const int32_t* d_off, const int32_t* d_size,
                             const double* d_tp, const double* d_rate, int32_t* d_opt,
                             int32_t* d_last, int64_t* d_count, double* d_coverage,
                             uint8_t* d_status, void* stream);

/* propose_small_segments (allocator.py:319-359): tp == 0 marks an absent
 * size-1 / size-2 triplet; ok = 0 is SmallSegmentsUnavailableError. */
int parva_propose_small_batch(int32_t n, const double* d_tp1, const double* d_tp2,
                              const double* d_freed, int64_t* d_k2, int64_t* d_k1,
                              uint8_t* d_ok, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PARVA_B200_H */
