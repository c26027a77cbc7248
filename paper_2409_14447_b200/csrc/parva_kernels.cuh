// parva_kernels.cuh — launcher interfaces between the kernels and capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/parva_b200.h"

namespace parva {

constexpr int kMaxMirror = 8;        // ranks of a fused all-gather (one NVLink domain)

struct PlanArgs {
  const double* pts;             // prepared (tp, lat) pairs (global)
  const double* idx_lat;         // prefix-argmax index (global; copied to smem)
  const uint16_t* idx_best;
  const double* idx_tp;          // tp in key order (index copy, 16-B padded)
  const int64_t* seg_start;
  const int32_t* seg_count;
  int n_tables;
  int64_t n_points;
  int max_seg_points = -1;       // tables->max_seg_points (PARVA_CFG_TINY needs <= 254)
  int n_scen;
  int n_svc;                     // services [scen_off[0], scen_off[0] + n_svc)
  const int32_t* scen_off;
  const int32_t* svc_table;
  const uint16_t* svc_table16;   // packed host format (used when non-null)
  const double* svc_rate;
  const double* svc_bound;
  int optimize, threshold;
  int cfg_given;                 // config records precomputed by K1
  int smem_index;                // index resident in shared memory
  void* cfg;                     // config records in cfg_format
  int cfg_format;                // PARVA_CFG_FULL / _COMPACT / _TINY
  parva_plan_record* plan;       // byte stride plan_bytes (128, or 64 + spill list)
  int plan_bytes;
  int spill_cap;
  int32_t* spill_count;          // 64-byte records: spill list header
  uint8_t* spill;                // spill_cap entries of kSpillEntry bytes
  // warp kernel (zero-copy host entry): half warps take scenarios from
  // work[0]; work[1] counts finished warps (the last one resets the counters,
  // so they are zero between launches)
  uint32_t* work = nullptr;
  int spill_direct = 0;          // 64-byte records: full record at spill + 128 * scenario
  // streamed inputs (warp kernel, zero-copy host entry): the packed input
  // block at stream_src (mapped host memory) is copied in kStreamSlice-byte
  // slices, in order, by n_loaders loader threads into stream_dst (device; the
  // scen_off / svc_* pointers point into it); slice s has landed when
  // slice_flag[s] == epoch
  const uint8_t* stream_src = nullptr;
  uint8_t* stream_dst = nullptr;
  int64_t stream_bytes = 0;
  uint32_t* slice_flag = nullptr;
  uint32_t epoch = 0;
  int n_loaders = 0;
  // asynchronous calls: the last warp stores epoch to done_word (mapped host
  // memory) after a system-scope fence; pdl launches the kernel with
  // programmatic stream serialization, so it may start while the previous
  // streamed call on the stream is still finishing its last scenarios
  uint32_t* done_word = nullptr;
  int pdl = 0;
  // slot ticket (overlapped and fused launches; parva_slot_ticket): every
  // CTA adds its scenario count to the slot's completion counter
  // (*slot_count, one fire-and-forget release reduction after its last
  // store); before its first store, thread 0 waits until the counter has
  // reached slot_wait -- every scenario of the slot's earlier launches is
  // done.  A wait that times out stores PARVA_LAUNCH_ERROR into *err_word
  // and the CTA exits without storing.
  unsigned long long* slot_count = nullptr;
  unsigned long long slot_wait = 0;
  int32_t* err_word = nullptr;
  unsigned long long ticket_timeout_ns = 60ull * 1000 * 1000 * 1000;   // PARVA_TICKET_TIMEOUT_MS
  // fused all-gather (device path): each tile's plan / config records (and,
  // for 64-byte plan records, the full records of spilled scenarios) are
  // also stored at mirror_plan[m] / mirror_cfg[m] / mirror_spill[m] (the same
  // record index), i.e. into this rank's part of slot s on every rank over
  // peer memory.  Before storing, the CTAs also wait until every rank has
  // released the slot's previous epoch (ack_row[m] >= ack_prev, written by
  // rank m's parva_gather_wait).  The last CTA (counter *done_ctas, reset
  // before publishing) stores flag_epoch into peer_flag[m] (this rank's flag
  // word of slot s on rank m) after a system-scope fence.
  int n_mirror = 0;
  uint8_t* mirror_plan[kMaxMirror] = {};
  uint8_t* mirror_cfg[kMaxMirror] = {};
  uint8_t* mirror_spill[kMaxMirror] = {};
  uint32_t* peer_flag[kMaxMirror] = {};
  const uint32_t* ack_row = nullptr;
  uint32_t ack_prev = 0, flag_epoch = 0;
  uint32_t* done_ctas = nullptr;
};

#ifndef PARVA_STREAM_SLICE
#define PARVA_STREAM_SLICE 8192
#endif
#ifndef PARVA_LOADER_BUFS
#define PARVA_LOADER_BUFS 3
#endif
constexpr int kStreamSlice = PARVA_STREAM_SLICE;   // streamed input slice (one TMA bulk copy)
constexpr int kLoaderBufs = PARVA_LOADER_BUFS;     // shared-memory slice buffers per loader

constexpr int kSpillEntry = 144;   // int32 scenario, 12 B pad, 128-byte record
constexpr int kMaxDevices = 64;    // per-device launch-configuration caches
constexpr int kWorkWords = 8;      // work counters of the warp kernel

int launch_configure_sweep(const parva_tables* t, int nq, const int32_t* q_table, const double* q_rate,
                           const double* q_bound, parva_config_record* out, cudaStream_t stream);
int launch_build_index(const parva_tables* t, parva_index* idx, int* d_err, cudaStream_t stream);
int launch_plan_batch(const PlanArgs& A, cudaStream_t stream);
int plan_batch_grid(const PlanArgs& A);
int add_plan_batch_node(cudaGraph_t g, const PlanArgs& A, const cudaGraphNode_t* deps, size_t ndeps,
                        cudaGraphNode_t* node);
size_t general_workspace(const parva_general_problem* p, int64_t cap);
int launch_plan_general(const parva_general_problem* p, parva_general_result* r, void* ws, size_t ws_bytes,
                        cudaStream_t stream);

}  // namespace parva
