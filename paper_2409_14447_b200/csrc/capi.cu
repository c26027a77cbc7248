// capi.cu — the extern "C" boundary declared in include/parva_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <emmintrin.h>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <sched.h>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "parva_common.cuh"
#include "parva_kernels.cuh"


#ifndef PARVA_SMEM_INDEX_LIMIT
#define PARVA_SMEM_INDEX_LIMIT (120 * 1024)
#endif
static constexpr size_t kSmemIndexLimit = PARVA_SMEM_INDEX_LIMIT;  // index bytes kept in shared memory

extern "C" {

int parva_abi_version(void) { return PARVA_ABI_VERSION; }

size_t parva_plan_batch_workspace(int32_t, int32_t) { return 0; }

int parva_build_index(const parva_tables* tables, parva_index* index, void* stream) {
  if (!tables || !index) return PARVA_BAD_INPUT;
  int* d_err = nullptr;
  if (cudaMallocAsync(&d_err, sizeof(int), (cudaStream_t)stream) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  cudaMemsetAsync(d_err, 0, sizeof(int), (cudaStream_t)stream);
  int rc = parva::launch_build_index(tables, index, d_err, (cudaStream_t)stream);
  int h_err = 0;
  cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaFreeAsync(d_err, (cudaStream_t)stream);
  if (rc != PARVA_OK) return rc;
  return h_err ? PARVA_CAPACITY : PARVA_OK;
}

int parva_configure_sweep(const parva_tables* tables, int32_t n_queries, const int32_t* d_q_table,
                          const double* d_q_rate, const double* d_q_bound, parva_config_record* d_out,
                          void* stream) {
  if (!tables || n_queries < 0) return PARVA_BAD_INPUT;
  return parva::launch_configure_sweep(tables, n_queries, d_q_table, d_q_rate, d_q_bound, d_out,
                                       (cudaStream_t)stream);
}

static int64_t cfg_record_bytes(int cfg_format) {
  return cfg_format == PARVA_CFG_TINY ? 8 : cfg_format == PARVA_CFG_COMPACT ? 16 : 32;
}

static int plan_batch_impl(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                           int32_t n_services, const int32_t* d_scen_off, const int32_t* d_svc_table, const double* d_svc_rate,
                           const double* d_svc_bound, int32_t optimize, int32_t threshold, void* d_cfg,
                           int cfg_format, parva_plan_record* d_plan, int cfg_given, cudaStream_t stream,
                           int pdl = 0, const parva_slot_ticket* ticket = nullptr,
                           const parva_mirror* mirror = nullptr) {
  parva::PlanArgs A;
  A.pdl = pdl;
  A.plan_bytes = 128;
  A.spill_cap = 0;
  A.spill_count = nullptr;
  A.spill = nullptr;
  if (ticket) {
    static long long s_timeout_ms = -1;   // PARVA_TICKET_TIMEOUT_MS (tests), default 60 s
    if (s_timeout_ms < 0) {
      const char* e = std::getenv("PARVA_TICKET_TIMEOUT_MS");
      s_timeout_ms = e ? std::max(1ll, std::atoll(e)) : 60000ll;
    }
    A.ticket_timeout_ns = (unsigned long long)s_timeout_ms * 1000000ull;
    A.slot_count = (unsigned long long*)ticket->d_count;
    A.slot_wait = ticket->wait_count;
    A.err_word = ticket->d_err;
  }
  if (mirror) {
    A.n_mirror = mirror->n;
    for (int m = 0; m < mirror->n; m++) {
      A.mirror_plan[m] = (uint8_t*)mirror->plan[m];
      A.mirror_cfg[m] = (uint8_t*)mirror->cfg[m];
      A.mirror_spill[m] = (uint8_t*)mirror->spill[m];
      A.peer_flag[m] = mirror->flag[m];
    }
    A.ack_row = mirror->d_acks;
    A.ack_prev = mirror->prev_epoch;
    A.flag_epoch = mirror->epoch;
    A.done_ctas = mirror->d_done;
    if (mirror->plan_bytes == 64) {
      // 64-byte records; a spilled scenario's full record at the same index
      // of the overflow area (local, then mirrored)
      A.plan_bytes = 64;
      A.spill = (uint8_t*)mirror->d_spill;
      A.spill_cap = n_scenarios;
      A.spill_direct = 1;
    }
  }
  A.pts = tables->d_pts;
  A.idx_lat = index ? index->d_lat_sorted : nullptr;
  A.idx_best = index ? index->d_best : nullptr;
  A.idx_tp = index ? index->d_tp : nullptr;
  A.seg_start = tables->d_seg_start;
  A.seg_count = tables->d_seg_count;
  A.n_tables = tables->n_tables;
  A.n_points = tables->n_points;
  A.max_seg_points = tables->max_seg_points;
  A.n_scen = n_scenarios;
  A.n_svc = n_services;
  A.scen_off = d_scen_off;
  A.svc_table = d_svc_table;
  A.svc_table16 = nullptr;
  A.svc_rate = d_svc_rate;
  A.svc_bound = d_svc_bound;
  A.optimize = optimize;
  A.threshold = threshold;
  A.cfg_given = cfg_given;
  // back-to-back (overlapped) launches read the index through L1 instead of
  // staging it per CTA: a CTA's 24 KB bulk copy is a serial prologue that
  // holds its SM slot, while the L1-resident index is shared by all the
  // SM's CTAs (measured: 22.6 -> 21.3 us per overlapped C2 step; a single
  // launch is faster with the staged copy, 31.7 vs 35 us)
  A.smem_index = !cfg_given && !pdl && tables->n_points * 18 <= (int64_t)kSmemIndexLimit;
#ifdef PARVA_NO_SMEM_INDEX   // (A/B builds: small CTAs read the index through L1)
  A.smem_index = 0;
#endif
  A.cfg = d_cfg;
  A.cfg_format = cfg_format;
  A.plan = d_plan;
  return parva::launch_plan_batch(A, stream);
}

static bool ticket_ok(const parva_slot_ticket* t) { return t && t->d_count; }

int parva_plan_batch(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                     int32_t n_services, const int32_t* d_scen_off, const int32_t* d_svc_table, const double* d_svc_rate,
                     const double* d_svc_bound, int32_t optimize, int32_t threshold, void* d_cfg,
                     int32_t cfg_format, parva_plan_record* d_plan, void* stream) {
  if (!tables || !index || n_scenarios < 0 || !d_cfg || !d_plan) return PARVA_BAD_INPUT;
  if (cfg_format < PARVA_CFG_FULL || cfg_format > PARVA_CFG_TINY) return PARVA_BAD_INPUT;
  return plan_batch_impl(tables, index, n_scenarios, n_services, d_scen_off, d_svc_table, d_svc_rate, d_svc_bound,
                         optimize, threshold, d_cfg, cfg_format, d_plan, 0, (cudaStream_t)stream);
}

// parva_plan_batch as a programmatic dependent launch: it may start while the
// previous overlapped call on the stream is still finishing (its CTAs take
// SM slots as the predecessor's retire); the slot ticket serializes the
// launches that share an output slot.
int parva_plan_batch_overlapped(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                                int32_t n_services, const int32_t* d_scen_off, const int32_t* d_svc_table,
                                const double* d_svc_rate, const double* d_svc_bound, int32_t optimize,
                                int32_t threshold, void* d_cfg, int32_t cfg_format, parva_plan_record* d_plan,
                                const parva_slot_ticket* ticket, void* stream) {
  if (!tables || !index || n_scenarios < 0 || !d_cfg || !d_plan || !ticket_ok(ticket)) return PARVA_BAD_INPUT;
  if (cfg_format < PARVA_CFG_FULL || cfg_format > PARVA_CFG_TINY) return PARVA_BAD_INPUT;
  if (n_scenarios == 0) return PARVA_BAD_INPUT;   // nothing would complete the ticket
  return plan_batch_impl(tables, index, n_scenarios, n_services, d_scen_off, d_svc_table, d_svc_rate, d_svc_bound,
                         optimize, threshold, d_cfg, cfg_format, d_plan, 0, (cudaStream_t)stream, 1, ticket);
}

// parva_plan_batch with a fused all-gather: every tile's records are also
// stored into this rank's sections of the slot on each rank (peer memory),
// and the last CTA stores the epoch into this rank's flag word on every rank.
int parva_plan_batch_fused(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                           int32_t n_services, const int32_t* d_scen_off, const int32_t* d_svc_table,
                           const double* d_svc_rate, const double* d_svc_bound, int32_t optimize, int32_t threshold,
                           void* d_cfg, int32_t cfg_format, parva_plan_record* d_plan, const parva_mirror* mirror,
                           void* stream) {
  if (!tables || !index || n_scenarios < 0 || !d_cfg || !d_plan || !mirror) return PARVA_BAD_INPUT;
  if (cfg_format < PARVA_CFG_FULL || cfg_format > PARVA_CFG_TINY) return PARVA_BAD_INPUT;
  if (mirror->n < 1 || mirror->n > parva::kMaxMirror || !mirror->d_acks || !mirror->d_done ||
      !ticket_ok(&mirror->ticket) || mirror->epoch == 0 || mirror->epoch == mirror->prev_epoch)
    return PARVA_BAD_INPUT;
  if (mirror->plan_bytes != 128 && mirror->plan_bytes != 64) return PARVA_BAD_INPUT;
  if (n_scenarios == 0) return PARVA_BAD_INPUT;   // nothing would publish the epoch
  // the records must fit this rank's sections (the kernel copies whole
  // record ranges into them)
  if (int64_t(n_scenarios) * mirror->plan_bytes > mirror->plan_capacity ||
      int64_t(n_services) * cfg_record_bytes(cfg_format) > mirror->cfg_capacity)
    return PARVA_BAD_INPUT;
  if (mirror->plan_bytes == 64 && (!mirror->d_spill || int64_t(n_scenarios) * 128 > mirror->spill_capacity))
    return PARVA_BAD_INPUT;
  for (int m = 0; m < mirror->n; m++)
    if (!mirror->plan[m] || !mirror->cfg[m] || !mirror->flag[m] || (mirror->plan_bytes == 64 && !mirror->spill[m]))
      return PARVA_BAD_INPUT;
  return plan_batch_impl(tables, index, n_scenarios, n_services, d_scen_off, d_svc_table, d_svc_rate, d_svc_bound,
                         optimize, threshold, d_cfg, cfg_format, d_plan, 0, (cudaStream_t)stream,
                         mirror->overlap ? 1 : 0, &mirror->ticket, mirror);
}

// Same as parva_plan_batch but the config records in d_cfg were produced by
// parva_configure_sweep (tables too large for the shared-memory index).
int parva_plan_batch_preconfigured(const parva_tables* tables, int32_t n_scenarios, int32_t n_services,
                                   const int32_t* d_scen_off,
                                   const int32_t* d_svc_table, int32_t optimize, int32_t threshold,
                                   parva_config_record* d_cfg, parva_plan_record* d_plan, void* stream) {
  if (!tables || n_scenarios < 0 || !d_cfg || !d_plan) return PARVA_BAD_INPUT;
  return plan_batch_impl(tables, nullptr, n_scenarios, n_services, d_scen_off, d_svc_table, nullptr, nullptr, optimize,
                         threshold, d_cfg, PARVA_CFG_FULL, d_plan, 1, (cudaStream_t)stream);
}

static size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

size_t parva_plan_host_scratch(int32_t n_scenarios, int32_t n_services) {
  return up256(size_t(n_scenarios + 1) * 4) + up256(size_t(n_services) * 4) + 2 * up256(size_t(n_services) * 8) +
         up256(size_t(n_services) * sizeof(parva_config_record)) + up256(size_t(n_scenarios) * sizeof(parva_plan_record));
}

// The host entry's chunked H2D -> plan -> D2H pipeline is an explicitly
// built CUDA graph, cached per (device, shape, tables, scratch); a call with
// new host pointers only updates the memcpy nodes (cudaGraphExecMemcpyNode-
// SetParams1D).  One graph launch replaces ~40 stream API calls.
struct HostGraph {
  int dev = -1, n_scen = 0, n_svc = 0, cfg_format = 0, optimize = 0, threshold = 0, chunks = 0;
  const void* pts = nullptr;
  const void* idx = nullptr;
  void* scratch = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> nodes;          // per chunk: 4 H2D, 2 D2H
  std::vector<const void*> host;               // host pointers the nodes were built with
  uint64_t last_use = 0;
};
static std::mutex g_graph_mu;
static std::vector<HostGraph> g_graphs;
static uint64_t g_graph_clock = 0;

static void free_graph(HostGraph& G) {
  if (G.exec) cudaGraphExecDestroy(G.exec);
  if (G.graph) cudaGraphDestroy(G.graph);
  G = HostGraph();
}

int parva_plan_host(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                    const int32_t* h_scen_off, const int32_t* h_svc_table, const double* h_svc_rate,
                    const double* h_svc_bound, int32_t optimize, int32_t threshold, void* h_cfg,
                    int32_t cfg_format, parva_plan_record* h_plan, void* d_scratch, size_t scratch_bytes,
                    void* stream) {
  if (!tables || !index || n_scenarios < 0) return PARVA_BAD_INPUT;
  if (cfg_format != PARVA_CFG_FULL && cfg_format != PARVA_CFG_COMPACT) return PARVA_BAD_INPUT;
  if (n_scenarios == 0) return PARVA_OK;
  const int32_t n_services = h_scen_off[n_scenarios];
  if (parva_plan_host_scratch(n_scenarios, n_services) > scratch_bytes) return PARVA_BAD_INPUT;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t cfg_sz = cfg_format == PARVA_CFG_COMPACT ? sizeof(parva_config_compact) : sizeof(parva_config_record);
  uint8_t* p = (uint8_t*)d_scratch;
  int32_t* d_off = (int32_t*)p; p += up256(size_t(n_scenarios + 1) * 4);
  int32_t* d_tab = (int32_t*)p; p += up256(size_t(n_services) * 4);
  double* d_rate = (double*)p; p += up256(size_t(n_services) * 8);
  double* d_bound = (double*)p; p += up256(size_t(n_services) * 8);
  uint8_t* d_cfg = p; p += up256(size_t(n_services) * sizeof(parva_config_record));
  parva_plan_record* d_plan = (parva_plan_record*)p;
  int chunks = n_scenarios / 2500;
  chunks = chunks < 1 ? 1 : (chunks > 8 ? 8 : chunks);
  if (const char* e = getenv("PARVA_HOST_CHUNKS")) chunks = atoi(e) > 0 ? atoi(e) : chunks;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* host[6] = {h_scen_off, h_svc_table, h_svc_rate, h_svc_bound, h_cfg, h_plan};

  std::lock_guard<std::mutex> lock(g_graph_mu);
  HostGraph* G = nullptr;
  for (auto& e : g_graphs)
    if (e.dev == dev && e.n_scen == n_scenarios && e.n_svc == n_services && e.cfg_format == cfg_format &&
        e.optimize == optimize && e.threshold == threshold && e.pts == tables->d_pts && e.idx == index->d_lat_sorted &&
        e.scratch == d_scratch && e.chunks == chunks) { G = &e; break; }
  auto chunk = [&](int i, int& a, int& b, int& sa, int& sb) {
    a = int((int64_t)n_scenarios * i / chunks);
    b = int((int64_t)n_scenarios * (i + 1) / chunks);
    sa = h_scen_off[a];
    sb = h_scen_off[b];
  };
  // memcpy node parameters of chunk i, copy j (0..3 H2D, 4..5 D2H)
  auto copy_args = [&](int i, int j, void** dst, const void** src, size_t* bytes, cudaMemcpyKind* kind) {
    int a, b, sa, sb;
    chunk(i, a, b, sa, sb);
    switch (j) {
      case 0: *dst = d_off + a; *src = h_scen_off + a; *bytes = size_t(b - a + 1) * 4; break;
      case 1: *dst = d_tab + sa; *src = h_svc_table + sa; *bytes = size_t(sb - sa) * 4; break;
      case 2: *dst = d_rate + sa; *src = h_svc_rate + sa; *bytes = size_t(sb - sa) * 8; break;
      case 3: *dst = d_bound + sa; *src = h_svc_bound + sa; *bytes = size_t(sb - sa) * 8; break;
      case 4: *dst = (uint8_t*)h_cfg + size_t(sa) * cfg_sz; *src = d_cfg + size_t(sa) * cfg_sz;
              *bytes = size_t(sb - sa) * cfg_sz; break;
      default: *dst = h_plan + a; *src = d_plan + a; *bytes = size_t(b - a) * sizeof(parva_plan_record); break;
    }
    *kind = j < 4 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  };
  if (!G) {
    if (g_graphs.size() >= 8) {
      auto victim = g_graphs.begin();
      for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
        if (it->last_use < victim->last_use) victim = it;
      free_graph(*victim);
      g_graphs.erase(victim);
    }
    g_graphs.emplace_back();
    G = &g_graphs.back();
    G->dev = dev; G->n_scen = n_scenarios; G->n_svc = n_services; G->cfg_format = cfg_format;
    G->optimize = optimize; G->threshold = threshold; G->pts = tables->d_pts; G->idx = index->d_lat_sorted;
    G->scratch = d_scratch; G->chunks = chunks;
    if (cudaGraphCreate(&G->graph, 0) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    G->nodes.assign(size_t(chunks) * 6, nullptr);
    cudaGraphNode_t prev_in[4] = {}, prev_out[2] = {};
    for (int i = 0; i < chunks; i++) {
      int a, b, sa, sb;
      chunk(i, a, b, sa, sb);
      cudaGraphNode_t in[4];
      for (int j = 0; j < 4; j++) {   // H2D in chunk order (chunk i after chunk i-1)
        void* dst; const void* src; size_t bytes; cudaMemcpyKind kind;
        copy_args(i, j, &dst, &src, &bytes, &kind);
        if (cudaGraphAddMemcpyNode1D(&in[j], G->graph, i ? &prev_in[j] : nullptr, i ? 1 : 0, dst, src, bytes,
                                     kind) != cudaSuccess) return PARVA_LAUNCH_ERROR;
        G->nodes[size_t(i) * 6 + j] = in[j];
        prev_in[j] = in[j];
      }
      parva::PlanArgs A;
      A.pts = tables->d_pts; A.idx_lat = index->d_lat_sorted; A.idx_best = index->d_best; A.idx_tp = index->d_tp;
      A.seg_start = tables->d_seg_start; A.seg_count = tables->d_seg_count; A.n_tables = tables->n_tables;
      A.n_points = tables->n_points; A.max_seg_points = tables->max_seg_points;
      A.n_scen = b - a; A.n_svc = sb - sa; A.scen_off = d_off + a; A.svc_table = d_tab;
      A.svc_table16 = nullptr;
      A.svc_rate = d_rate; A.svc_bound = d_bound; A.optimize = optimize; A.threshold = threshold;
      A.cfg_given = 0; A.smem_index = tables->n_points * 18 <= (int64_t)kSmemIndexLimit; A.cfg = d_cfg;
      A.cfg_format = cfg_format; A.plan = d_plan + a;
      A.plan_bytes = 128; A.spill_cap = 0; A.spill_count = nullptr; A.spill = nullptr;
      cudaGraphNode_t kn;
      if (parva::add_plan_batch_node(G->graph, A, in, 4, &kn) != PARVA_OK) return PARVA_LAUNCH_ERROR;
      for (int j = 4; j < 6; j++) {   // D2H after this chunk's plan and the previous chunk's D2H
        void* dst; const void* src; size_t bytes; cudaMemcpyKind kind;
        copy_args(i, j, &dst, &src, &bytes, &kind);
        cudaGraphNode_t deps[2] = {kn, prev_out[j - 4]};
        cudaGraphNode_t o;
        if (cudaGraphAddMemcpyNode1D(&o, G->graph, deps, i ? 2 : 1, dst, src, bytes, kind) != cudaSuccess)
          return PARVA_LAUNCH_ERROR;
        G->nodes[size_t(i) * 6 + j] = o;
        prev_out[j - 4] = o;
      }
    }
    if (cudaGraphInstantiate(&G->exec, G->graph, 0) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    G->host.assign(host, host + 6);
  } else if (!std::equal(G->host.begin(), G->host.end(), host)) {
    for (int i = 0; i < chunks; i++)
      for (int j = 0; j < 6; j++) {
        void* dst; const void* src; size_t bytes; cudaMemcpyKind kind;
        copy_args(i, j, &dst, &src, &bytes, &kind);
        if (cudaGraphExecMemcpyNodeSetParams1D(G->exec, G->nodes[size_t(i) * 6 + j], dst, src, bytes, kind) !=
            cudaSuccess) return PARVA_LAUNCH_ERROR;
      }
    G->host.assign(host, host + 6);
  }
  G->last_use = ++g_graph_clock;
  if (cudaGraphLaunch(G->exec, s) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  return cudaStreamSynchronize(s) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

// ------------------------------------------------------------ packed host
static int64_t up256l(int64_t x) { return (x + 255) & ~int64_t(255); }

static int64_t cfg_bytes(int32_t cfg_format) {
  return cfg_format == PARVA_CFG_TINY ? sizeof(parva_config_tiny)
         : cfg_format == PARVA_CFG_COMPACT ? sizeof(parva_config_compact) : sizeof(parva_config_record);
}

int parva_packed_layout(int32_t k, int32_t m, int32_t cfg_format, int32_t plan_bytes, parva_chunk_layout* L) {
  if (!L || k < 0 || m < 0 || (plan_bytes != 64 && plan_bytes != 128)) return PARVA_BAD_INPUT;
  if (cfg_format < PARVA_CFG_FULL || cfg_format > PARVA_CFG_TINY) return PARVA_BAD_INPUT;
  L->in_scen_off = 0;
  L->in_rate = ((int64_t(k) + 1) * 4 + 15) & ~int64_t(15);
  L->in_bound = L->in_rate + int64_t(m) * 8;
  L->in_table = L->in_bound + int64_t(m) * 8;
  L->in_bytes = up256l(L->in_table + int64_t(m) * 2);
  L->plan_bytes = plan_bytes;
  L->spill_cap = plan_bytes == 64 ? 16 + k / 256 : 0;
  L->out_plan = 0;
  L->out_cfg = int64_t(k) * plan_bytes;
  L->out_spill = (L->out_cfg + int64_t(m) * cfg_bytes(cfg_format) + 15) & ~int64_t(15);
  L->out_bytes = up256l(L->out_spill + (plan_bytes == 64 ? 16 + int64_t(L->spill_cap) * parva::kSpillEntry : 0));
  return PARVA_OK;
}

size_t parva_plan_host_packed_scratch(int32_t n_chunks, const int32_t* k, const int32_t* m, int32_t cfg_format,
                                      int32_t plan_bytes) {
  size_t total = 0;
  for (int c = 0; c < n_chunks; c++) {
    parva_chunk_layout L;
    if (parva_packed_layout(k[c], m[c], cfg_format, plan_bytes, &L) != PARVA_OK) return 0;
    total += size_t(L.in_bytes) + size_t(L.out_bytes);
  }
  return total + 256;
}

struct PackedGraph {
  int dev = -1, n_chunks = 0, cfg_format = 0, plan_bytes = 0, optimize = 0, threshold = 0;
  std::vector<int32_t> k, m;
  const void* pts = nullptr;
  const void* idx = nullptr;
  void* scratch = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> in_nodes, out_nodes;
  std::vector<const void*> host_in;
  std::vector<void*> host_out;
  uint64_t last_use = 0;
};
static std::vector<PackedGraph> g_packed;

int parva_plan_host_packed(const parva_tables* tables, const parva_index* index, int32_t n_chunks,
                           const int32_t* h_k, const int32_t* h_m, const void* const* h_in, void* const* h_out,
                           int32_t optimize, int32_t threshold, int32_t cfg_format, int32_t plan_bytes,
                           void* d_scratch, size_t scratch_bytes, void* stream) {
  if (!tables || !index || n_chunks <= 0) return PARVA_BAD_INPUT;
  const size_t need = parva_plan_host_packed_scratch(n_chunks, h_k, h_m, cfg_format, plan_bytes);
  if (need == 0 || need > scratch_bytes) return PARVA_BAD_INPUT;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_graph_mu);
  PackedGraph* G = nullptr;
  for (auto& e : g_packed)
    if (e.dev == dev && e.n_chunks == n_chunks && e.cfg_format == cfg_format && e.plan_bytes == plan_bytes &&
        e.optimize == optimize &&
        e.threshold == threshold && e.pts == tables->d_pts && e.idx == index->d_lat_sorted &&
        e.scratch == d_scratch && std::equal(e.k.begin(), e.k.end(), h_k) && std::equal(e.m.begin(), e.m.end(), h_m)) {
      G = &e;
      break;
    }
  // device blocks: [in_0 | out_0 | in_1 | out_1 | ...] in scratch
  std::vector<parva_chunk_layout> L(n_chunks);
  std::vector<uint8_t*> d_in(n_chunks), d_out(n_chunks);
  {
    uint8_t* p = (uint8_t*)(((uintptr_t)d_scratch + 255) & ~uintptr_t(255));
    for (int c = 0; c < n_chunks; c++) {
      parva_packed_layout(h_k[c], h_m[c], cfg_format, plan_bytes, &L[c]);
      d_in[c] = p; p += L[c].in_bytes;
      d_out[c] = p; p += L[c].out_bytes;
    }
  }
  if (!G) {
    if (g_packed.size() >= 8) {
      auto victim = g_packed.begin();
      for (auto it = g_packed.begin(); it != g_packed.end(); ++it)
        if (it->last_use < victim->last_use) victim = it;
      if (victim->exec) cudaGraphExecDestroy(victim->exec);
      if (victim->graph) cudaGraphDestroy(victim->graph);
      g_packed.erase(victim);
    }
    g_packed.emplace_back();
    G = &g_packed.back();
    G->dev = dev; G->n_chunks = n_chunks; G->cfg_format = cfg_format; G->plan_bytes = plan_bytes; G->optimize = optimize;
    G->threshold = threshold; G->k.assign(h_k, h_k + n_chunks); G->m.assign(h_m, h_m + n_chunks);
    G->pts = tables->d_pts; G->idx = index->d_lat_sorted; G->scratch = d_scratch;
    if (cudaGraphCreate(&G->graph, 0) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    G->in_nodes.resize(n_chunks);
    G->out_nodes.resize(n_chunks);
    for (int c = 0; c < n_chunks; c++) {
      cudaGraphNode_t* dep_in = c ? &G->in_nodes[c - 1] : nullptr;
      if (cudaGraphAddMemcpyNode1D(&G->in_nodes[c], G->graph, dep_in, c ? 1 : 0, d_in[c], h_in[c], L[c].in_bytes,
                                   cudaMemcpyHostToDevice) != cudaSuccess) return PARVA_LAUNCH_ERROR;
      cudaGraphNode_t pre = G->in_nodes[c];
      if (plan_bytes == 64) {   // zero the spill count before the chunk's plan
        cudaMemsetParams mp = {};
        mp.dst = d_out[c] + L[c].out_spill;
        mp.value = 0; mp.elementSize = 4; mp.width = 4; mp.height = 1; mp.pitch = 0;
        cudaGraphNode_t ms;
        if (cudaGraphAddMemsetNode(&ms, G->graph, &G->in_nodes[c], 1, &mp) != cudaSuccess) return PARVA_LAUNCH_ERROR;
        pre = ms;
      }
      cudaGraphNode_t kn;
      if (h_k[c] > 0) {
        parva::PlanArgs A;
        A.pts = tables->d_pts; A.idx_lat = index->d_lat_sorted; A.idx_best = index->d_best; A.idx_tp = index->d_tp;
        A.seg_start = tables->d_seg_start; A.seg_count = tables->d_seg_count; A.n_tables = tables->n_tables;
        A.n_points = tables->n_points; A.max_seg_points = tables->max_seg_points;
        A.n_scen = h_k[c]; A.n_svc = h_m[c];
        A.scen_off = (const int32_t*)(d_in[c] + L[c].in_scen_off);
        A.svc_table = nullptr; A.svc_table16 = (const uint16_t*)(d_in[c] + L[c].in_table);
        A.svc_rate = (const double*)(d_in[c] + L[c].in_rate);
        A.svc_bound = (const double*)(d_in[c] + L[c].in_bound);
        A.optimize = optimize; A.threshold = threshold; A.cfg_given = 0;
        A.smem_index = tables->n_points * 18 <= (int64_t)kSmemIndexLimit;
        A.cfg = d_out[c] + L[c].out_cfg; A.cfg_format = cfg_format;
        A.plan = (parva_plan_record*)(d_out[c] + L[c].out_plan);
        A.plan_bytes = plan_bytes; A.spill_cap = L[c].spill_cap;
        A.spill_count = (int32_t*)(d_out[c] + L[c].out_spill);
        A.spill = d_out[c] + L[c].out_spill + 16;
        if (parva::add_plan_batch_node(G->graph, A, &pre, 1, &kn) != PARVA_OK) return PARVA_LAUNCH_ERROR;
      } else {
        kn = pre;
      }
      cudaGraphNode_t deps[2] = {kn, c ? G->out_nodes[c - 1] : nullptr};
      if (cudaGraphAddMemcpyNode1D(&G->out_nodes[c], G->graph, deps, c ? 2 : 1, h_out[c], d_out[c],
                                   L[c].out_bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    }
    if (cudaGraphInstantiate(&G->exec, G->graph, 0) != cudaSuccess) return PARVA_LAUNCH_ERROR;
    G->host_in.assign(h_in, h_in + n_chunks);
    G->host_out.assign(h_out, h_out + n_chunks);
  } else {
    for (int c = 0; c < n_chunks; c++) {
      if (G->host_in[c] != h_in[c]) {
        if (cudaGraphExecMemcpyNodeSetParams1D(G->exec, G->in_nodes[c], d_in[c], h_in[c], L[c].in_bytes,
                                               cudaMemcpyHostToDevice) != cudaSuccess) return PARVA_LAUNCH_ERROR;
        G->host_in[c] = h_in[c];
      }
      if (G->host_out[c] != h_out[c]) {
        if (cudaGraphExecMemcpyNodeSetParams1D(G->exec, G->out_nodes[c], h_out[c], d_out[c], L[c].out_bytes,
                                               cudaMemcpyDeviceToHost) != cudaSuccess) return PARVA_LAUNCH_ERROR;
        G->host_out[c] = h_out[c];
      }
    }
  }
  G->last_use = ++g_graph_clock;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaGraphLaunch(G->exec, s) != cudaSuccess) return PARVA_LAUNCH_ERROR;
  return cudaStreamSynchronize(s) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

// ------------------------------------------------------------ mapped host
int parva_mapped_layout(int32_t k, int32_t m, int32_t cfg_format, int32_t plan_bytes, parva_chunk_layout* L) {
  const int rc = parva_packed_layout(k, m, cfg_format, plan_bytes, L);
  if (rc != PARVA_OK) return rc;
  // the overflow area holds one full record per scenario (no spill list)
  L->spill_cap = plan_bytes == 64 ? k : 0;
  L->out_bytes = up256l(L->out_spill + (plan_bytes == 64 ? int64_t(k) * 128 : 0));
  return PARVA_OK;
}

static int loaders_for(int64_t in_bytes) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("PARVA_LOADERS");
    env = e ? std::max(0, std::atoi(e)) : 0;
  }
  if (env > 0) return env;
  // 16 loader CTAs x 3 x 8 KB in flight: PCIe-rate streaming while the
  // slices still land nearly in order (16 / 32 / 48 measured within 3%;
  // pipelined calls stream two inputs at once)
  return (int)std::min<int64_t>(16, std::max<int64_t>(1, (in_bytes + parva::kStreamSlice - 1) / parva::kStreamSlice));
}

int64_t parva_stream_bytes(int32_t n_scenarios, const int32_t* h_scen_off, int32_t chunk_scen) {
  if (n_scenarios < 0 || !h_scen_off || chunk_scen < 1) return -1;
  const int32_t n_ch = n_scenarios == 0 ? 0 : (n_scenarios + chunk_scen - 1) / chunk_scen;
  int64_t total = parva_stream_header_bytes(n_ch);
  for (int32_t c = 0; c < n_ch; c++) {
    const int32_t a = c * chunk_scen, b = std::min(n_scenarios, a + chunk_scen);
    parva_chunk_layout L;
    if (parva_packed_layout(b - a, h_scen_off[b] - h_scen_off[a], PARVA_CFG_TINY, 64, &L) != PARVA_OK) return -1;
    total += L.in_bytes;
  }
  return total;
}

int64_t parva_stream_pack(int32_t n_scenarios, const int32_t* h_scen_off, const uint16_t* h_table,
                          const double* h_rate, const double* h_bound, int32_t chunk_scen, void* h_block,
                          int64_t capacity) {
  const int64_t need = parva_stream_bytes(n_scenarios, h_scen_off, chunk_scen);
  if (need < 0 || need > capacity || !h_block) return -1;
  if (n_scenarios > 0 && h_scen_off[0] != 0) return -1;
  for (int32_t k = 0; k < n_scenarios; k++)
    if (h_scen_off[k + 1] < h_scen_off[k]) return -1;
  uint8_t* out = (uint8_t*)h_block;
  const int32_t n_ch = n_scenarios == 0 ? 0 : (n_scenarios + chunk_scen - 1) / chunk_scen;
  std::memset(out, 0, (size_t)parva_stream_header_bytes(n_ch));
  reinterpret_cast<int32_t*>(out)[0] = n_ch;
  reinterpret_cast<int32_t*>(out)[1] = chunk_scen;
  parva_stream_chunk* tab = reinterpret_cast<parva_stream_chunk*>(out + 16);
  int64_t off = parva_stream_header_bytes(n_ch);
  for (int32_t c = 0; c < n_ch; c++) {
    const int32_t a = c * chunk_scen, b = std::min(n_scenarios, a + chunk_scen);
    const int32_t sa = h_scen_off[a], sb = h_scen_off[b];
    parva_chunk_layout L;
    parva_packed_layout(b - a, sb - sa, PARVA_CFG_TINY, 64, &L);
    // one table-id sequence repeated by every scenario of the chunk?
    const int32_t t0 = h_scen_off[a + 1] - sa;
    bool tmpl = t0 > 0 && b - a > 1;
    for (int32_t k = a + 1; tmpl && k < b; k++) {
      const int32_t ka = h_scen_off[k];
      tmpl = h_scen_off[k + 1] - ka == t0 && std::memcmp(h_table + ka, h_table + sa, size_t(t0) * 2) == 0;
    }
    // template chunks: no offsets (scenario k owns [k t0, (k+1) t0)) and the
    // table ids once; otherwise offsets | rates | bounds | table ids
    const int32_t n_tab = tmpl ? t0 : sb - sa;
    const int64_t rate_at = tmpl ? 0 : L.in_rate;
    const int64_t table_at = rate_at + int64_t(sb - sa) * 16;
    const int64_t blk_bytes = (table_at + int64_t(n_tab) * 2 + 15) & ~int64_t(15);   // 16-B aligned blocks
    tab[c].scen_lo = a; tab[c].svc_lo = sa; tab[c].k = b - a; tab[c].m = sb - sa; tab[c].offset = off;
    tab[c].tmpl = tmpl ? t0 : 0; tab[c].reserved = 0;
    uint8_t* blk = out + off;
    std::memset(blk, 0, (size_t)blk_bytes);
    if (!tmpl) {
      int32_t* so = reinterpret_cast<int32_t*>(blk + L.in_scen_off);
      for (int32_t k = a; k <= b; k++) so[k - a] = h_scen_off[k] - sa;
    }
    std::memcpy(blk + rate_at, h_rate + sa, size_t(sb - sa) * 8);
    std::memcpy(blk + rate_at + int64_t(sb - sa) * 8, h_bound + sa, size_t(sb - sa) * 8);
    std::memcpy(blk + table_at, h_table + sa, size_t(n_tab) * 2);
    off += blk_bytes;
  }
  return off;
}

// ------------------------------------------------------------ host pack pool
// A small persistent pool of host threads for parva_stream_pack_arrays: the
// caller's thread takes part, workers sleep on a condition variable between
// calls (no OpenMP runtime next to torch's).
namespace {
// Workers spin (pause) for a while after each call before sleeping on a
// condition variable: a pipelined caller packs a batch every ~50-100 us, and
// a futex wake-up of every worker per call cost ~55 us on the B200 host.
// A call's parameters live in one of two job records (by generation); a
// worker registers in the record (active) before re-checking that the
// generation is still current, so a call never returns -- and its record is
// never rewritten -- while a worker still reads it.
class PackPool {
 public:
  explicit PackPool(int n) {
    const char* e = std::getenv("PARVA_PACK_SPIN_US");
    spin_us_ = e ? std::max(0, std::atoi(e)) : 2000;
    for (int i = 0; i < n; i++) th_.emplace_back([this] { worker(); });
  }
  ~PackPool() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> lk(mu_);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  // fn(task) for task in [0, n_tasks), on up to `width` threads (caller included)
  void run(int n_tasks, int width, const std::function<void(int)>& fn) {
    if (width <= 1 || n_tasks <= 1 || th_.empty()) {   // the caller alone: no handshake at all
      for (int i = 0; i < n_tasks; i++) fn(i);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);   // one call at a time
    const uint64_t g = gen_.load() + 1;
    Job& J = jobs_[g & 1];
    while (J.active.load() != 0) spin_pause();      // (a stale worker of generation g - 2 leaving)
    J.fn = &fn;
    J.n_tasks = n_tasks;
    J.width = std::min(width - 1, n_tasks - 1);
    J.next.store(0);
    J.taken.store(0);
    J.remaining.store(n_tasks);
    gen_.store(g);
    if (sleepers_.load() > 0) {
      std::lock_guard<std::mutex> lk(mu_);
      cv_.notify_all();
    }
    drain(J);
    // every task is done; a worker still leaving drain() reads only this
    // record's counters, and the record is reused two calls later, after
    // its active count has dropped to zero (above)
    while (J.remaining.load() != 0) spin_pause();
  }

 private:
  struct Job {
    const std::function<void(int)>* fn = nullptr;
    int n_tasks = 0, width = 0;
    std::atomic<int> next{0}, taken{0}, remaining{0}, active{0};
  };
  static void spin_pause() { __builtin_ia32_pause(); }
  static void drain(Job& J) {
    for (;;) {
      const int i = J.next.fetch_add(1);
      if (i >= J.n_tasks) return;
      (*J.fn)(i);
      J.remaining.fetch_sub(1);
    }
  }
  void worker() {
    uint64_t seen = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      uint64_t g;
      for (int k = 0; (g = gen_.load()) == seen && !stop_.load(); k++) {
        spin_pause();
        if ((k & 4095) == 4095) std::this_thread::yield();   // cede the core if another thread wants it
        if ((k & 255) == 255 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(spin_us_)) {
          std::unique_lock<std::mutex> lk(mu_);
          sleepers_.fetch_add(1);
          cv_.wait(lk, [&] { return gen_.load() != seen || stop_.load(); });
          sleepers_.fetch_sub(1);
        }
      }
      if (stop_.load()) return;
      seen = g;
      Job& J = jobs_[g & 1];
      J.active.fetch_add(1);
      if (gen_.load() == g && J.taken.fetch_add(1) < J.width) drain(J);
      J.active.fetch_sub(1);
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_;
  Job jobs_[2];
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> sleepers_{0};
  std::atomic<bool> stop_{false};
  int spin_us_ = 2000;
};

PackPool& pack_pool() {
  // default: all cores but two (the calling thread takes part in every
  // pack; one more core stays free for a thread waiting on the GPU -- the
  // workers spin, and an oversubscribed core stalls a whole pack for a
  // scheduler quantum)
  // cores: this process's CPU affinity; with one process per GPU
  // (LOCAL_WORLD_SIZE from torchrun) and no launcher pinning, its share
  static PackPool pool([] {
    const char* e = std::getenv("PARVA_PACK_THREADS");
    const int all = (int)std::thread::hardware_concurrency();
    int hw = all;
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0 && CPU_COUNT(&set) > 0) hw = CPU_COUNT(&set);
    const char* lw = std::getenv("LOCAL_WORLD_SIZE");
    const int ranks = (lw && *lw) ? std::max(1, std::atoi(lw)) : 1;
    if (hw >= all && ranks > 1) hw = std::max(1, hw / ranks);
    int n = (e && *e) ? std::atoi(e) : hw - 1;
    return std::max(0, std::min(n, 64) - 1);
  }());
  return pool;
}
}  // namespace

// copy into pinned memory; with PARVA_PACK_NT=1 non-temporal 16-byte stores
// (no read-for-ownership of the destination; A/B switch)
static bool pack_nt() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("PARVA_PACK_NT");
    v = (e && *e == '1') ? 1 : 0;
  }
  return v == 1;
}
static void pack_copy(void* dst, const void* src, size_t bytes) {
  uint8_t* d = (uint8_t*)dst;
  const uint8_t* p = (const uint8_t*)src;
  if (!pack_nt() || ((uintptr_t)d & 15)) {
    std::memcpy(d, p, bytes);
    return;
  }
  size_t i = 0;
  for (; i + 64 <= bytes; i += 64) {
    const __m128i a = _mm_loadu_si128((const __m128i*)(p + i));
    const __m128i b = _mm_loadu_si128((const __m128i*)(p + i + 16));
    const __m128i c = _mm_loadu_si128((const __m128i*)(p + i + 32));
    const __m128i e = _mm_loadu_si128((const __m128i*)(p + i + 48));
    _mm_stream_si128((__m128i*)(d + i), a);
    _mm_stream_si128((__m128i*)(d + i + 16), b);
    _mm_stream_si128((__m128i*)(d + i + 32), c);
    _mm_stream_si128((__m128i*)(d + i + 48), e);
  }
  for (; i + 16 <= bytes; i += 16) _mm_stream_si128((__m128i*)(d + i), _mm_loadu_si128((const __m128i*)(p + i)));
  if (i < bytes) std::memcpy(d + i, p + i, bytes - i);
}

// Streamed input block from plain arrays (int32 table ids), multi-threaded:
// pass 1 sizes every chunk (template detection), a prefix sum places them,
// pass 2 writes the header and the chunk blocks.  Table ids outside
// [0, 65535) are stored as 0xFFFF (no table: the kernel reports
// PARVA_BAD_INPUT for the service, as for any id >= n_tables).
int64_t parva_stream_pack_arrays(int32_t n_scenarios, const int32_t* h_scen_off, const int32_t* h_table,
                                 const double* h_rate, const double* h_bound, int32_t chunk_scen, void* h_block,
                                 int64_t capacity, int32_t n_threads) {
  if (n_scenarios < 0 || !h_scen_off || chunk_scen < 1 || !h_block || capacity < 16) return -1;
  if (n_scenarios > 0 && (!h_table || !h_rate || !h_bound || h_scen_off[0] != 0)) return -1;
  const int32_t n_ch = n_scenarios == 0 ? 0 : (n_scenarios + chunk_scen - 1) / chunk_scen;
  PackPool& pool = pack_pool();
  const int width = n_threads > 0 ? std::min(n_threads, pool.size()) : pool.size();
  constexpr int kChunksPerTask = 4;
  const int n_tasks = (n_ch + kChunksPerTask - 1) / kChunksPerTask;
  std::vector<int64_t> blk(n_ch + 1, 0);
  std::vector<int32_t> tmpl(n_ch, 0);
  std::atomic<int> bad{0};
  // pass 1: offsets valid, template?, block bytes
  pool.run(n_tasks, width, [&](int task) {
    for (int32_t c = task * kChunksPerTask; c < std::min(n_ch, (task + 1) * kChunksPerTask); c++) {
      const int32_t a = c * chunk_scen, b = std::min(n_scenarios, a + chunk_scen);
      for (int32_t k = a; k < b; k++)
        if (h_scen_off[k + 1] < h_scen_off[k]) { bad.store(1); return; }
      const int32_t sa = h_scen_off[a], sb = h_scen_off[b];
      const int32_t t0 = h_scen_off[a + 1] - sa;
      bool tm = t0 > 0 && b - a > 1;
      for (int32_t k = a + 1; tm && k < b; k++) {
        const int32_t ka = h_scen_off[k];
        tm = h_scen_off[k + 1] - ka == t0 && std::memcmp(h_table + ka, h_table + sa, size_t(t0) * 4) == 0;
      }
      const int64_t m = sb - sa;
      const int64_t rate_at = tm ? 0 : ((int64_t)(b - a + 1) * 4 + 15) & ~int64_t(15);
      const int64_t table_at = rate_at + m * 16;
      tmpl[c] = tm ? t0 : 0;
      blk[c + 1] = (table_at + (tm ? t0 : m) * 2 + 15) & ~int64_t(15);
    }
  });
  if (bad.load()) return -1;
  const int64_t head = parva_stream_header_bytes(n_ch);
  blk[0] = head;
  for (int32_t c = 0; c < n_ch; c++) blk[c + 1] += blk[c];   // blk[c] = offset of chunk c
  const int64_t total = blk[n_ch];
  if (total > capacity) return -1;
  uint8_t* out = (uint8_t*)h_block;
  std::memset(out, 0, (size_t)head);
  reinterpret_cast<int32_t*>(out)[0] = n_ch;
  reinterpret_cast<int32_t*>(out)[1] = chunk_scen;
  parva_stream_chunk* tab = reinterpret_cast<parva_stream_chunk*>(out + 16);
  // pass 2: chunk table entries and blocks
  pool.run(n_tasks, width, [&](int task) {
    for (int32_t c = task * kChunksPerTask; c < std::min(n_ch, (task + 1) * kChunksPerTask); c++) {
      const int32_t a = c * chunk_scen, b = std::min(n_scenarios, a + chunk_scen);
      const int32_t sa = h_scen_off[a], sb = h_scen_off[b];
      const int64_t m = sb - sa;
      const bool tm = tmpl[c] > 0;
      tab[c].scen_lo = a; tab[c].svc_lo = sa; tab[c].k = b - a; tab[c].m = (int32_t)m; tab[c].offset = blk[c];
      tab[c].tmpl = tmpl[c]; tab[c].reserved = 0;
      uint8_t* p = out + blk[c];
      const int64_t rate_at = tm ? 0 : ((int64_t)(b - a + 1) * 4 + 15) & ~int64_t(15);
      if (!tm) {
        int32_t* so = reinterpret_cast<int32_t*>(p);
        for (int32_t k = a; k <= b; k++) so[k - a] = h_scen_off[k] - sa;
        std::memset(p + int64_t(b - a + 1) * 4, 0, size_t(rate_at - int64_t(b - a + 1) * 4));
      }
      pack_copy(p + rate_at, h_rate + sa, size_t(m) * 8);
      pack_copy(p + rate_at + m * 8, h_bound + sa, size_t(m) * 8);
      uint16_t* t16 = reinterpret_cast<uint16_t*>(p + rate_at + m * 16);
      const int64_t nt = tm ? tmpl[c] : m;
      for (int64_t i = 0; i < nt; i++) {
        const int32_t v = h_table[sa + i];
        t16[i] = (v < 0 || v >= 65535) ? (uint16_t)0xFFFF : (uint16_t)v;
      }
      const int64_t end = rate_at + m * 16 + nt * 2;
      std::memset(p + end, 0, size_t(blk[c + 1] - blk[c] - end));
    }
    if (pack_nt()) _mm_sfence();
  });
  return total;
}

// scratch head: work counters, slice flags
static size_t mapped_head_bytes(int64_t n_slices) {
  return up256(size_t(parva::kWorkWords) * 4) + up256(size_t(n_slices) * 4);
}

size_t parva_plan_host_mapped_scratch(int64_t in_bytes) {
  if (in_bytes < 0) return 0;
  const int64_t n_slices = (in_bytes + parva::kStreamSlice - 1) / parva::kStreamSlice;
  return 256 + mapped_head_bytes(n_slices) + up256(size_t(in_bytes));
}

// (device, pointer) -> device address of a pinned block, or the pointer
// itself for device memory; pageable memory is rejected.  A small cache of
// the blocks used last keeps cudaPointerGetAttributes off the per-call path.
struct MappedPtr {
  int dev = -1;
  const void* p = nullptr;
  void* d = nullptr;
  bool host = false;
};
static MappedPtr g_mapped_ptrs[8];
static unsigned g_mapped_ptr_next = 0;
static std::mutex g_mapped_mu;

static bool mapped_ptr(int dev, const void* p, void** d, bool* host) {
  {
    std::lock_guard<std::mutex> lock(g_mapped_mu);
    for (const auto& e : g_mapped_ptrs)
      if (e.dev == dev && e.p == p) { *d = e.d; *host = e.host; return true; }
  }
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  *host = at.type == cudaMemoryTypeHost;
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) *d = const_cast<void*>(p);
  else if (at.type != cudaMemoryTypeHost) return false;      // pageable memory cannot be mapped
  else if (cudaHostGetDevicePointer(d, const_cast<void*>(p), 0) != cudaSuccess) { cudaGetLastError(); return false; }
  std::lock_guard<std::mutex> lock(g_mapped_mu);
  MappedPtr& e = g_mapped_ptrs[g_mapped_ptr_next++ % 8];
  e.dev = dev; e.p = p; e.d = *d; e.host = *host;
  return true;
}

// scratch -> its call slot: the epoch of its slice flags (flags hold the
// epoch of the call that wrote them), and for asynchronous calls a completion
// word in pinned host memory (the kernel stores the epoch of each finished
// call) plus the epoch last submitted, so a new call on the same scratch
// first waits for the previous one
struct MappedSlot {
  int dev = -1;
  void* scratch = nullptr;
  size_t bytes = 0;
  uint32_t epoch = 0;
  uint32_t submitted = 0;       // epoch of the last asynchronous call (0 = none)
  cudaStream_t stream = nullptr;
  const void* h_out = nullptr;  // output block of the last call
  const void* h_in = nullptr;   // input block of the last call
  uint32_t* d_done = nullptr;   // device address of its completion word
};
constexpr int kMappedSlots = 1024;
static std::vector<MappedSlot> g_mapped_slots;
static uint32_t* g_done_host = nullptr;   // kMappedSlots completion words (pinned, mapped, portable)

// Forget a block or scratch (call before freeing it, so a later allocation at
// the same address is looked up again and a scratch's flags are re-zeroed).
void parva_forget_block(const void* p) {
  {
    std::lock_guard<std::mutex> lock(g_mapped_mu);
    for (auto& e : g_mapped_ptrs)
      if (e.p == p) e = MappedPtr{};
  }
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (auto& e : g_mapped_slots)
    if (e.scratch == p) e = MappedSlot{};
}

static bool done_reached(uint32_t slot, uint32_t epoch) {
  const uint32_t v = *reinterpret_cast<volatile uint32_t*>(g_done_host + slot);
  return (int32_t)(v - epoch) >= 0;
}

// Spin until the call (slot, epoch) has published completion; the stream is
// queried now and then so a failed launch cannot hang the host.
static int wait_done(uint32_t slot, uint32_t epoch, cudaStream_t s) {
  for (uint64_t i = 0;; i++) {
    __builtin_ia32_pause();
    if (done_reached(slot, epoch)) {
      std::atomic_thread_fence(std::memory_order_acquire);
      return PARVA_OK;
    }
    if ((i & 4095) == 4095) {
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) return done_reached(slot, epoch) ? PARVA_OK : PARVA_LAUNCH_ERROR;
      if (e != cudaErrorNotReady) return PARVA_LAUNCH_ERROR;
    }
  }
}

static int plan_host_mapped(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                            int32_t n_services, const void* h_in, int64_t in_bytes, void* h_out, int32_t optimize,
                            int32_t threshold, int32_t cfg_format, int32_t plan_bytes, void* d_scratch,
                            size_t scratch_bytes, void* stream, uint64_t* ticket) {
  if (ticket) *ticket = 0;
  if (!tables || !index || !h_in || !h_out || !d_scratch || n_scenarios < 0 || n_services < 0 || in_bytes < 16 ||
      in_bytes % 16 != 0 || int64_t(n_scenarios) > in_bytes / 4)
    return PARVA_BAD_INPUT;
  parva_chunk_layout L;
  if (parva_mapped_layout(n_scenarios, n_services, cfg_format, plan_bytes, &L) != PARVA_OK) return PARVA_BAD_INPUT;
  const size_t need = parva_plan_host_mapped_scratch(in_bytes);
  if (need == 0 || need > scratch_bytes) return PARVA_BAD_INPUT;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0;
  cudaGetDevice(&dev);
  // pinned host blocks are mapped to device addresses (device blocks are used
  // as they are); the lookup of the last blocks used is cached per device
  bool in_host = false, out_host = false;
  void* d_in = nullptr;
  void* d_out = nullptr;
  if (!mapped_ptr(dev, h_in, &d_in, &in_host) || !mapped_ptr(dev, h_out, &d_out, &out_host)) return PARVA_BAD_INPUT;
  if (!in_host) return PARVA_BAD_INPUT;   // the streamed input block must be pinned host memory
  uint8_t* base = (uint8_t*)(((uintptr_t)d_scratch + 255) & ~uintptr_t(255));
  const int64_t n_slices = (in_bytes + parva::kStreamSlice - 1) / parva::kStreamSlice;
  uint32_t* work = (uint32_t*)base;
  uint32_t* flags = (uint32_t*)(base + up256(size_t(parva::kWorkWords) * 4));
  const size_t head = mapped_head_bytes(n_slices);
  uint8_t* staging = base + head;
  uint32_t epoch = 0, slot = 0, pending = 0;
  uint32_t* d_done = nullptr;
  cudaStream_t pending_stream = nullptr;
  struct Busy { uint32_t slot, epoch; cudaStream_t stream; };
  std::vector<Busy> out_busy;
  {
    std::lock_guard<std::mutex> lock(g_graph_mu);
    if (ticket && !g_done_host) {
      void* p = nullptr;
      if (cudaHostAlloc(&p, kMappedSlots * 4, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
        return PARVA_LAUNCH_ERROR;
      std::memset(p, 0, kMappedSlots * 4);
      g_done_host = (uint32_t*)p;
    }
    int E = -1, free_slot = -1;
    for (int i = 0; i < (int)g_mapped_slots.size(); i++) {
      const auto& e = g_mapped_slots[i];
      if (e.dev == dev && e.scratch == d_scratch && e.bytes == scratch_bytes) { E = i; break; }
      if (!e.scratch && free_slot < 0) free_slot = i;
    }
    if (E < 0 || g_mapped_slots[E].epoch == 0xFFFFFFFFu) {
      // first use of this scratch: zero the counters and flags
      if (E >= 0 && g_mapped_slots[E].submitted &&
          wait_done((uint32_t)E, g_mapped_slots[E].submitted, g_mapped_slots[E].stream) != PARVA_OK)
        return PARVA_LAUNCH_ERROR;
      if (cudaStreamSynchronize(s) != cudaSuccess || cudaMemset(base, 0, head) != cudaSuccess)
        return PARVA_LAUNCH_ERROR;
      if (E < 0) E = free_slot;
      if (E < 0) {
        if ((int)g_mapped_slots.size() >= kMappedSlots) return PARVA_CAPACITY;
        g_mapped_slots.emplace_back();
        E = (int)g_mapped_slots.size() - 1;
      }
      MappedSlot& M = g_mapped_slots[E];
      M = MappedSlot{};
      M.dev = dev; M.scratch = d_scratch; M.bytes = scratch_bytes;
      if (g_done_host) g_done_host[E] = 0;
    }
    // an unfinished call on another scratch that writes the same output
    // block must complete first too (two calls never write one block at once)
    for (int i = 0; i < (int)g_mapped_slots.size(); i++) {
      const MappedSlot& e = g_mapped_slots[i];
      if (i != E && e.h_out == h_out && e.submitted && !done_reached((uint32_t)i, e.submitted))
        out_busy.push_back({(uint32_t)i, e.submitted, e.stream});
    }
    MappedSlot& M = g_mapped_slots[E];
    slot = (uint32_t)E;
    pending = M.submitted;
    pending_stream = M.stream;
    epoch = ++M.epoch;
    M.h_out = h_out;
    M.h_in = h_in;
    if (ticket) { M.submitted = epoch; M.stream = s; }
    else M.submitted = 0;
  }
  // one call in flight per scratch and per output block: an unfinished
  // asynchronous call on either must complete first
  if (pending && wait_done(slot, pending, pending_stream) != PARVA_OK) return PARVA_LAUNCH_ERROR;
  for (const auto& b : out_busy)
    if (wait_done(b.slot, b.epoch, b.stream) != PARVA_OK) return PARVA_LAUNCH_ERROR;
  if (ticket) {
    {
      std::lock_guard<std::mutex> lock(g_graph_mu);
      d_done = g_mapped_slots[slot].d_done;
    }
    if (!d_done) {
      if (cudaHostGetDevicePointer((void**)&d_done, g_done_host + slot, 0) != cudaSuccess) {
        cudaGetLastError();
        return PARVA_LAUNCH_ERROR;
      }
      std::lock_guard<std::mutex> lock(g_graph_mu);
      g_mapped_slots[slot].d_done = d_done;
    }
  }
  if (n_scenarios > 0) {
    uint8_t* out = (uint8_t*)d_out;
    parva::PlanArgs A;
    A.pts = tables->d_pts; A.idx_lat = index->d_lat_sorted; A.idx_best = index->d_best; A.idx_tp = index->d_tp;
    A.seg_start = tables->d_seg_start; A.seg_count = tables->d_seg_count; A.n_tables = tables->n_tables;
    A.n_points = tables->n_points; A.max_seg_points = tables->max_seg_points;
    A.n_scen = n_scenarios; A.n_svc = n_services;
    A.scen_off = nullptr; A.svc_table = nullptr; A.svc_table16 = nullptr; A.svc_rate = nullptr; A.svc_bound = nullptr;
    A.optimize = optimize; A.threshold = threshold; A.cfg_given = 0;
    A.smem_index = tables->n_points * 18 <= (int64_t)kSmemIndexLimit;
    A.cfg = out + L.out_cfg; A.cfg_format = cfg_format;
    A.plan = (parva_plan_record*)(out + L.out_plan);
    A.plan_bytes = plan_bytes; A.spill_cap = L.spill_cap;
    A.spill_count = nullptr;
    A.spill = out + L.out_spill;
    A.spill_direct = 1;
    A.work = work;
    A.stream_src = (const uint8_t*)d_in;
    A.stream_dst = staging;
    A.stream_bytes = in_bytes;
    A.slice_flag = flags;
    A.epoch = epoch;
    A.n_loaders = loaders_for(in_bytes);
    A.done_word = d_done;
    A.pdl = ticket ? 1 : 0;
    const int rc = parva::launch_plan_batch(A, s);
    if (rc != PARVA_OK) {
      if (ticket) {   // nothing will complete this epoch
        std::lock_guard<std::mutex> lock(g_graph_mu);
        g_mapped_slots[slot].submitted = 0;
      }
      return rc;
    }
  } else if (ticket) {
    g_done_host[slot] = epoch;     // nothing to launch: complete at once (host store, in submission order)
  }
  if (ticket) {
    *ticket = (uint64_t)slot << 32 | epoch;
    return PARVA_OK;
  }
  return cudaStreamSynchronize(s) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
}

int parva_plan_host_mapped(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                           int32_t n_services, const void* h_in, int64_t in_bytes, void* h_out, int32_t optimize,
                           int32_t threshold, int32_t cfg_format, int32_t plan_bytes, void* d_scratch,
                           size_t scratch_bytes, void* stream) {
  return plan_host_mapped(tables, index, n_scenarios, n_services, h_in, in_bytes, h_out, optimize, threshold,
                          cfg_format, plan_bytes, d_scratch, scratch_bytes, stream, nullptr);
}

int parva_plan_host_mapped_submit(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                                  int32_t n_services, const void* h_in, int64_t in_bytes, void* h_out,
                                  int32_t optimize, int32_t threshold, int32_t cfg_format, int32_t plan_bytes,
                                  void* d_scratch, size_t scratch_bytes, void* stream, uint64_t* ticket) {
  if (!ticket) return PARVA_BAD_INPUT;
  return plan_host_mapped(tables, index, n_scenarios, n_services, h_in, in_bytes, h_out, optimize, threshold,
                          cfg_format, plan_bytes, d_scratch, scratch_bytes, stream, ticket);
}

// Pack + submit in one call: waits for any unfinished call still reading
// h_in (the block is rewritten here), packs the caller's plain arrays into it
// on the pack pool, then submits as parva_plan_host_mapped_submit.
int parva_plan_host_arrays_submit(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                                  const int32_t* h_scen_off, const int32_t* h_table, const double* h_rate,
                                  const double* h_bound, int32_t chunk_scen, void* h_in, int64_t in_capacity,
                                  void* h_out, int32_t optimize, int32_t threshold, int32_t cfg_format,
                                  int32_t plan_bytes, void* d_scratch, size_t scratch_bytes, void* stream,
                                  uint64_t* ticket) {
  if (!ticket || !h_in || !h_scen_off || n_scenarios < 0) return PARVA_BAD_INPUT;
  *ticket = 0;
  struct Busy { uint32_t slot, epoch; cudaStream_t stream; };
  std::vector<Busy> busy;
  {
    std::lock_guard<std::mutex> lock(g_graph_mu);
    for (int i = 0; i < (int)g_mapped_slots.size(); i++) {
      const MappedSlot& e = g_mapped_slots[i];
      if (e.h_in == h_in && e.submitted && g_done_host && !done_reached((uint32_t)i, e.submitted))
        busy.push_back({(uint32_t)i, e.submitted, e.stream});
    }
  }
  for (const auto& b : busy)
    if (wait_done(b.slot, b.epoch, b.stream) != PARVA_OK) return PARVA_LAUNCH_ERROR;
  const int64_t in_bytes = parva_stream_pack_arrays(n_scenarios, h_scen_off, h_table, h_rate, h_bound, chunk_scen,
                                                    h_in, in_capacity, 0);
  if (in_bytes < 0) return PARVA_BAD_INPUT;
  const int32_t n_services = n_scenarios ? h_scen_off[n_scenarios] : 0;
  return plan_host_mapped(tables, index, n_scenarios, n_services, h_in, in_bytes, h_out, optimize, threshold,
                          cfg_format, plan_bytes, d_scratch, scratch_bytes, stream, ticket);
}

int parva_plan_host_mapped_wait(uint64_t ticket) {
  const uint32_t slot = (uint32_t)(ticket >> 32), epoch = (uint32_t)ticket;
  if (epoch == 0) return PARVA_OK;                  // an empty call's ticket
  cudaStream_t s = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_graph_mu);
    if (!g_done_host || slot >= g_mapped_slots.size()) return PARVA_BAD_INPUT;
    s = g_mapped_slots[slot].stream;
  }
  return wait_done(slot, epoch, s);
}

size_t parva_plan_general_workspace(const parva_general_problem* p, int32_t gpu_cap) {
  return parva::general_workspace(p, gpu_cap);
}

int parva_plan_general(const parva_general_problem* p, parva_general_result* r, void* d_workspace,
                       size_t workspace_bytes, void* stream) {
  if (!p || !r) return PARVA_BAD_INPUT;
  return parva::launch_plan_general(p, r, d_workspace, workspace_bytes, (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------- simulator seeding
// numpy's SeedSequence(seed).spawn(n)[i] -> default_rng(child) PCG64 state,
// restated (numpy/random/bit_generator.pyx: SeedSequence.mix_entropy,
// generate_state; _pcg64.pyx / pcg64.h: pcg64_set_seed -> pcg64_srandom_r).
// Host code: replaces ~11 us of Python object construction per service.
namespace {
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16, kPool = 4;

inline uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> kXShift;
  return v;
}
inline uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kXShift;
  return r;
}
}  // namespace

int parva_sim_seed_states(const uint32_t* seed_words, int32_t n_seed_words, int64_t first_child, int64_t n_children,
                          uint64_t* out) {
  if (!seed_words || n_seed_words < 1 || n_seed_words > 64 || first_child < 0 || n_children < 0 || !out)
    return PARVA_BAD_INPUT;
  typedef unsigned __int128 u128;
  const u128 kMult = ((u128)0x2360ed051fc65da4ull << 64) | 0x4385df649fccf645ull;
  uint32_t ent[80];
  for (int64_t c = 0; c < n_children; c++) {
    // assembled entropy: run entropy (zero-padded to the pool size, since a
    // spawn key follows), then the spawn key (child index as uint32 words)
    int ne = 0;
    for (int i = 0; i < n_seed_words; i++) ent[ne++] = seed_words[i];
    while (ne < kPool) ent[ne++] = 0u;
    uint64_t key = (uint64_t)(first_child + c);
    if (key == 0) ent[ne++] = 0u;
    while (key) { ent[ne++] = (uint32_t)key; key >>= 32; }
    // mix_entropy
    uint32_t pool[kPool];
    uint32_t h = kInitA;
    for (int i = 0; i < kPool; i++) pool[i] = hashmix(i < ne ? ent[i] : 0u, h);
    for (int s = 0; s < kPool; s++)
      for (int d = 0; d < kPool; d++)
        if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], h));
    for (int s = kPool; s < ne; s++)
      for (int d = 0; d < kPool; d++) pool[d] = mixw(pool[d], hashmix(ent[s], h));
    // generate_state(4, uint64): 8 uint32 words from the cycled pool
    uint32_t w[8];
    uint32_t hb = kInitB;
    for (int i = 0; i < 8; i++) {
      uint32_t v = pool[i % kPool];
      v ^= hb;
      hb *= kMultB;
      v *= hb;
      v ^= v >> kXShift;
      w[i] = v;
    }
    uint64_t val[4];
    for (int k = 0; k < 4; k++) val[k] = (uint64_t)w[2 * k] | (uint64_t)w[2 * k + 1] << 32;
    // pcg64_srandom_r(initstate = val[0]:val[1], initseq = val[2]:val[3])
    const u128 initstate = ((u128)val[0] << 64) | val[1];
    const u128 initseq = ((u128)val[2] << 64) | val[3];
    const u128 inc = (initseq << 1) | 1u;
    u128 st = 0;
    st = st * kMult + inc;
    st += initstate;
    st = st * kMult + inc;
    out[4 * c + 0] = (uint64_t)(st >> 64);
    out[4 * c + 1] = (uint64_t)st;
    out[4 * c + 2] = (uint64_t)(inc >> 64);
    out[4 * c + 3] = (uint64_t)inc;
  }
  return PARVA_OK;
}
