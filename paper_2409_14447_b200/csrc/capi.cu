// capi.cu — the extern "C" boundary declared in include/parva_b200.h.
#include <cuda_runtime.h>

#include "parva_common.cuh"
#include "parva_kernels.cuh"


static constexpr size_t kSmemIndexLimit = 150 * 1024;  // index bytes kept in shared memory

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

static int plan_batch_impl(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                           const int32_t* d_scen_off, const int32_t* d_svc_table, const double* d_svc_rate,
                           const double* d_svc_bound, int32_t optimize, int32_t threshold,
                           parva_config_record* d_cfg, parva_plan_record* d_plan, double* d_ledger_val,
                           uint8_t* d_ledger_order, int cfg_given, cudaStream_t stream) {
  parva::PlanArgs A;
  A.pts = tables->d_pts;
  A.idx_lat = index ? index->d_lat_sorted : nullptr;
  A.idx_best = index ? index->d_best : nullptr;
  A.idx_tp = index ? index->d_tp : nullptr;
  A.seg_start = tables->d_seg_start;
  A.seg_count = tables->d_seg_count;
  A.n_tables = tables->n_tables;
  A.n_points = tables->n_points;
  A.n_scen = n_scenarios;
  A.scen_off = d_scen_off;
  A.svc_table = d_svc_table;
  A.svc_rate = d_svc_rate;
  A.svc_bound = d_svc_bound;
  A.optimize = optimize;
  A.threshold = threshold;
  A.cfg_given = cfg_given;
  A.smem_index = !cfg_given && tables->n_points * 18 <= (int64_t)kSmemIndexLimit;
  A.cfg = d_cfg;
  A.plan = d_plan;
  A.ledger_val = d_ledger_val;
  A.ledger_order = d_ledger_order;
  return parva::launch_plan_batch(A, stream);
}

int parva_plan_batch(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                     const int32_t* d_scen_off, const int32_t* d_svc_table, const double* d_svc_rate,
                     const double* d_svc_bound, int32_t optimize, int32_t threshold,
                     parva_config_record* d_cfg, parva_plan_record* d_plan, double* d_ledger_val,
                     uint8_t* d_ledger_order, void* stream) {
  if (!tables || n_scenarios < 0 || !d_cfg || !d_plan) return PARVA_BAD_INPUT;
  const int cfg_given = index == nullptr;
  if (cfg_given) return PARVA_BAD_INPUT;
  return plan_batch_impl(tables, index, n_scenarios, d_scen_off, d_svc_table, d_svc_rate, d_svc_bound,
                         optimize, threshold, d_cfg, d_plan, d_ledger_val, d_ledger_order, 0,
                         (cudaStream_t)stream);
}

// Same as parva_plan_batch but the config records in d_cfg were produced by
// parva_configure_sweep (tables too large for the shared-memory index).
int parva_plan_batch_preconfigured(const parva_tables* tables, int32_t n_scenarios, const int32_t* d_scen_off,
                                   const int32_t* d_svc_table, int32_t optimize, int32_t threshold,
                                   parva_config_record* d_cfg, parva_plan_record* d_plan,
                                   double* d_ledger_val, uint8_t* d_ledger_order, void* stream) {
  if (!tables || n_scenarios < 0 || !d_cfg || !d_plan) return PARVA_BAD_INPUT;
  return plan_batch_impl(tables, nullptr, n_scenarios, d_scen_off, d_svc_table, nullptr, nullptr, optimize,
                         threshold, d_cfg, d_plan, d_ledger_val, d_ledger_order, 1, (cudaStream_t)stream);
}

size_t parva_plan_host_scratch(int32_t n_scenarios, int32_t n_services) {
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  return up(size_t(n_scenarios + 1) * 4) + up(size_t(n_services) * 4) + 2 * up(size_t(n_services) * 8) +
         up(size_t(n_services) * sizeof(parva_config_record)) + up(size_t(n_scenarios) * sizeof(parva_plan_record));
}

int parva_plan_host(const parva_tables* tables, const parva_index* index, int32_t n_scenarios,
                    const int32_t* h_scen_off, const int32_t* h_svc_table, const double* h_svc_rate,
                    const double* h_svc_bound, int32_t optimize, int32_t threshold, parva_config_record* h_cfg,
                    parva_plan_record* h_plan, void* d_scratch, size_t scratch_bytes, void* stream) {
  if (!tables || !index || n_scenarios < 0) return PARVA_BAD_INPUT;
  const int32_t n_services = h_scen_off[n_scenarios];
  if (parva_plan_host_scratch(n_scenarios, n_services) > scratch_bytes) return PARVA_BAD_INPUT;
  cudaStream_t s = (cudaStream_t)stream;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint8_t* p = (uint8_t*)d_scratch;
  int32_t* d_off = (int32_t*)p; p += up(size_t(n_scenarios + 1) * 4);
  int32_t* d_tab = (int32_t*)p; p += up(size_t(n_services) * 4);
  double* d_rate = (double*)p; p += up(size_t(n_services) * 8);
  double* d_bound = (double*)p; p += up(size_t(n_services) * 8);
  parva_config_record* d_cfg = (parva_config_record*)p; p += up(size_t(n_services) * sizeof(parva_config_record));
  parva_plan_record* d_plan = (parva_plan_record*)p;
  cudaMemcpyAsync(d_off, h_scen_off, size_t(n_scenarios + 1) * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_tab, h_svc_table, size_t(n_services) * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_rate, h_svc_rate, size_t(n_services) * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_bound, h_svc_bound, size_t(n_services) * 8, cudaMemcpyHostToDevice, s);
  int rc = plan_batch_impl(tables, index, n_scenarios, d_off, d_tab, d_rate, d_bound, optimize, threshold, d_cfg,
                           d_plan, nullptr, nullptr, 0, s);
  if (rc != PARVA_OK) return rc;
  cudaMemcpyAsync(h_cfg, d_cfg, size_t(n_services) * sizeof(parva_config_record), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h_plan, d_plan, size_t(n_scenarios) * sizeof(parva_plan_record), cudaMemcpyDeviceToHost, s);
  return cudaStreamSynchronize(s) == cudaSuccess ? PARVA_OK : PARVA_LAUNCH_ERROR;
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
