// capi.cu -- the C ABI (include/graphmat_b200.h).  Every entry point catches
// the library's exceptions and turns them into a gm_status plus a thread-local
// message, the way the reference CLI maps InputError/EngineError to exit codes
// (tools/sgraph.cpp:24, 293-354).
#include <string>
#include <vector>

#include "api_internal.cuh"
#include "dist.cuh"

namespace gm {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launches_so_far() { return g_launches.load(); }
}  // namespace gm

namespace {

thread_local std::string g_last_error;

template <typename F>
gm_status guarded(F&& f) {
  try {
    f();
    return GM_OK;
  } catch (const gm::Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return GM_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GM_EENGINE;
  }
}

gm::Graph* handle(gm_graph_t g) {
  if (!g) gm::fail(GM_EUSAGE, "null graph handle");
  return reinterpret_cast<gm::Graph*>(g);
}

void copy_stats(const std::vector<gm_iteration_stats>& st, gm_iteration_stats* out, int64_t cap,
                int64_t* n_out) {
  if (n_out) *n_out = int64_t(st.size());
  if (!out) return;
  for (size_t i = 0; i < st.size() && int64_t(i) < cap; ++i) out[i] = st[i];
}

}  // namespace

extern "C" {

GM_API const char* gm_last_error(void) { return g_last_error.c_str(); }

GM_API const char* gm_version(void) { return "graphmat_b200 0.1 (sm_100a)"; }

GM_API uint64_t gm_kernel_launches(void) { return gm::g_launches.load(); }

GM_API gm_status gm_graph_create(const gm_edge_list* edges, uint64_t num_vertices, uint32_t flags,
                                 int32_t value_storage, gm_graph_t* out) {
  return guarded([&] {
    if (!edges || !out) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_graph_t>(gm::graph_create(*edges, num_vertices, flags, value_storage));
  });
}

GM_API gm_status gm_graph_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b,
                                        double c, uint64_t seed, int32_t permute, uint32_t flags,
                                        int32_t weights, gm_graph_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_graph_t>(
        gm::graph_generate_rmat(scale, edge_factor, a, b, c, seed, permute, flags, weights));
  });
}

GM_API gm_status gm_graph_generate_bipartite(uint32_t users, uint32_t items, double c_numerator,
                                             uint32_t cap, uint64_t seed, uint32_t flags,
                                             gm_graph_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_graph_t>(
        gm::graph_generate_bipartite(users, items, c_numerator, cap, seed, flags));
  });
}

GM_API gm_status gm_graph_destroy(gm_graph_t g) {
  return guarded([&] { gm::graph_destroy(reinterpret_cast<gm::Graph*>(g)); });
}

GM_API gm_status gm_graph_get_info(gm_graph_t g, gm_graph_info* info) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (!info) gm::fail(GM_EUSAGE, "null info");
    info->num_vertices = h->n;
    info->num_edges = h->m;
    info->flags = h->flags;
    info->value_type = h->value_type;
    info->forward_built = h->out_built ? 1 : 0;
    info->device = h->device;
    info->device_bytes = h->device_bytes();
    info->nonzero_out_degree = h->nonzero_outdeg;
  });
}

GM_API gm_status gm_graph_ensure_forward(gm_graph_t g) {
  return guarded([&] { gm::ensure_forward(*handle(g)); });
}

GM_API gm_status gm_graph_export_edges(gm_graph_t g, uint32_t* src, uint32_t* dst, void* values) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if ((!src || !dst) && h->m) gm::fail(GM_EUSAGE, "null output arrays");
    gm::export_edges(*h, src, dst, values);
  });
}

GM_API gm_status gm_degree_vector(gm_graph_t g, int32_t kind, uint64_t* out) {
  return guarded([&] {
    if (kind != 0 && kind != 1) gm::fail(GM_EUSAGE, "degree kind must be 0 (IN) or 1 (OUT)");
    gm::degree_vector(*handle(g), kind, out);
  });
}

GM_API gm_status gm_pick_source(gm_graph_t g, uint64_t seed, uint64_t* out) {
  return guarded([&] { *out = gm::pick_source(*handle(g), seed); });
}

GM_API void* gm_graph_stream(gm_graph_t g) {
  return g ? reinterpret_cast<void*>(reinterpret_cast<gm::Graph*>(g)->stream) : nullptr;
}

GM_API gm_status gm_graph_synchronize(gm_graph_t g) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    GM_CUDA(cudaStreamSynchronize(h->stream));
    h->host_async.sync();
  });
}

// ---- multi-GPU: communicator + sharded graph ----------------------------------
namespace {
gm::Comm* comm_of(gm_comm_t c) {
  if (!c) gm::fail(GM_EUSAGE, "null communicator");
  return reinterpret_cast<gm::Comm*>(c);
}
gm::DGraph* dgraph_of(gm_dgraph_t g) {
  if (!g) gm::fail(GM_EUSAGE, "null sharded graph");
  return reinterpret_cast<gm::DGraph*>(g);
}
}  // namespace

GM_API gm_status gm_comm_create_local(int32_t nshards, const int32_t* devices, gm_comm_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null output");
    *out = reinterpret_cast<gm_comm_t>(gm::comm_create_local(nshards, devices));
  });
}

GM_API gm_status gm_comm_nccl_unique_id(void* id128) {
  return guarded([&] {
    if (!id128) gm::fail(GM_EUSAGE, "null id buffer");
    gm::comm_nccl_unique_id(id128);
  });
}

GM_API gm_status gm_comm_create_nccl(int32_t nranks, int32_t rank, int32_t device,
                                     const void* id128, gm_comm_t* out) {
  return guarded([&] {
    if (!out || !id128) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_comm_t>(gm::comm_create_nccl(nranks, rank, device, id128));
  });
}

GM_API gm_status gm_comm_destroy(gm_comm_t c) {
  return guarded([&] { gm::comm_release(reinterpret_cast<gm::Comm*>(c)); });
}

GM_API gm_status gm_dgraph_generate_rmat(gm_comm_t c, uint32_t scale, uint32_t edge_factor,
                                         double a, double b, double cc, uint64_t seed,
                                         uint32_t flags, int32_t weights, gm_dgraph_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null output");
    *out = reinterpret_cast<gm_dgraph_t>(
        gm::dgraph_generate_rmat(comm_of(c), scale, edge_factor, a, b, cc, seed, flags, weights));
  });
}

GM_API gm_status gm_dgraph_create(gm_comm_t c, const gm_edge_list* edges, uint64_t num_vertices,
                                  uint32_t flags, int32_t value_storage, gm_dgraph_t* out) {
  return guarded([&] {
    if (!out || !edges) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_dgraph_t>(
        gm::dgraph_create(comm_of(c), *edges, num_vertices, flags, value_storage));
  });
}

GM_API gm_status gm_dgraph_destroy(gm_dgraph_t g) {
  return guarded([&] { delete reinterpret_cast<gm::DGraph*>(g); });
}

GM_API gm_status gm_dgraph_shard_info(gm_dgraph_t g, int32_t local_shard, gm_dshard_info* info) {
  return guarded([&] {
    gm::DGraph* d = dgraph_of(g);
    if (!info || local_shard < 0 || local_shard >= d->comm->L) gm::fail(GM_EUSAGE, "bad shard");
    const gm::DShard& s = d->sh[size_t(local_shard)];
    info->num_vertices = d->n;
    info->num_edges = d->m;
    info->row_begin = s.lo;
    info->row_end = s.hi;
    info->local_edges = s.in.nnz;
    info->device_bytes = d->device_bytes(local_shard);
    info->nonzero_out_degree = d->nonzero_outdeg;
    info->shards = d->comm->P;
    info->local_shards = d->comm->L;
    info->first_shard = d->comm->first;
    info->device = d->comm->dev[size_t(local_shard)];
  });
}

GM_API void* gm_dgraph_stream(gm_dgraph_t g, int32_t local_shard) {
  if (!g) return nullptr;
  gm::DGraph* d = reinterpret_cast<gm::DGraph*>(g);
  if (local_shard < 0 || local_shard >= d->comm->L) return nullptr;
  return reinterpret_cast<void*>(d->comm->st[size_t(local_shard)]);
}

GM_API gm_status gm_dgraph_pick_source(gm_dgraph_t g, uint64_t seed, uint64_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null output");
    *out = gm::dpick_source(*dgraph_of(g), seed);
  });
}

GM_API gm_status gm_dgraph_degrees(gm_dgraph_t g, int32_t local_shard, int32_t kind, uint32_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null output");
    gm::ddegrees(*dgraph_of(g), local_shard, kind, out);
  });
}

GM_API gm_status gm_dgraph_bfs(gm_dgraph_t g, uint64_t root, int64_t max_iters, int32_t* out_level,
                               int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                               int64_t* n_stats) {
  return guarded([&] {
    const auto st = gm::dbfs(*dgraph_of(g), root, max_iters, out_level, out_on_device != 0);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_dgraph_sssp(gm_dgraph_t g, uint64_t source, int64_t max_iters,
                                uint32_t* out_dist, int32_t out_on_device,
                                gm_iteration_stats* stats, int64_t cap, int64_t* n_stats) {
  return guarded([&] {
    const auto st = gm::dsssp(*dgraph_of(g), source, max_iters, out_dist, out_on_device != 0);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_dgraph_generate_bipartite(gm_comm_t c, uint32_t users, uint32_t items,
                                              double c_numerator, uint32_t cap, uint64_t seed,
                                              gm_dgraph_t* out) {
  return guarded([&] {
    if (!out) gm::fail(GM_EUSAGE, "null output");
    *out = reinterpret_cast<gm_dgraph_t>(
        gm::dgraph_generate_bipartite(comm_of(c), users, items, c_numerator, cap, seed));
  });
}

GM_API gm_status gm_dgraph_cf(gm_dgraph_t g, const gm_cf_config* cfg, const float* init_factors,
                              float* out_factors, double* rmse_trace, gm_iteration_stats* stats,
                              int64_t cap, int64_t* n_stats) {
  return guarded([&] {
    if (!cfg) gm::fail(GM_EUSAGE, "null config");
    if (cfg->factors_on_device) gm::fail(GM_EUSAGE, "dgraph cf: host factor buffers only");
    const auto st = gm::dcf(*dgraph_of(g), cfg->k, cfg->gamma, cfg->lambda, cfg->iterations,
                            init_factors, out_factors, rmse_trace);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_dgraph_pagerank(gm_dgraph_t g, const gm_pagerank_config* cfg, float* out_rank,
                                    int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                                    int64_t* n_stats) {
  return guarded([&] {
    if (!cfg) gm::fail(GM_EUSAGE, "null config");
    const auto st = gm::dpagerank(*dgraph_of(g), cfg->damping, cfg->iterations, out_rank,
                                  out_on_device != 0);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_kernel_timer_start(gm_graph_t g) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    h->ktimer.on = true;
    h->ktimer.used = 0;
    h->ktimer.name = "";
  });
}

GM_API gm_status gm_kernel_timer_stop(gm_graph_t g, double* total_ms, int64_t* launches,
                                      char* name, size_t name_cap) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    gm::KernelTimer& t = h->ktimer;
    GM_CUDA(cudaStreamSynchronize(h->stream));
    double ms = 0.0;
    for (size_t i = 0; i + 1 < t.used; i += 2) {
      float x = 0.f;
      GM_CUDA(cudaEventElapsedTime(&x, t.ev[i], t.ev[i + 1]));
      ms += x;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = int64_t(t.used / 2);
    if (name && name_cap) {
      std::strncpy(name, t.name, name_cap - 1);
      name[name_cap - 1] = 0;
    }
    t.on = false;
    t.used = 0;
  });
}

namespace {
// out_on_device: GM_OUT_HOST, GM_OUT_DEVICE or GM_OUT_DEVICE_ASYNC (device
// output, no host synchronisation -- so no stats either).
void check_out_mode(int32_t mode, const gm_iteration_stats* stats, const int64_t* n_stats,
                    bool host_async_ok = false) {
  if (mode < GM_OUT_HOST || mode > (host_async_ok ? GM_OUT_HOST_ASYNC : GM_OUT_DEVICE_ASYNC))
    gm::fail(GM_EUSAGE, "bad out_on_device mode");
  if ((mode == GM_OUT_DEVICE_ASYNC || mode == GM_OUT_HOST_ASYNC) && (stats || n_stats))
    gm::fail(GM_EUSAGE, "an async output mode returns before the run ends: pass no stats buffer");
}
}  // namespace

GM_API gm_status gm_pagerank(gm_graph_t g, const gm_pagerank_config* cfg, float* out_rank,
                             int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                             int64_t* n_stats) {
  return guarded([&] {
    if (!cfg) gm::fail(GM_EUSAGE, "null config");
    check_out_mode(out_on_device, stats, n_stats, /*host_async_ok=*/true);
    gm::Graph& G = *handle(g);
    if (out_on_device == GM_OUT_HOST_ASYNC && out_rank && G.n) {
      // the ranks land in a device staging buffer; its copy to the caller's
      // pinned memory runs on the copy stream while the next call computes
      float* stage = static_cast<float*>(G.host_async.stage(G.stream, G.n * 4));
      gm::pagerank(G, cfg->damping, cfg->iterations, stage, true, false, true);
      G.host_async.issue(G.stream, out_rank, G.n * 4);
      return;
    }
    auto st = gm::pagerank(G, cfg->damping, cfg->iterations,
                           out_on_device == GM_OUT_HOST_ASYNC ? nullptr : out_rank,
                           out_on_device != 0, stats != nullptr || n_stats != nullptr,
                           out_on_device >= GM_OUT_DEVICE_ASYNC);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_bfs(gm_graph_t g, uint64_t root, int64_t max_iters, int32_t* out_level,
                        int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                        int64_t* n_stats) {
  return guarded([&] {
    check_out_mode(out_on_device, stats, n_stats, /*host_async_ok=*/true);
    const bool host_async = out_on_device == GM_OUT_HOST_ASYNC;
    auto st = gm::bfs(*handle(g), root, max_iters, out_level,
                      out_on_device != 0 && !host_async, stats != nullptr || n_stats != nullptr,
                      out_on_device == GM_OUT_DEVICE_ASYNC || host_async);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_sssp(gm_graph_t g, uint64_t source, int64_t max_iters, uint32_t* out_dist,
                         int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                         int64_t* n_stats) {
  return guarded([&] {
    check_out_mode(out_on_device, stats, n_stats, /*host_async_ok=*/true);
    gm::Graph& G = *handle(g);
    if (out_on_device == GM_OUT_HOST_ASYNC && out_dist && G.n) {
      uint32_t* stage = static_cast<uint32_t*>(G.host_async.stage(G.stream, G.n * 4));
      gm::sssp(G, source, max_iters, stage, true, false, true);
      G.host_async.issue(G.stream, out_dist, G.n * 4);
      return;
    }
    auto st = gm::sssp(G, source, max_iters, out_on_device == GM_OUT_HOST_ASYNC ? nullptr : out_dist,
                       out_on_device != 0, stats != nullptr || n_stats != nullptr,
                       out_on_device >= GM_OUT_DEVICE_ASYNC);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_cf(gm_graph_t g, const gm_cf_config* cfg, const float* init_factors,
                       float* out_factors, double* rmse_trace, gm_iteration_stats* stats,
                       int64_t cap, int64_t* n_stats) {
  return guarded([&] {
    if (!cfg) gm::fail(GM_EUSAGE, "null config");
    auto st = gm::cf(*handle(g), cfg->k, cfg->gamma, cfg->lambda, cfg->iterations, init_factors,
                     out_factors, rmse_trace, cfg->factors_on_device != 0);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_triangle_count(gm_graph_t g, uint64_t* total, uint64_t* local_counts) {
  return guarded([&] {
    if (!total) gm::fail(GM_EUSAGE, "null argument");
    *total = gm::triangle_count(*handle(g), local_counts);
  });
}

GM_API gm_status gm_edges_load_text(const char* path, int32_t weighted, gm_edges_t* out) {
  return guarded([&] {
    if (!path || !out) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_edges_t>(new gm::EdgeBuffer(gm::io::load_edge_list(path, weighted != 0)));
  });
}

GM_API gm_status gm_edges_load_matrix_market(const char* path, gm_edges_t* out) {
  return guarded([&] {
    if (!path || !out) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_edges_t>(new gm::EdgeBuffer(gm::io::load_matrix_market(path)));
  });
}

GM_API gm_status gm_edges_read_binary(const char* path, gm_edges_t* out) {
  return guarded([&] {
    if (!path || !out) gm::fail(GM_EUSAGE, "null argument");
    *out = reinterpret_cast<gm_edges_t>(new gm::EdgeBuffer(gm::io::read_binary(path)));
  });
}

GM_API gm_status gm_edges_view(gm_edges_t e, uint64_t* num_vertices, uint64_t* num_edges,
                               const uint64_t** src, const uint64_t** dst, const double** values) {
  return guarded([&] {
    if (!e) gm::fail(GM_EUSAGE, "null edge buffer");
    const auto* b = reinterpret_cast<const gm::EdgeBuffer*>(e);
    if (num_vertices) *num_vertices = b->num_vertices;
    if (num_edges) *num_edges = b->src.size();
    if (src) *src = b->src.data();
    if (dst) *dst = b->dst.data();
    if (values) *values = b->val.data();
  });
}

GM_API gm_status gm_edges_free(gm_edges_t e) {
  return guarded([&] { delete reinterpret_cast<gm::EdgeBuffer*>(e); });
}

GM_API gm_status gm_edges_write_binary(const char* path, const uint64_t* src, const uint64_t* dst,
                                       const double* values, uint64_t num_edges,
                                       uint64_t num_vertices) {
  return guarded([&] {
    if (!path || (num_edges && (!src || !dst))) gm::fail(GM_EUSAGE, "null argument");
    gm::io::write_binary(path, src, dst, values, num_edges, num_vertices);
  });
}

GM_API gm_status gm_edges_write_text(const char* path, const uint64_t* src, const uint64_t* dst,
                                     const double* values, uint64_t num_edges) {
  return guarded([&] {
    if (!path || (num_edges && (!src || !dst))) gm::fail(GM_EUSAGE, "null argument");
    gm::io::write_edge_list(path, src, dst, values, num_edges);
  });
}

GM_API gm_status gm_write_results(const char* path, const double* values, uint64_t n) {
  return guarded([&] {
    if (!path || (n && !values)) gm::fail(GM_EUSAGE, "null argument");
    gm::io::write_results(path, values, n);
  });
}

GM_API gm_status gm_write_vector_results(const char* path, const double* rows, uint64_t n,
                                         uint64_t k) {
  return guarded([&] {
    if (!path || (n && k && !rows)) gm::fail(GM_EUSAGE, "null argument");
    gm::io::write_vector_results(path, rows, n, k);
  });
}

GM_API gm_status gm_write_report(const char* path, const gm_run_report* report) {
  return guarded([&] {
    if (!path || !report) gm::fail(GM_EUSAGE, "null argument");
    if ((report->n_iterations && !report->iteration_seconds) ||
        (report->n_extras && (!report->extra_keys || !report->extra_values)))
      gm::fail(GM_EUSAGE, "null report arrays");
    gm::io::write_report(path, *report);
  });
}

GM_API gm_status gm_measure_fp32_fma(double* tflops) {
  return guarded([&] {
    if (!tflops) gm::fail(GM_EUSAGE, "null argument");
    *tflops = gm::measure_fp32_fma();
  });
}

GM_API uint64_t gm_fnv1a64(const void* data, uint64_t size) {
  return gm::io::fnv1a64(data, data ? size : 0);
}

GM_API gm_status gm_fnv1a64_file(const char* path, uint64_t* out) {
  return guarded([&] {
    if (!path || !out) gm::fail(GM_EUSAGE, "null argument");
    *out = gm::io::fnv1a64_file(path);
  });
}

GM_API gm_status gm_program_sizes(int32_t program, size_t* vertex_bytes, size_t* message_bytes,
                                  size_t* reduced_bytes) {
  return guarded([&] { gm::program_sizes(program, vertex_bytes, message_bytes, reduced_bytes); });
}

GM_API gm_status gm_run_graph_program(gm_graph_t g, int32_t program, const double* params,
                                      void* props, uint8_t* active, int64_t max_iters,
                                      gm_iteration_stats* stats, int64_t cap, int64_t* n_stats) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (h->n && (!props || !active)) gm::fail(GM_EUSAGE, "null property / activity arrays");
    auto st = gm::run_program(*h, program, params, props, active, max_iters);
    copy_stats(st, stats, cap, n_stats);
  });
}

GM_API gm_status gm_superstep_phases(gm_graph_t g, int32_t program, const double* params,
                                     const void* props, const uint8_t* active, void* x,
                                     uint8_t* x_valid, int32_t run_spmv, void* y,
                                     uint8_t* y_valid) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (h->n && (!props || !active)) gm::fail(GM_EUSAGE, "null property / activity arrays");
    gm::superstep_phases(*h, program, params, props, active, x, x_valid, run_spmv, y, y_valid);
  });
}

GM_API gm_status gm_graph_permutation(gm_graph_t g, uint32_t* caller_to_internal) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (!caller_to_internal && h->n) gm::fail(GM_EUSAGE, "null output");
    if (h->relabeled) {
      GM_CUDA(cudaMemcpy(caller_to_internal, h->perm.get(), h->n * 4, cudaMemcpyDeviceToHost));
    } else {
      for (uint64_t v = 0; v < h->n; ++v) caller_to_internal[v] = uint32_t(v);
    }
  });
}

GM_API gm_status gm_graph_csr(gm_graph_t g, int32_t which, const uint64_t** ptr_dev,
                              const uint32_t** idx_dev, uint64_t* rows, uint64_t* nnz) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (which != 0 && which != 1) gm::fail(GM_EUSAGE, "csr: which must be 0 (G^T) or 1 (G)");
    if (!ptr_dev || !idx_dev || !rows || !nnz) gm::fail(GM_EUSAGE, "null argument");
    if (which == 1) gm::ensure_forward(*h);
    const gm::Csr& c = which == 1 ? h->fwd() : h->in;
    *ptr_dev = c.ptr.get();
    *idx_dev = c.idx.get();
    *rows = h->n;
    *nnz = c.nnz;
  });
}

GM_API gm_status gm_pagerank_shard_init(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                        float* x_block_dev, double* dangling_block) {
  return guarded([&] {
    const double d = gm::pagerank_shard_init(*handle(g), row_begin, row_end, x_block_dev);
    if (dangling_block) *dangling_block = d;
  });
}

GM_API gm_status gm_pagerank_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                        const float* x_full_dev, double base, double damping,
                                        float* x_block_dev, double* dangling_block) {
  return guarded([&] {
    const double d = gm::pagerank_shard_step(*handle(g), row_begin, row_end, x_full_dev, base,
                                             damping, x_block_dev);
    if (dangling_block) *dangling_block = d;
  });
}

GM_API gm_status gm_pagerank_shard_step_peers(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                              const float* x_full_dev, double base, double damping,
                                              const uint64_t* peer_buffers, int32_t npeers,
                                              int64_t offset, uint64_t limit,
                                              double* dangling_block) {
  return guarded([&] {
    if (!peer_buffers || npeers < 1) gm::fail(GM_EUSAGE, "null peer buffers");
    std::vector<float*> peers(static_cast<size_t>(npeers));
    for (int32_t q = 0; q < npeers; ++q) peers[q] = reinterpret_cast<float*>(peer_buffers[q]);
    const double d = gm::pagerank_shard_step_peers(*handle(g), row_begin, row_end, x_full_dev,
                                                   base, damping, peers.data(), npeers, offset,
                                                   limit);
    if (dangling_block) *dangling_block = d;
  });
}

GM_API gm_status gm_pagerank_shard_init_peers(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                              const uint64_t* peer_buffers, int32_t npeers,
                                              int64_t offset, uint64_t limit,
                                              double* dangling_block) {
  return guarded([&] {
    if (!peer_buffers || npeers < 1) gm::fail(GM_EUSAGE, "null peer buffers");
    std::vector<float*> peers(static_cast<size_t>(npeers));
    for (int32_t q = 0; q < npeers; ++q) peers[q] = reinterpret_cast<float*>(peer_buffers[q]);
    const double d = gm::pagerank_shard_init_peers(*handle(g), row_begin, row_end, peers.data(),
                                                   npeers, offset, limit);
    if (dangling_block) *dangling_block = d;
  });
}

GM_API gm_status gm_ipc_alloc(uint64_t bytes, void** dev_ptr) {
  return guarded([&] {
    if (!dev_ptr) gm::fail(GM_EUSAGE, "null output");
    *dev_ptr = nullptr;
    GM_CUDA(cudaMalloc(dev_ptr, bytes ? bytes : 1));
  });
}

GM_API gm_status gm_ipc_free(void* dev_ptr) {
  return guarded([&] {
    if (dev_ptr) GM_CUDA(cudaFree(dev_ptr));
  });
}

GM_API gm_status gm_ipc_handle(void* dev_ptr, void* handle64) {
  return guarded([&] {
    if (!dev_ptr || !handle64) gm::fail(GM_EUSAGE, "null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
    cudaIpcMemHandle_t h;
    GM_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    memcpy(handle64, &h, 64);
  });
}

GM_API gm_status gm_ipc_open(const void* handle64, void** dev_ptr) {
  return guarded([&] {
    if (!handle64 || !dev_ptr) gm::fail(GM_EUSAGE, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    *dev_ptr = nullptr;
    GM_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

GM_API gm_status gm_ipc_close(void* dev_ptr) {
  return guarded([&] {
    if (dev_ptr) GM_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  });
}

GM_API gm_status gm_pagerank_shard_ranks(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                         float* ranks_block_host) {
  return guarded([&] { gm::pagerank_shard_ranks(*handle(g), row_begin, row_end, ranks_block_host); });
}

GM_API gm_status gm_pagerank_shard_active(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                          uint64_t* prefix_len) {
  return guarded([&] {
    if (!prefix_len) gm::fail(GM_EUSAGE, "null argument");
    *prefix_len = gm::pagerank_shard_active(*handle(g), row_begin, row_end);
  });
}

GM_API gm_status gm_pagerank_shard_pack(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                        uint64_t block_stride, uint64_t lmax) {
  return guarded(
      [&] { gm::pagerank_shard_pack(*handle(g), row_begin, row_end, block_stride, lmax); });
}

GM_API gm_status gm_bfs_shard_init(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                   uint64_t root_internal) {
  return guarded([&] { gm::bfs_shard_init(*handle(g), row_begin, row_end, root_internal); });
}

GM_API gm_status gm_bfs_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                   const uint32_t* frontier_dev, const uint32_t* visited_dev,
                                   int32_t level, int32_t pull, uint32_t* next_block_dev,
                                   uint64_t* found, uint64_t* found_edges) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (h->n && (!frontier_dev || !visited_dev || (row_end > row_begin && !next_block_dev)))
      gm::fail(GM_EUSAGE, "null bitmap");
    gm::bfs_shard_step(*h, row_begin, row_end, frontier_dev, visited_dev, level, pull,
                       next_block_dev, found, found_edges);
  });
}

GM_API gm_status gm_cf_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end, int32_t k,
                                  const float* factors_full_dev, float gamma, float lambda,
                                  float* factors_block_dev, double* sq_err_sum, uint64_t* changed) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (h->n && (!factors_full_dev || (row_end > row_begin && !factors_block_dev)))
      gm::fail(GM_EUSAGE, "null factors");
    gm::cf_shard_step(*h, row_begin, row_end, k, factors_full_dev, gamma, lambda,
                      factors_block_dev, sq_err_sum, changed);
  });
}

GM_API gm_status gm_sssp_shard_init(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                    uint64_t root_internal) {
  return guarded([&] { gm::sssp_shard_init(*handle(g), row_begin, row_end, root_internal); });
}

GM_API gm_status gm_sssp_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                    const uint32_t* msg_dev, int32_t pull, uint32_t* msg_block_dev,
                                    uint64_t* changed, uint64_t* changed_edges) {
  return guarded([&] {
    gm::Graph* h = handle(g);
    if (h->n && (!msg_dev || (row_end > row_begin && !msg_block_dev)))
      gm::fail(GM_EUSAGE, "null message vector");
    gm::sssp_shard_step(*h, row_begin, row_end, msg_dev, pull, msg_block_dev, changed,
                        changed_edges);
  });
}

GM_API gm_status gm_sssp_shard_dists(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                     uint32_t* dist_block_host) {
  return guarded([&] {
    if (!dist_block_host && row_end > row_begin) gm::fail(GM_EUSAGE, "null output");
    gm::sssp_shard_dists(*handle(g), row_begin, row_end, dist_block_host);
  });
}

GM_API gm_status gm_bfs_shard_push(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                   const uint32_t* next_block_dev, const uint64_t* peer_bitmaps,
                                   int32_t npeers) {
  return guarded([&] {
    if (!peer_bitmaps || npeers < 1) gm::fail(GM_EUSAGE, "null peer bitmaps");
    if (row_end > row_begin && !next_block_dev) gm::fail(GM_EUSAGE, "null bitmap");
    std::vector<uint32_t*> peers(static_cast<size_t>(npeers));
    for (int32_t q = 0; q < npeers; ++q) peers[q] = reinterpret_cast<uint32_t*>(peer_bitmaps[q]);
    gm::bfs_shard_push(*handle(g), row_begin, row_end, next_block_dev, peers.data(), npeers);
  });
}

GM_API gm_status gm_push_block(gm_graph_t g, const void* src_dev, uint64_t bytes,
                               const uint64_t* peer_buffers, int32_t npeers, uint64_t dst_offset) {
  return guarded([&] {
    if (!peer_buffers || npeers < 1) gm::fail(GM_EUSAGE, "null peer buffers");
    if (bytes && !src_dev) gm::fail(GM_EUSAGE, "null source block");
    std::vector<void*> peers(static_cast<size_t>(npeers));
    for (int32_t q = 0; q < npeers; ++q) peers[q] = reinterpret_cast<void*>(peer_buffers[q]);
    gm::push_block(*handle(g), src_dev, bytes, peers.data(), npeers, dst_offset);
  });
}

GM_API gm_status gm_bitmap_or(gm_graph_t g, uint32_t* dst_dev, const uint32_t* src_dev,
                              uint64_t words) {
  return guarded([&] {
    if (words && (!dst_dev || !src_dev)) gm::fail(GM_EUSAGE, "null bitmap");
    gm::bitmap_or(*handle(g), dst_dev, src_dev, words);
  });
}

GM_API gm_status gm_bfs_shard_levels(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                     int32_t* levels_block_host) {
  return guarded([&] {
    if (!levels_block_host && row_end > row_begin) gm::fail(GM_EUSAGE, "null output");
    gm::bfs_shard_levels(*handle(g), row_begin, row_end, levels_block_host);
  });
}

// detail::balanced_row_boundaries (dcsc.hpp:81-105): boundary p is the smallest
// row i with cum(i) * parts >= p * total.
GM_API gm_status gm_balanced_row_boundaries(const uint64_t* row_nnz, uint64_t n, uint64_t parts,
                                            uint64_t* bounds) {
  return guarded([&] {
    if (parts == 0) gm::fail(GM_EUSAGE, "parts must be positive");
    std::vector<uint64_t> cum(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) cum[i + 1] = cum[i] + row_nnz[i];
    const uint64_t total = cum[n];
    bounds[0] = 0;
    bounds[parts] = n;
    for (uint64_t p = 1; p < parts; ++p) {
      const unsigned __int128 target = (unsigned __int128)p * total;
      uint64_t lo = bounds[p - 1], hi = n;
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if ((unsigned __int128)cum[mid] * parts >= target)
          hi = mid;
        else
          lo = mid + 1;
      }
      bounds[p] = lo;
    }
  });
}

}  // extern "C"
