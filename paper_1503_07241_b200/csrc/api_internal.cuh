// api_internal.cuh -- C++ entry points behind the C ABI (capi.cu).
#pragma once

#include <vector>

#include "graph.cuh"

namespace gm {

// generic_programs.cu
void program_sizes(int prog, size_t* v, size_t* m, size_t* r);
std::vector<gm_iteration_stats> run_program(Graph& g, int prog, const double* params, void* props,
                                            uint8_t* active, int64_t max_iters);
void superstep_phases(Graph& g, int prog, const double* params, const void* props,
                      const uint8_t* active, void* x, uint8_t* x_valid, int run_spmv, void* y,
                      uint8_t* y_valid);

// pagerank.cu
std::vector<gm_iteration_stats> pagerank(Graph& g, double damping, int64_t iters, float* out,
                                         bool out_on_device, bool collect_stats,
                                         bool async = false);
// pagerank_hub.cu: the single-GPU default (pagerank() dispatches to it)
bool pagerank_hub_enabled(const Graph& g);
std::vector<gm_iteration_stats> pagerank_hub(Graph& g, double damping, int64_t iters, float* out,
                                             bool out_on_device, bool collect_stats,
                                         bool async = false);
double pagerank_shard_init(Graph& g, uint64_t lo, uint64_t hi, float* x_block);
double pagerank_shard_step(Graph& g, uint64_t lo, uint64_t hi, const float* x_full, double base,
                           double damping, float* x_block);
void pagerank_shard_ranks(Graph& g, uint64_t lo, uint64_t hi, float* out_host);
uint64_t pagerank_shard_active(Graph& g, uint64_t lo, uint64_t hi);
double pagerank_shard_init_peers(Graph& g, uint64_t lo, uint64_t hi, float* const* peers,
                                 int npeers, int64_t offset, uint64_t limit);
double pagerank_shard_step_peers(Graph& g, uint64_t lo, uint64_t hi, const float* x_full,
                                 double base, double damping, float* const* peers, int npeers,
                                 int64_t offset, uint64_t limit);
void bfs_shard_init(Graph& g, uint64_t lo, uint64_t hi, uint64_t root_internal);
void bfs_shard_step(Graph& g, uint64_t lo, uint64_t hi, const uint32_t* frontier,
                    const uint32_t* visited, int32_t lvl, int32_t pull, uint32_t* next_block,
                    uint64_t* found, uint64_t* found_edges);
void bfs_shard_levels(Graph& g, uint64_t lo, uint64_t hi, int32_t* out_host);
void push_block(Graph& g, const void* src, uint64_t bytes, void* const* peers, int npeers,
                uint64_t dst_offset);
void bitmap_or(Graph& g, uint32_t* dst, const uint32_t* src, uint64_t words);
void bfs_shard_push(Graph& g, uint64_t lo, uint64_t hi, const uint32_t* next_block,
                    uint32_t* const* peers, int npeers);
void cf_shard_step(Graph& g, uint64_t lo, uint64_t hi, int64_t k, const float* f_full, float gamma,
                   float lambda, float* f_block, double* sq_sum, uint64_t* changed);
void sssp_shard_init(Graph& g, uint64_t lo, uint64_t hi, uint64_t root_internal);
void sssp_shard_step(Graph& g, uint64_t lo, uint64_t hi, const uint32_t* msg, int32_t pull,
                     uint32_t* msg_block, uint64_t* changed, uint64_t* changed_edges);
void sssp_shard_dists(Graph& g, uint64_t lo, uint64_t hi, uint32_t* out_host);
void pagerank_shard_pack(Graph& g, uint64_t lo, uint64_t hi, uint64_t stride, uint64_t lmax);
// traversal.cu
std::vector<gm_iteration_stats> bfs(Graph& g, uint64_t root, int64_t max_iters, int32_t* out,
                                    bool out_on_device, bool collect_stats,
                                         bool async = false);
std::vector<gm_iteration_stats> sssp(Graph& g, uint64_t root, int64_t max_iters, uint32_t* out,
                                     bool out_on_device, bool collect_stats,
                                         bool async = false);
// cf.cu
uint64_t triangle_count(Graph& g, uint64_t* local_host);

// Files (gmio.cu): the reference's formats, host side.
struct EdgeBuffer {
  std::vector<uint64_t> src, dst;
  std::vector<double> val;
  uint64_t num_vertices = 0;
};
namespace io {
EdgeBuffer load_edge_list(const std::string& path, bool weighted);
EdgeBuffer load_matrix_market(const std::string& path);
EdgeBuffer read_binary(const std::string& path);
void write_binary(const std::string& path, const uint64_t* src, const uint64_t* dst,
                  const double* val, uint64_t m, uint64_t n);
void write_edge_list(const std::string& path, const uint64_t* src, const uint64_t* dst,
                     const double* val, uint64_t m);
void write_results(const std::string& path, const double* values, uint64_t n);
void write_vector_results(const std::string& path, const double* rows, uint64_t n, uint64_t k);
void write_report(const std::string& path, const gm_run_report& r);
uint64_t fnv1a64(const void* data, uint64_t size);
uint64_t fnv1a64_file(const std::string& path);
}  // namespace io
double measure_fp32_fma();
std::vector<gm_iteration_stats> cf(Graph& g, int64_t k, float gamma, float lambda, int64_t iters,
                                   const float* init, float* out, double* rmse_trace,
                                   bool on_device = false);


}  // namespace gm
