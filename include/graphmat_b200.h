/*
 * graphmat_b200.h -- C ABI of the B200-native GraphMat superstep backend.
 *
 * The reference (semigraph, /root/reference/proj) exposes its superstep path as
 * C++20 templates only (no C ABI, no FFI).  Each entry point below replaces one
 * reference interface; the citation is the reference file:line it stands in for
 * (paths relative to /root/reference/proj).  All pointers are plain host pointers
 * unless the matching *_on_device flag is set.  The library copies its inputs,
 * owns every device allocation and never retains caller pointers.
 *
 * Errors: every call returns a gm_status; gm_last_error() returns the message
 * of the last failure on the calling thread.  Codes mirror the reference CLI's
 * exit codes (tools/sgraph.cpp:24): usage 1, InputError 2, EngineError 3.
 *
 * Threading: one handle is driven by one host thread at a time (the reference
 * Engine is not re-entrant either, include/semigraph/engine.hpp:55-57).
 */
#ifndef GRAPHMAT_B200_H
#define GRAPHMAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GM_API __attribute__((visibility("default")))
#else
#define GM_API
#endif

typedef enum {
  GM_OK = 0,
  GM_EUSAGE = 1,  /* bad arguments / API misuse            (sgraph.cpp:24 usage)       */
  GM_EINPUT = 2,  /* semigraph::InputError                  (core.hpp:44-50)            */
  GM_EENGINE = 3, /* semigraph::EngineError                 (core.hpp:52-57)            */
  GM_ECUDA = 4,   /* CUDA runtime failure                                              */
  GM_ENCCL = 5    /* NCCL failure (multi-GPU sharding)                                 */
} gm_status;

typedef struct gm_graph* gm_graph_t;

typedef enum { GM_ID_U32 = 0, GM_ID_U64 = 1 } gm_id_type;

/* Edge value storage types.  The reference stores EdgeTriple<E>::value
 * (core.hpp:35-42); the device stores the narrowest type the program needs. */
typedef enum {
  GM_VAL_NONE = 0,
  GM_VAL_F64 = 1,
  GM_VAL_F32 = 2,
  GM_VAL_U8 = 3,
  GM_VAL_I64 = 4,
  GM_VAL_U32 = 5
} gm_value_type;

/* Structure-of-arrays edge list; replaces std::span<const EdgeTriple<E>>
 * (dcsc.hpp:243-245).  Ids are 0-based like the library side of the reference. */
typedef struct {
  const void* src;
  const void* dst;
  const void* values; /* may be NULL (every edge gets value 1, like unweighted loads) */
  int64_t count;
  int32_t id_type;    /* gm_id_type */
  int32_t value_type; /* gm_value_type of `values` as passed */
  int32_t on_device;  /* 1: src/dst/values are device pointers */
  int32_t reserved;
} gm_edge_list;

enum {
  GM_PREPROCESS = 1u,   /* io::preprocess cleanup: drop self loops, dedup keep-first (io.cpp:184-196) */
  GM_SYMMETRIZE = 2u,   /* PreprocessMode::SYMMETRIZE (io.cpp:198-204); implies GM_PREPROCESS      */
  GM_RELABEL = 4u,      /* internal degree-ordered vertex ids (results stay in caller ids)          */
  GM_NEED_FORWARD = 8u, /* build CSR(G) eagerly (Graph::ensure_forward, dcsc.hpp:201-215)           */
  GM_DAGIFY = 16u,      /* PreprocessMode::DAGIFY (io.cpp:198-207): symmetrize, keep src < dst      */
  GM_BIPARTITE_CHECK = 32u /* PreprocessMode::BIPARTITE_CHECK (io.cpp:208-219): reject an edge whose
                              source is a destination or destination a source; GM_EINPUT          */
};
/* With GM_RELABEL, GM_SHARDS(P) deals the degree-ordered vertices round-robin
 * over P equal contiguous row blocks (internal id = (k % P) * N/P + k / P for
 * degree rank k), so block r = [r*N/P, (r+1)*N/P) of G^T carries ~1/P of the
 * nonzeros: the 1-D row partition of dcsc.hpp:77-105 for P GPUs.  N % P == 0. */
#define GM_SHARDS(p) ((uint32_t)(p) << 16)

/* Mirrors semigraph::IterationStats (engine.hpp:32-39) plus device counters. */
typedef struct {
  int64_t iteration;
  int64_t active_before;
  int64_t messages_generated;
  int64_t vertices_updated;
  double spmv_seconds;
  double total_seconds;
  int64_t edges_processed;   /* adjacency entries read by the SpMV / SpMSpV        */
  int64_t bytes_algorithmic; /* DESIGN.md formula for the kernel that ran          */
  int32_t direction;         /* 0 = pull SpMV over G^T, 1 = push SpMSpV over G     */
  int32_t reserved;
  double comm_seconds;       /* sharded runs: exchange + barrier time of the step  */
} gm_iteration_stats;

typedef struct {
  uint64_t num_vertices;
  uint64_t num_edges;
  uint32_t flags;
  int32_t value_type;
  int32_t forward_built;
  int32_t device;
  uint64_t device_bytes;
  uint64_t nonzero_out_degree;
} gm_graph_info;

GM_API const char* gm_last_error(void);
GM_API const char* gm_version(void);
/* Process-wide count of this library's kernel launches (benchmark evidence). */
GM_API uint64_t gm_kernel_launches(void);

/* ---- graph construction: replaces build_graph (dcsc.hpp:243-274) and, with
 *      GM_PREPROCESS / GM_SYMMETRIZE, io::preprocess (io.cpp:184-222). ----------
 * Rejects out-of-range endpoints and, without GM_PREPROCESS, duplicate edges
 * with the reference's messages (dcsc.hpp:252-256, 148-150).  value_storage
 * selects the device value type (GM_VAL_NONE drops values). */
GM_API gm_status gm_graph_create(const gm_edge_list* edges, uint64_t num_vertices,
                                 uint32_t flags, int32_t value_storage, gm_graph_t* out);
/* Seeded R-MAT (semantics of io::rmat_generate,
 * io.cpp:224-255, made counter-based + permuted) generated and ingested on the
 * GPU.  weights = GM_VAL_U8 attaches seeded integer weights in [1,255]. */
GM_API gm_status gm_graph_generate_rmat(uint32_t scale, uint32_t edge_factor, double a,
                                        double b, double c, uint64_t seed, int32_t permute,
                                        uint32_t flags, int32_t weights, gm_graph_t* out);
/* Seeded Zipf bipartite rating graph (stands in for io::bipartite_generate,
 * io.cpp:257-288): users [0,U), items [U,U+I), uint8 ratings in 1..5. */
GM_API gm_status gm_graph_generate_bipartite(uint32_t users, uint32_t items,
                                             double c_numerator, uint32_t cap, uint64_t seed,
                                             uint32_t flags, gm_graph_t* out);
GM_API gm_status gm_graph_destroy(gm_graph_t g);
GM_API gm_status gm_graph_get_info(gm_graph_t g, gm_graph_info* info);
/* Graph::ensure_forward (dcsc.hpp:201-215). */
GM_API gm_status gm_graph_ensure_forward(gm_graph_t g);
/* The stored edge list in caller ids, sorted by (src, dst): the same list
 * io::preprocess returns (io.cpp:184-222).  values typed by the storage type. */
GM_API gm_status gm_graph_export_edges(gm_graph_t g, uint32_t* src, uint32_t* dst,
                                       void* values);
/* degree_vector (engine.hpp:295-312); kind 0 = IN, 1 = OUT. */
GM_API gm_status gm_degree_vector(gm_graph_t g, int32_t kind, uint64_t* out);
/* Seed-chosen vertex with nonzero out-degree (BASELINE configs[1..2]). */
GM_API gm_status gm_pick_source(gm_graph_t g, uint64_t seed, uint64_t* out);
/* The cudaStream_t every call on this handle is issued on (for event timing). */
GM_API void* gm_graph_stream(gm_graph_t g);
/* Wait for every call issued on this handle (see GM_OUT_DEVICE_ASYNC). */
GM_API gm_status gm_graph_synchronize(gm_graph_t g);
/* Measurement: CUDA-event timing of each launch of the handle's dominant
 * kernel (k_bfs_coop, k_pr_hub / k_pr_spmv, the SSSP / CF superstep kernels)
 * between _start and _stop; _stop synchronises and returns the summed
 * duration, the number of timed launches and the kernel's name.  No reference
 * counterpart: the reference times whole supersteps (engine.hpp:177-188). */
GM_API gm_status gm_kernel_timer_start(gm_graph_t g);
GM_API gm_status gm_kernel_timer_stop(gm_graph_t g, double* total_ms, int64_t* launches,
                                      char* name, size_t name_cap);

/* out_on_device of gm_pagerank / gm_bfs / gm_sssp:
 *   GM_OUT_HOST         the output pointer is host memory; returns when written;
 *   GM_OUT_DEVICE       device memory; returns when written;
 *   GM_OUT_DEVICE_ASYNC device memory; returns once the run is enqueued on
 *                       gm_graph_stream(g) (like a cuBLAS call): read the
 *                       output after gm_graph_synchronize or a stream wait.
 *                       Stats need the host, so stats/n_stats must be null. */
#define GM_OUT_HOST 0
#define GM_OUT_DEVICE 1
#define GM_OUT_DEVICE_ASYNC 2
/*   GM_OUT_HOST_ASYNC   host memory, pinned by the caller; returns once
 *                       the run and the copy into it are enqueued: the copy
 *                       runs on a second stream from a double-buffered device
 *                       staging area, so it overlaps the next call's kernels
 *                       (read the output after gm_graph_synchronize). */
#define GM_OUT_HOST_ASYNC 3

/* ---- fast programs (specialised kernels) --------------------------------- */
typedef struct {
  double damping;     /* BASELINE: 0.85                          */
  int64_t iterations; /* fixed supersteps, all vertices active   */
} gm_pagerank_config;

/* Normalised PageRank (BASELINE configs[0]); the reference program shape is
 * PageRankProgram (algorithms/pagerank.hpp:36-63) driven like the CF driver
 * (algorithms/collaborative_filtering.hpp:181-193). out_rank: n floats. */
GM_API gm_status gm_pagerank(gm_graph_t g, const gm_pagerank_config* cfg, float* out_rank,
                             int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                             int64_t* n_stats);
/* algo::bfs (algorithms/traversal.hpp:119-123): int32 level, -1 unreached.
 * Direction-optimising push/pull; pull when frontier edges > alpha * m. */
GM_API gm_status gm_bfs(gm_graph_t g, uint64_t root, int64_t max_iters, int32_t* out_level,
                        int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                        int64_t* n_stats);
/* algo::sssp (algorithms/traversal.hpp:125-133) on integer weights:
 * uint32 distance, UINT32_MAX unreached. */
GM_API gm_status gm_sssp(gm_graph_t g, uint64_t source, int64_t max_iters, uint32_t* out_dist,
                         int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                         int64_t* n_stats);

typedef struct {
  int64_t k;
  float gamma;
  float lambda;
  int64_t iterations;
  int32_t factors_on_device; /* 1: init_factors / out_factors are device pointers */
  int32_t reserved;
} gm_cf_config;
/* collaborative_filtering_gd (algorithms/collaborative_filtering.hpp:134-211)
 * in fp32.  init_factors / out_factors: n*k floats (row-major, caller ids).
 * rmse_trace[it] = RMSE over ratings after iteration it. */
GM_API gm_status gm_cf(gm_graph_t g, const gm_cf_config* cfg, const float* init_factors,
                       float* out_factors, double* rmse_trace, gm_iteration_stats* stats,
                       int64_t cap, int64_t* n_stats);

/* algo::triangle_count (algorithms/triangle_count.hpp:115-134) on a DAG-form
 * graph (every stored edge src < dst in caller ids; build with GM_DAGIFY):
 * total triangles, and optionally TriangleState::local_count per vertex
 * (host array of n, caller order): local[w] = sum over stored v -> w of
 * |N_in(v) & N_in(w)|.  A stored edge with src >= dst is GM_EINPUT with the
 * reference's message ("... violates src < dst; run DAGIFY preprocessing first"). */
GM_API gm_status gm_triangle_count(gm_graph_t g, uint64_t* total, uint64_t* local_counts);

/* Measurement helper (bench.py's CF roofline): sustained FP32 FMA
 * throughput of this GPU in TFLOP/s (2 flops per FMA). */
GM_API gm_status gm_measure_fp32_fma(double* tflops);

/* ---- files: the reference's formats (src/io.cpp, src/report.cpp) --------- */
/* Host-side edge buffer: caller ids (0-based) as u64, values as f64 (1.0 for
 * unweighted inputs), num_vertices as the reference's EdgeList reports it. */
typedef struct gm_edges_s* gm_edges_t;
/* io::load_edge_list (io.cpp:85-110): "src dst [weight]" lines, 1-based ids,
 * '#'/'%' comments; InputError messages carry path:line. */
GM_API gm_status gm_edges_load_text(const char* path, int32_t weighted, gm_edges_t* out);
/* io::load_matrix_market (io.cpp:112-182): coordinate real|pattern|integer,
 * general|symmetric (symmetric entries expanded, diagonal once). */
GM_API gm_status gm_edges_load_matrix_market(const char* path, gm_edges_t* out);
/* io::read_binary (io.cpp:317-362): "GMB1", n, m, then (src, dst, value) u64/u64/f64 LE. */
GM_API gm_status gm_edges_read_binary(const char* path, gm_edges_t* out);
/* Borrowed views into the buffer (valid until gm_edges_free). */
GM_API gm_status gm_edges_view(gm_edges_t e, uint64_t* num_vertices, uint64_t* num_edges,
                               const uint64_t** src, const uint64_t** dst, const double** values);
GM_API gm_status gm_edges_free(gm_edges_t e);
/* io::write_binary (io.cpp:290-315); values may be null (1.0). */
GM_API gm_status gm_edges_write_binary(const char* path, const uint64_t* src, const uint64_t* dst,
                                       const double* values, uint64_t num_edges,
                                       uint64_t num_vertices);
/* io::write_edge_list (io.cpp:364-373): 1-based "src dst %.17g" lines. */
GM_API gm_status gm_edges_write_text(const char* path, const uint64_t* src, const uint64_t* dst,
                                     const double* values, uint64_t num_edges);
/* bench::write_results / write_vector_results (report.cpp:53-75): one
 * "v<TAB>x[<TAB>x...]" line per vertex, 1-based, %.17g. rows: n*k row-major. */
GM_API gm_status gm_write_results(const char* path, const double* values, uint64_t n);
GM_API gm_status gm_write_vector_results(const char* path, const double* rows, uint64_t n,
                                         uint64_t k);
/* bench::RunReport (report.hpp:13-24) and write_report (report.cpp:77-102). */
typedef struct {
  const char* algorithm;
  const char* graph;
  uint32_t threads;
  uint64_t partitions;
  const double* iteration_seconds; /* IterationStats::total_seconds per superstep */
  uint64_t n_iterations;
  double total_seconds;
  uint64_t checksum;               /* FNV-1a 64 of the results file */
  const char* const* extra_keys;
  const char* const* extra_values;
  uint64_t n_extras;
} gm_run_report;
GM_API gm_status gm_write_report(const char* path, const gm_run_report* report);
/* bench::fnv1a64 / fnv1a64_file (report.cpp:27-51). */
GM_API uint64_t gm_fnv1a64(const void* data, uint64_t size);
GM_API gm_status gm_fnv1a64_file(const char* path, uint64_t* out);

/* ---- generic engine: any VertexProgram, exact reference semantics -------- */
/* Built-in instantiations of the device-side VertexProgram template (see
 * paper_1503_07241_b200/csrc/engine.cuh).  Fold order per row is ascending
 * internal source id, which equals the reference order (engine.hpp:59-66) on
 * graphs built without GM_RELABEL. */
typedef enum {
  GM_PROG_PAGERANK_REF = 1,    /* PageRankProgram, pagerank.hpp:36-63 (fp64)          */
  GM_PROG_BFS_REF = 2,         /* BfsProgram, traversal.hpp:39-63 (fp64)              */
  GM_PROG_SSSP_REF = 3,        /* SsspProgram, traversal.hpp:67-91 (fp64 weights).
                                  BFS_REF / SSSP_REF fold min lane-parallel, which is
                                  bit-identical to the reference's sequential fold for
                                  NaN-free distances and weights (algo::sssp rejects
                                  NaN / negative weights, traversal.hpp:125-133);
                                  with a NaN in props or weights the run is GM_EINPUT. */
  GM_PROG_SEMIRING_I64 = 4,    /* tests/acceptance.cpp:94-116                          */
  GM_PROG_ADD_PROBE = 5,       /* tests/test_engine.cpp:31-43                          */
  GM_PROG_IN_ADD_PROBE = 6,    /* tests/test_engine.cpp:206-223                        */
  GM_PROG_SELECTIVE_PROBE = 7, /* tests/test_engine.cpp:172-184 (vertex 0 declines)    */
  GM_PROG_THROWING_APPLY = 8,  /* tests/test_engine.cpp:67-80                          */
  GM_PROG_BOTH_ORDER_PROBE = 9,/* tests/test_engine.cpp:45-65                          */
  GM_PROG_FIXED_PROBE = 10,    /* tests/test_engine.cpp:133-143                        */
  GM_PROG_NORM_PAGERANK = 11   /* BASELINE PageRank as a generic fp64 program          */
} gm_program_id;

/* sizeof(vertex_t), sizeof(message_t), sizeof(reduced_t) of a program. */
GM_API gm_status gm_program_sizes(int32_t program, size_t* vertex_bytes, size_t* message_bytes,
                                  size_t* reduced_bytes);
/* Engine::run_graph_program (engine.hpp:193-213).  props (n * vertex_bytes) and
 * active (n bytes, 0/1) are the caller's VertexPropertyStore (core.hpp:179-222),
 * read on entry and written back on return.  params: program scalar (double*)
 * or NULL. */
GM_API gm_status gm_run_graph_program(gm_graph_t g, int32_t program, const double* params,
                                      void* props, uint8_t* active, int64_t max_iters,
                                      gm_iteration_stats* stats, int64_t cap, int64_t* n_stats);
/* Phase-level access: Engine::generate_messages (engine.hpp:76-98) and, when
 * run_spmv != 0, Engine::generalized_spmv (engine.hpp:104-134).  x (n *
 * message_bytes) / y (n * reduced_bytes) values are written where valid. */
GM_API gm_status gm_superstep_phases(gm_graph_t g, int32_t program, const double* params,
                                     const void* props, const uint8_t* active, void* x,
                                     uint8_t* x_valid, int32_t run_spmv, void* y,
                                     uint8_t* y_valid);

/* Zero-copy view of the device CSR in internal ids: which 0 = CSR(G^T) (rows =
 * destinations, the matrix the reference stores, dcsc.hpp:243-274), 1 = CSR(G)
 * (built on demand like ensure_forward, dcsc.hpp:201-215).  The pointers stay
 * valid until gm_graph_destroy and must not be written.  For validation
 * harnesses and callers that run their own kernels on the graph. */
GM_API gm_status gm_graph_csr(gm_graph_t g, int32_t which, const uint64_t** ptr_dev,
                              const uint32_t** idx_dev, uint64_t* rows, uint64_t* nnz);

/* ---- multi-GPU sharding (1-D row blocks of G^T, one process per GPU) ----- */
/* caller id -> internal id (n entries, host); identity without GM_RELABEL. */
GM_API gm_status gm_graph_permutation(gm_graph_t g, uint32_t* caller_to_internal);
/* PageRank over the rows [row_begin, row_end) of G^T this rank owns (internal
 * ids; with GM_SHARDS(P) rank r owns [r*N/P, (r+1)*N/P)).  x_block_dev receives
 * the block of the message vector; the caller all-gathers the blocks of every
 * rank into x_full_dev (n floats, internal order) and sums the dangling masses
 * into base = (1-d)/N + d*D/N for the next superstep. */
GM_API gm_status gm_pagerank_shard_init(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                        float* x_block_dev, double* dangling_block);
GM_API gm_status gm_pagerank_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                        const float* x_full_dev, double base, double damping,
                                        float* x_block_dev, double* dangling_block);
GM_API gm_status gm_pagerank_shard_ranks(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                         float* ranks_block_host);
/* Exchange only the part of each block that is ever gathered (SURVEY 8e,
 * mitigation 1: dangling vertices' messages are never read).  _active gives
 * this block's prefix length L (last non-dangling offset + 1; with GM_SHARDS
 * the dangling vertices form each block's tail); the ranks agree on
 * Lmax = max L, then _pack remaps the owned rows' columns to the packed
 * message layout (block b's entry o at b*Lmax + o).  After packing,
 * x_full_dev of gm_pagerank_shard_step holds P*Lmax floats and each rank
 * contributes x_block_dev[0, Lmax). */
GM_API gm_status gm_pagerank_shard_active(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                          uint64_t* prefix_len);
GM_API gm_status gm_pagerank_shard_pack(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                        uint64_t block_stride, uint64_t lmax);
/* The superstep with the all-gather fused into the SpMV epilogue: instead of
 * x_block_dev, every message of this block's gathered prefix (row - row_begin
 * < limit) is stored at [row + offset] of each of the npeers (1..8) device
 * buffers -- every rank's full message vector for the NEXT superstep, mapped
 * into this process with gm_ipc_open (the local one included), so the
 * transfer rides NVLink inside the kernel and no collective moves data.
 * offset: 0 for the unpacked layout, rank*Lmax - row_begin for the packed one.
 * The caller double-buffers the full vectors (read x_full_dev, write the
 * other one) and keeps one collective per superstep as the barrier (the
 * dangling-mass all-reduce).  _init_peers stores the initial messages the
 * same way (instead of gm_pagerank_shard_init's x_block_dev). */
GM_API gm_status gm_pagerank_shard_init_peers(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                              const uint64_t* peer_buffers, int32_t npeers,
                                              int64_t offset, uint64_t limit,
                                              double* dangling_block);
GM_API gm_status gm_pagerank_shard_step_peers(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                              const float* x_full_dev, double base, double damping,
                                              const uint64_t* peer_buffers, int32_t npeers,
                                              int64_t offset, uint64_t limit,
                                              double* dangling_block);
/* Device buffers shareable across processes (cudaMalloc + CUDA IPC): a
 * 64-byte handle per buffer, opened by the peers into their address space. */
GM_API gm_status gm_ipc_alloc(uint64_t bytes, void** dev_ptr);
GM_API gm_status gm_ipc_free(void* dev_ptr);
GM_API gm_status gm_ipc_handle(void* dev_ptr, void* handle64);
GM_API gm_status gm_ipc_open(const void* handle64, void** dev_ptr);
GM_API gm_status gm_ipc_close(void* dev_ptr);
/* BFS over the rows [row_begin, row_end) of a symmetric graph this rank owns
 * (32-vertex aligned; GM_SHARDS(P) blocks).  All bitmaps are device u32 words
 * in internal ids: frontier_dev / visited_dev cover all n vertices and are
 * identical on every rank; next_block_dev receives this block's
 * next-frontier bits (word 0 = row_begin).  The caller all-gathers the blocks
 * into the next frontier, ORs it into visited and sums found / found_edges
 * over the ranks (push/pull: pull once frontier edges > 5% of m, push again
 * once the frontier < n/24).  Levels stay on the device until _levels. */
GM_API gm_status gm_bfs_shard_init(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                   uint64_t root_internal);
GM_API gm_status gm_bfs_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                   const uint32_t* frontier_dev, const uint32_t* visited_dev,
                                   int32_t level, int32_t pull, uint32_t* next_block_dev,
                                   uint64_t* found, uint64_t* found_edges);
GM_API gm_status gm_bfs_shard_levels(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                     int32_t* levels_block_host);
/* The frontier exchange as peer stores instead of an all-gather: the block's
 * next-frontier words (next_block_dev, after _step) are stored at word
 * row_begin/32 of each of the npeers (1..8) bitmaps -- every rank's
 * frontier for the next superstep, mapped with gm_ipc_open, the local one
 * included.  Double-buffer the frontiers; the found-count all-reduce is the
 * barrier. */
GM_API gm_status gm_bfs_shard_push(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                   const uint32_t* next_block_dev, const uint64_t* peer_bitmaps,
                                   int32_t npeers);
/* Store `bytes` of a device block at byte `dst_offset` of each of the npeers
 * (1..8) peer buffers (CUDA IPC mappings: NVLink copies), on the graph's
 * stream -- the exchange of the SSSP message blocks and CF factor blocks
 * without an all-gather (double-buffer the targets; the count all-reduce is
 * the barrier). */
GM_API gm_status gm_push_block(gm_graph_t g, const void* src_dev, uint64_t bytes,
                               const uint64_t* peer_buffers, int32_t npeers, uint64_t dst_offset);
/* dst |= src over `words` device u32 words, on the graph's stream (visited |=
 * frontier when the frontier lives in IPC memory). */
GM_API gm_status gm_bitmap_or(gm_graph_t g, uint32_t* dst_dev, const uint32_t* src_dev,
                              uint64_t words);
/* SSSP (BSP Bellman-Ford, traversal.hpp:67-115) over the rows [row_begin,
 * row_end) this rank owns (32-vertex aligned), u8/u32 weights.  msg_dev: the
 * full uint32 message vector, identical on every rank -- the superstep-start
 * distance of each frontier vertex, UINT32_MAX elsewhere (init: 0 at the
 * root).  _step relaxes the frontier into the owned distances (pull: every
 * owned row takes min over in-neighbours u of msg[u] + w; push: the frontier's
 * out-edges into the block) and writes this block's next messages to
 * msg_block_dev (the new distance of each vertex that improved, else
 * UINT32_MAX) plus the improved count and their out-edges; the caller
 * all-gathers the blocks into the next msg and sums the counts (pull once the
 * frontier's out-edges exceed m/6; stop at 0 improved).  Replaces the
 * partitioned engine.hpp:224-260 loop for SsspProgram across GPUs. */
GM_API gm_status gm_sssp_shard_init(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                    uint64_t root_internal);
GM_API gm_status gm_sssp_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                    const uint32_t* msg_dev, int32_t pull, uint32_t* msg_block_dev,
                                    uint64_t* changed, uint64_t* changed_edges);
GM_API gm_status gm_sssp_shard_dists(gm_graph_t g, uint64_t row_begin, uint64_t row_end,
                                     uint32_t* dist_block_host);
/* Collaborative filtering (CfGdProgram, collaborative_filtering.hpp:51-90,
 * BOTH routes) over the vertices [row_begin, row_end) this rank owns.
 * factors_full_dev: the superstep-start factors of all n vertices (internal
 * order, n x k fp32, identical on every rank); the step writes the owned
 * vertices' next factors to factors_block_dev ((row_end - row_begin) x k),
 * the squared errors of the ratings stored in the owned rows of G (each
 * rating once across the ranks: sum them for the RMSE of the input factors)
 * and the number of owned vertices whose factors changed.  The same work
 * items and fold order as gm_cf: the caller's all-gather of the blocks
 * reproduces the single-GPU factors bit for bit. */
GM_API gm_status gm_cf_shard_step(gm_graph_t g, uint64_t row_begin, uint64_t row_end, int32_t k,
                                  const float* factors_full_dev, float gamma, float lambda,
                                  float* factors_block_dev, double* sq_err_sum, uint64_t* changed);
/* ---- multi-GPU behind the ABI: communicator + row-sharded graph -----------
 * The reference runs every row partition of G^T from one run_graph_program
 * call (engine.hpp:193-213; partitions by balanced_row_boundaries,
 * dcsc.hpp:77-105).  Here a partition ("shard") lives on a GPU and holds only
 * its rows; the superstep loop, the exchange and the termination test run
 * inside the library.
 *
 * A communicator spans P shards:
 *   gm_comm_create_local  one process drives every shard, devices[i] being the
 *                         GPU of shard i (repeats allowed: virtual shards on
 *                         one GPU); the exchange is peer memory over NVLink;
 *   gm_comm_create_nccl   one process per GPU (shard = rank), NCCL (libnccl
 *                         loaded at run time; GM_ENCCL on failure) plus CUDA
 *                         IPC mappings for the peer stores.  Rank 0 creates the
 *                         128-byte id with gm_comm_nccl_unique_id and the
 *                         caller distributes it (as NCCL applications do).
 * Every gm_dgraph_* call is collective: each process of the communicator
 * makes it, in the same order.  The communicator must outlive its graphs. */
typedef struct gm_comm* gm_comm_t;
typedef struct gm_dgraph* gm_dgraph_t;
GM_API gm_status gm_comm_create_local(int32_t nshards, const int32_t* devices, gm_comm_t* out);
GM_API gm_status gm_comm_nccl_unique_id(void* id128);
GM_API gm_status gm_comm_create_nccl(int32_t nranks, int32_t rank, int32_t device,
                                     const void* id128, gm_comm_t* out);
GM_API gm_status gm_comm_destroy(gm_comm_t c);

typedef struct {
  uint64_t num_vertices;       /* global                                          */
  uint64_t num_edges;          /* global stored entries of CSR(G^T)               */
  uint64_t row_begin, row_end; /* this shard's caller-id rows                      */
  uint64_t local_edges;        /* entries of this shard's CSR(G^T) rows           */
  uint64_t device_bytes;       /* graph bytes on this shard's GPU                  */
  uint64_t nonzero_out_degree; /* global (directed graphs)                         */
  int32_t shards, local_shards, first_shard, device;
} gm_dshard_info;

/* Sharded ingest (dcsc.hpp:110-164 + io::preprocess, io.cpp:184-222): every
 * shard generates 1/P of the seeded R-MAT stream (the same graph as
 * gm_graph_generate_rmat with permute = 1), the edges travel all-to-all to
 * the owner of their destination row, which deduplicates and builds CSR(G^T)
 * of its rows (entries ascending by caller id) -- plus CSR(G) of its rows
 * for directed graphs with GM_NEED_FORWARD or weights.  Boundaries balance
 * entries like balanced_row_boundaries (dcsc.hpp:81-105), 32-row aligned. */
GM_API gm_status gm_dgraph_generate_rmat(gm_comm_t c, uint32_t scale, uint32_t edge_factor,
                                         double a, double b, double cc, uint64_t seed,
                                         uint32_t flags, int32_t weights, gm_dgraph_t* out);
/* build_graph over a communicator: each process passes its share of the edge
 * list (any subset; a local communicator passes the whole list), the library
 * routes every edge to its owner.  Errors as gm_graph_create, agreed by all
 * ranks.  u32 ids, no values. */
GM_API gm_status gm_dgraph_create(gm_comm_t c, const gm_edge_list* edges, uint64_t num_vertices,
                                  uint32_t flags, int32_t value_storage, gm_dgraph_t* out);
GM_API gm_status gm_dgraph_destroy(gm_dgraph_t g);
GM_API gm_status gm_dgraph_shard_info(gm_dgraph_t g, int32_t local_shard, gm_dshard_info* info);
GM_API void* gm_dgraph_stream(gm_dgraph_t g, int32_t local_shard);
/* gm_pick_source on the sharded graph (same vertex for the same graph). */
GM_API gm_status gm_dgraph_pick_source(gm_dgraph_t g, uint64_t seed, uint64_t* out);
/* degree_vector (engine.hpp:295-312) of a local shard's rows: kind 0 = IN, 1 = OUT. */
GM_API gm_status gm_dgraph_degrees(gm_dgraph_t g, int32_t local_shard, int32_t kind, uint32_t* out);
/* Outputs of the sharded programs: the owned rows of this process's shards,
 * concatenated in shard order -- the whole caller-order vector for a local
 * communicator, rows [row_begin, row_end) for an NCCL rank.  Stats are
 * global (identical on every rank) with comm_seconds per superstep. */
/* algo::bfs (traversal.hpp:119-123) on a symmetric sharded graph. */
GM_API gm_status gm_dgraph_bfs(gm_dgraph_t g, uint64_t root, int64_t max_iters, int32_t* out_level,
                               int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                               int64_t* n_stats);
/* algo::sssp (traversal.hpp:125-133) on a directed sharded graph with u8
 * weights (gm_dgraph_generate_rmat weights = GM_VAL_U8): uint32 distances. */
GM_API gm_status gm_dgraph_sssp(gm_dgraph_t g, uint64_t source, int64_t max_iters,
                                uint32_t* out_dist, int32_t out_on_device,
                                gm_iteration_stats* stats, int64_t cap, int64_t* n_stats);
/* The Zipf bipartite rating graph of gm_graph_generate_bipartite, sharded:
 * each shard draws 1/P of the rating stream; users and items are owned by
 * row blocks like any vertex, each shard storing its vertices' raters
 * (CSR(G^T) rows) and rated items (CSR(G) rows) with u8 ratings. */
GM_API gm_status gm_dgraph_generate_bipartite(gm_comm_t c, uint32_t users, uint32_t items,
                                              double c_numerator, uint32_t cap, uint64_t seed,
                                              gm_dgraph_t* out);
/* collaborative_filtering_gd (collaborative_filtering.hpp:134-211) on the
 * sharded rating graph, K = 20 fp32: init_factors (n*k, host, caller ids) in;
 * out_factors receives the whole final matrix on every process (each shard
 * holds it after the last exchange); rmse_trace[it] after iteration it. */
GM_API gm_status gm_dgraph_cf(gm_dgraph_t g, const gm_cf_config* cfg, const float* init_factors,
                              float* out_factors, double* rmse_trace, gm_iteration_stats* stats,
                              int64_t cap, int64_t* n_stats);
/* gm_pagerank on a directed sharded graph; ranks bitwise independent of P. */
GM_API gm_status gm_dgraph_pagerank(gm_dgraph_t g, const gm_pagerank_config* cfg, float* out_rank,
                                    int32_t out_on_device, gm_iteration_stats* stats, int64_t cap,
                                    int64_t* n_stats);

/* Row-block boundaries balanced by stored entries, like
 * detail::balanced_row_boundaries (dcsc.hpp:81-105).  row_nnz: n counts;
 * bounds: parts+1 entries. */
GM_API gm_status gm_balanced_row_boundaries(const uint64_t* row_nnz, uint64_t n, uint64_t parts,
                                            uint64_t* bounds);

#ifdef __cplusplus
}
#endif
#endif /* GRAPHMAT_B200_H */
