/*
 * graphmat_oracle.h -- CPU restatement of the GraphMat/semigraph superstep path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1503_07241_b200/) links,
 * loads or calls this code.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker.
 *
 * Every algorithm here restates a reference function (paths relative to
 * /root/reference/proj):
 *   or_bfs / or_sssp*      include/semigraph/algorithms/traversal.hpp:39-115 driven by
 *                          Engine::run_graph_program (include/semigraph/engine.hpp:193-213)
 *   or_pagerank_ref        include/semigraph/algorithms/pagerank.hpp:36-110 and
 *                          tests/support/oracles.cpp:106-143 (activity gated, non-normalised)
 *   or_pagerank_norm       BASELINE configs[0] formula driven through the engine phases
 *                          (engine.hpp:76-172) with the CF driver's all-active pattern
 *                          (algorithms/collaborative_filtering.hpp:181-193)
 *   or_cf_gd               algorithms/collaborative_filtering.hpp:51-211
 *   or_semiring_spmv       tests/support/oracles.cpp:33-50 (dense_spmv) over stored entries
 *   or_preprocess          src/io.cpp:184-222 (self loops, stable dedup keep-first,
 *                          SYMMETRIZE, DAGIFY, BIPARTITE_CHECK)
 *   or_triangle_count      include/semigraph/algorithms/triangle_count.hpp:35-134 (gather the
 *                          ascending in-neighbour lists, intersect along every stored edge)
 * The generators (R-MAT with Philox counters + seeded bijection, Zipf bipartite) are the
 * seeded generators this repo defines for the BASELINE configs (the reference's mt19937
 * stream, src/io.cpp:224-288, is sequential and has no permutation); the CUDA ingest
 * implements the same definitions independently and tests compare them bit for bit.
 */
#ifndef GRAPHMAT_ORACLE_H
#define GRAPHMAT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors semigraph::IterationStats (include/semigraph/engine.hpp:32-39). */
typedef struct {
  int64_t iteration;
  int64_t active_before;
  int64_t messages_generated;
  int64_t vertices_updated;
  double spmv_seconds;
  double total_seconds;
} or_stats;

/* ---------------- generators ---------------- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t or_mix64(uint64_t x);
uint32_t or_permute(uint32_t x, unsigned scale, uint64_t seed);
/* Writes (edge_factor << scale) raw tuples. permute != 0 applies the seeded bijection. */
int64_t or_rmat_generate(unsigned scale, unsigned edge_factor, double a, double b, double c,
                         uint64_t seed, int permute, uint32_t* src, uint32_t* dst);
uint8_t or_edge_weight(uint64_t seed, uint32_t src, uint32_t dst);
void or_edge_weights(uint64_t seed, int64_t m, const uint32_t* src, const uint32_t* dst,
                     uint8_t* w);
/* Raw user->item draws; src == NULL only counts. Returns the raw tuple count. */
int64_t or_bipartite_generate(uint32_t users, uint32_t items, double c_numerator,
                              uint32_t cap, uint64_t seed, uint32_t* src, uint32_t* dst);
uint8_t or_rating(uint64_t seed, uint32_t user, uint32_t item);
void or_ratings(uint64_t seed, int64_t m, const uint32_t* src, const uint32_t* dst, uint8_t* r);
uint32_t or_pick_source(uint64_t seed, uint64_t n, const uint32_t* degree);

/* ---------------- preprocessing / CSR ---------------- */
/* In place. Removes self loops, stable-sorts by (src,dst), keeps the first of each
 * duplicate; symmetrize appends reverses and cleans again (src/io.cpp:184-206).
 * Arrays must have room for 2*m entries when symmetrize != 0. vals may be NULL. */
/* mode 0 NONE, 1 SYMMETRIZE, 2 DAGIFY (symmetrize, keep src < dst), 3 BIPARTITE_CHECK.
 * src/dst/vals need room for 2m entries for modes 1-2.  Returns the new count,
 * or -1 for BIPARTITE_CHECK failure with *bad = index (in the returned sorted
 * order) of the first edge whose source is also a destination or vice versa. */
int64_t or_preprocess(int64_t m, uint32_t* src, uint32_t* dst, double* vals, int mode);
int64_t or_preprocess_checked(int64_t m, uint32_t* src, uint32_t* dst, double* vals, int mode,
                              int64_t* bad);
/* Triangles of a DAG-form graph (every edge src < dst).  local[w] = sum over
 * stored v -> w of |N_in(v) & N_in(w)| (TriangleState::local_count).  Returns
 * the total, or -1 with *bad_src, *bad_dst = the first edge (by (src, dst))
 * violating src < dst. */
int64_t or_triangle_count(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                          uint64_t* local, uint32_t* bad_src, uint32_t* bad_dst);
/* Counting-sort CSR keyed by row[], entries keep input order (stable). */
void or_csr_build(uint64_t n, int64_t m, const uint32_t* row, const uint32_t* col,
                  const double* vals, uint64_t* ptr, uint32_t* idx, double* out_vals);

/* ---------------- programs ---------------- */
/* BSP BFS; level -1 = unreached. CSR(G) = out-neighbours. Returns #supersteps. */
int64_t or_bfs(uint64_t n, const uint64_t* optr, const uint32_t* oidx, uint32_t root,
               int64_t max_iters, int32_t* level, or_stats* st, int64_t cap);
/* BSP Bellman-Ford, integer weights (per CSR(G) entry); UINT32_MAX = unreached. */
int64_t or_sssp(uint64_t n, const uint64_t* optr, const uint32_t* oidx, const uint32_t* w,
                uint32_t root, int64_t max_iters, uint32_t* dist, or_stats* st, int64_t cap);
/* Same with double weights and +inf, bit-for-bit the reference SsspProgram. */
int64_t or_sssp_f64(uint64_t n, const uint64_t* optr, const uint32_t* oidx, const double* w,
                    uint32_t root, int64_t max_iters, double* dist, or_stats* st, int64_t cap);
/* Normalised PageRank (fp64): CSR(G^T) in-neighbours ascending. */
void or_pagerank_norm(uint64_t n, const uint64_t* iptr, const uint32_t* iidx,
                      const uint32_t* outdeg, double damping, int64_t iters, double* rank,
                      or_stats* st);
/* Reference PageRank (activity gated, r + (1-r)*sum, init 1.0). Returns #supersteps. */
int64_t or_pagerank_ref(uint64_t n, const uint64_t* iptr, const uint32_t* iidx,
                        const uint32_t* outdeg, double r, int64_t iters, double* rank,
                        or_stats* st);
/* CF gradient descent (fp64, reference fold orders). factors: n*k in/out.
 * CSR(G^T): rows = items, cols = users; CSR(G): rows = users, cols = items. */
void or_cf_gd(uint64_t n, const uint64_t* tptr, const uint32_t* tidx, const double* tval,
              const uint64_t* fptr, const uint32_t* fidx, const double* fval, int64_t k,
              double gamma, double lambda, int64_t iters, double* factors,
              double* objective_trace, double* rmse_trace, int64_t* updated);
/* Same update carried in fp32 (the GPU's arithmetic type), for tighter comparisons. */
void or_cf_gd_f32(uint64_t n, const uint64_t* tptr, const uint32_t* tidx, const double* tval,
                  const uint64_t* fptr, const uint32_t* fidx, const double* fval, int64_t k,
                  float gamma, float lambda, int64_t iters, float* factors,
                  double* rmse_trace, int64_t* updated);
/* updated (may be NULL): IterationStats::vertices_updated per iteration. */
/* y[k] = sum over stored (k,j) with xvalid[j] of A[k,j]*x[j]; yvalid iff any term. */
void or_semiring_spmv(uint64_t n, const uint64_t* iptr, const uint32_t* iidx,
                      const int64_t* vals, const int64_t* x, const uint8_t* xvalid, int64_t* y,
                      uint8_t* yvalid);

#ifdef __cplusplus
}
#endif
#endif
