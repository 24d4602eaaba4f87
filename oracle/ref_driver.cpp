// ref_driver.cpp -- C entry points that run the UNMODIFIED reference engine.
//
// TEST INFRASTRUCTURE ONLY.  This file is ours; the engine it drives is the
// reference's header-only library, included from where it lies
// (/root/reference/proj/include/semigraph, never copied).  oracle/Makefile
// compiles it into oracle/_ref/libsemigraph_ref.so, which tests use to pin the
// C restatement (graphmat_oracle.c) and bench.py uses as the CPU baseline
// (cpu_baseline.kind = "reference", bench.py --impl reference).
//
// Everything below calls the reference's own public API:
//   build_graph               include/semigraph/dcsc.hpp:243-274
//   Engine phases / run loop  include/semigraph/engine.hpp:76-213
//   algo::bfs / algo::sssp    include/semigraph/algorithms/traversal.hpp:119-133
//   algo::pagerank            include/semigraph/algorithms/pagerank.hpp:73-110
//   collaborative_filtering_gd include/semigraph/algorithms/collaborative_filtering.hpp:134-211
//   algo::triangle_count      include/semigraph/algorithms/triangle_count.hpp:115-134
//   io::preprocess            src/io.cpp:184-222 (compiled from the reference tree with it)
//   io loaders / writers      src/io.cpp:85-373, bench:: report writers src/report.cpp
// The one new program is the BASELINE-normalised PageRank, which
// BASELINE configs[0] needs and the reference does not ship; it is driven
// through the reference engine phases exactly like the CF driver does.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "semigraph/algorithms/collaborative_filtering.hpp"
#include "semigraph/algorithms/pagerank.hpp"
#include "semigraph/algorithms/traversal.hpp"
#include "semigraph/algorithms/triangle_count.hpp"
#include "semigraph/engine.hpp"
#include "semigraph/io.hpp"
#include "semigraph/report.hpp"

using namespace semigraph;

extern "C" {
typedef struct {
  int64_t iteration, active_before, messages_generated, vertices_updated;
  double spmv_seconds, total_seconds;
} ref_stats;
}

namespace {

thread_local std::string g_err;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

unsigned resolve_threads(unsigned t) {
  if (t == 0) t = std::thread::hardware_concurrency();
  return t == 0 ? 1 : t;
}

std::vector<EdgeTriple<double>> triples(int64_t m, const uint32_t* src, const uint32_t* dst,
                                        const double* vals) {
  std::vector<EdgeTriple<double>> e(static_cast<std::size_t>(m));
  for (int64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i], vals ? vals[i] : 1.0};
  return e;
}

void copy_stats(const std::vector<IterationStats>& s, ref_stats* out, int64_t cap,
                int64_t* n_out) {
  if (n_out) *n_out = static_cast<int64_t>(s.size());
  if (!out) return;
  for (std::size_t i = 0; i < s.size() && static_cast<int64_t>(i) < cap; ++i) {
    out[i] = {static_cast<int64_t>(s[i].iteration), static_cast<int64_t>(s[i].active_before),
              static_cast<int64_t>(s[i].messages_generated),
              static_cast<int64_t>(s[i].vertices_updated), s[i].spmv_seconds,
              s[i].total_seconds};
  }
}

// Status codes mirror the reference CLI (tools/sgraph.cpp:24): 2 input, 3 engine.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InputError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// BASELINE configs[0] PageRank as a VertexProgram on the reference concept
// (core.hpp:239-253); shape follows PageRankProgram (pagerank.hpp:36-63).
struct NormalizedPageRank {
  using vertex_t = algo::PageRankState;
  using edge_t = double;
  using message_t = double;
  using reduced_t = double;
  double damping = 0.85;
  double base = 0.0;
  ScatterDirection direction() const { return ScatterDirection::OUT; }
  std::optional<message_t> send_message(const vertex_t& v, VertexId) const {
    if (v.out_degree == 0) return std::nullopt;
    return v.rank / static_cast<double>(v.out_degree);
  }
  reduced_t process_message(const message_t& m, const edge_t&, const vertex_t&) const {
    return m;
  }
  reduced_t reduce(const reduced_t& a, const reduced_t& b) const { return a + b; }
  reduced_t reduce_identity() const { return 0.0; }
  vertex_t apply(const reduced_t& sum, const vertex_t& old) const {
    return {base + damping * sum, old.out_degree};
  }
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_hardware_threads(void) { return static_cast<int>(resolve_threads(0)); }

int ref_bfs(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst, uint64_t root,
            int64_t max_iters, unsigned threads, double* out_dist, ref_stats* st, int64_t cap,
            int64_t* n_stats, double* algo_seconds) {
  return guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, nullptr);
    auto g = build_graph<algo::DistanceState>(e, n, std::size_t(threads) * 8);
    EngineConfig cfg;
    cfg.thread_count = threads;
    cfg.max_iterations = static_cast<std::size_t>(max_iters);
    Engine eng(cfg);
    std::vector<IterationStats> stats;
    const double t0 = now_s();
    auto d = algo::bfs(g, eng, root, &stats);
    if (algo_seconds) *algo_seconds = now_s() - t0;
    std::memcpy(out_dist, d.data(), sizeof(double) * n);
    copy_stats(stats, st, cap, n_stats);
  });
}

int ref_sssp(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst, const double* w,
             uint64_t root, int64_t max_iters, unsigned threads, double* out_dist,
             ref_stats* st, int64_t cap, int64_t* n_stats, double* algo_seconds) {
  return guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, w);
    auto g = build_graph<algo::DistanceState>(e, n, std::size_t(threads) * 8);
    EngineConfig cfg;
    cfg.thread_count = threads;
    cfg.max_iterations = static_cast<std::size_t>(max_iters);
    Engine eng(cfg);
    std::vector<IterationStats> stats;
    const double t0 = now_s();
    auto d = algo::sssp(g, eng, root, &stats);
    if (algo_seconds) *algo_seconds = now_s() - t0;
    std::memcpy(out_dist, d.data(), sizeof(double) * n);
    copy_stats(stats, st, cap, n_stats);
  });
}

int ref_pagerank(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst, double r,
                 int64_t iters, unsigned threads, double* out_rank, ref_stats* st,
                 int64_t cap, int64_t* n_stats, double* algo_seconds) {
  return guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, nullptr);
    auto g = build_graph<algo::PageRankState>(e, n, std::size_t(threads) * 8);
    EngineConfig cfg;
    cfg.thread_count = threads;
    Engine eng(cfg);
    algo::PageRankConfig pc;
    pc.r = r;
    pc.max_iterations = static_cast<std::size_t>(iters);
    std::vector<IterationStats> stats;
    const double t0 = now_s();
    auto rk = algo::pagerank(g, eng, pc, &stats);
    if (algo_seconds) *algo_seconds = now_s() - t0;
    std::memcpy(out_rank, rk.data(), sizeof(double) * n);
    copy_stats(stats, st, cap, n_stats);
  });
}

int ref_pagerank_norm(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                      double damping, int64_t iters, unsigned threads, double* out_rank,
                      ref_stats* st, int64_t cap, int64_t* n_stats, double* algo_seconds) {
  return guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, nullptr);
    auto g = build_graph<algo::PageRankState>(e, n, std::size_t(threads) * 8);
    EngineConfig cfg;
    cfg.thread_count = threads;
    Engine eng(cfg);
    const auto deg = degree_vector(eng, g, DegreeKind::OUT);
    auto& props = g.properties();
    const double nd = static_cast<double>(n);
    for (VertexId v = 0; v < n; ++v) props[v] = {1.0 / nd, deg[v]};
    std::vector<IterationStats> stats;
    const double t0 = now_s();
    for (int64_t it = 1; it <= iters; ++it) {
      IterationStats s;
      const double ts = now_s();
      double dangling = 0.0;
      for (VertexId v = 0; v < n; ++v)
        if (props[v].out_degree == 0) dangling += props[v].rank;
      NormalizedPageRank prog;
      prog.damping = damping;
      prog.base = (1.0 - damping) / nd + damping * dangling / nd;
      props.set_all_active(true);
      s.active_before = n;
      auto x = eng.generate_messages(g, prog);
      s.messages_generated = x.count_valid();
      const double t1 = now_s();
      auto y = eng.generalized_spmv(g, x, prog);
      s.spmv_seconds = now_s() - t1;
      s.vertices_updated = eng.apply_and_activate(g, y, prog);
      for (VertexId v = 0; v < n; ++v)
        if (!y.valid(v)) props[v] = prog.apply(0.0, props[v]);
      s.total_seconds = now_s() - ts;
      s.iteration = static_cast<std::size_t>(it);
      stats.push_back(s);
    }
    if (algo_seconds) *algo_seconds = now_s() - t0;
    for (VertexId v = 0; v < n; ++v) out_rank[v] = props[v].rank;
    copy_stats(stats, st, cap, n_stats);
  });
}

// factors: n*k doubles (in: injected start, out: final). Sides follow the
// reference inference (users = rating sources). per_iteration != 0 runs the
// driver one iteration at a time (state carries over in the graph) so the
// RMSE after every iteration can be read; algo time then covers those calls.
int ref_cf(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
           const double* ratings, int64_t k, double gamma, double lambda, int64_t iters,
           unsigned threads, int per_iteration, double* factors, double* objective_trace,
           double* rmse_trace, double* algo_seconds, int64_t* updated) {
  return guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, ratings);
    auto g = build_graph<algo::LatentVector>(e, n, std::size_t(threads) * 8);
    EngineConfig cfg;
    cfg.thread_count = threads;
    Engine eng(cfg);
    auto& props = g.properties();
    for (VertexId v = 0; v < n; ++v)
      props[v].p.assign(factors + v * k, factors + (v + 1) * k);
    algo::CfConfig cc;
    cc.k = static_cast<std::size_t>(k);
    cc.gamma = gamma;
    cc.lambda = lambda;
    auto rmse_now = [&]() {
      double sq = 0.0;
      for (const auto& t : e) {
        double dot = 0.0;
        for (int64_t d = 0; d < k; ++d) dot += props[t.src].p[d] * props[t.dst].p[d];
        const double err = t.value - dot;
        sq += err * err;
      }
      return m ? std::sqrt(sq / static_cast<double>(m)) : 0.0;
    };
    double algo = 0.0;
    if (per_iteration) {
      cc.iterations = 1;
      for (int64_t it = 0; it < iters; ++it) {
        const double t0 = now_s();
        std::vector<IterationStats> st;
        auto res = algo::collaborative_filtering_gd(g, eng, cc, &st);
        algo += now_s() - t0;
        if (updated) updated[it] = static_cast<int64_t>(st.back().vertices_updated);
        if (objective_trace) objective_trace[it] = res.objective_trace.back();
        if (rmse_trace) rmse_trace[it] = rmse_now();
      }
    } else {
      cc.iterations = static_cast<std::size_t>(iters);
      const double t0 = now_s();
      std::vector<IterationStats> st;
      auto res = algo::collaborative_filtering_gd(g, eng, cc, &st);
      algo = now_s() - t0;
      if (updated)
        for (std::size_t i = 0; i < st.size(); ++i)
          updated[i] = static_cast<int64_t>(st[i].vertices_updated);
      if (objective_trace)
        for (std::size_t i = 0; i < res.objective_trace.size(); ++i)
          objective_trace[i] = res.objective_trace[i];
    }
    if (algo_seconds) *algo_seconds = algo;
    for (VertexId v = 0; v < n; ++v)
      std::memcpy(factors + v * k, props[v].p.data(), sizeof(double) * k);
  });
}

// ---- build once, run many (the bench's reference arm: graph build is not
// part of the timed algorithm, tools/sgraph.cpp:101-103) ----------------------
struct RefDistGraph {
  Graph<algo::DistanceState, double> g;
  unsigned threads;
};
struct RefPrGraph {
  Graph<algo::PageRankState, double> g;
  unsigned threads;
};

void* ref_dist_graph_new(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                         const double* w, unsigned threads) {
  RefDistGraph* h = nullptr;
  const int rc = guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, w);
    h = new RefDistGraph{build_graph<algo::DistanceState>(e, n, std::size_t(threads) * 8), threads};
  });
  return rc == 0 ? h : nullptr;
}

void ref_dist_graph_free(void* h) { delete static_cast<RefDistGraph*>(h); }

// kind 0 = BFS, 1 = SSSP on a prebuilt graph.
int ref_dist_run(void* hv, int kind, uint64_t root, int64_t max_iters, double* out_dist,
                 ref_stats* st, int64_t cap, int64_t* n_stats, double* algo_seconds) {
  return guarded([&] {
    auto* h = static_cast<RefDistGraph*>(hv);
    EngineConfig cfg;
    cfg.thread_count = h->threads;
    cfg.max_iterations = static_cast<std::size_t>(max_iters);
    Engine eng(cfg);
    std::vector<IterationStats> stats;
    const double t0 = now_s();
    auto d = kind == 0 ? algo::bfs(h->g, eng, root, &stats) : algo::sssp(h->g, eng, root, &stats);
    if (algo_seconds) *algo_seconds = now_s() - t0;
    if (out_dist) std::memcpy(out_dist, d.data(), sizeof(double) * d.size());
    copy_stats(stats, st, cap, n_stats);
  });
}

void* ref_pr_graph_new(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                       unsigned threads) {
  RefPrGraph* h = nullptr;
  const int rc = guarded([&] {
    threads = resolve_threads(threads);
    auto e = triples(m, src, dst, nullptr);
    h = new RefPrGraph{build_graph<algo::PageRankState>(e, n, std::size_t(threads) * 8), threads};
  });
  return rc == 0 ? h : nullptr;
}

void ref_pr_graph_free(void* h) { delete static_cast<RefPrGraph*>(h); }

// BASELINE-normalised PageRank on a prebuilt graph (same driver as ref_pagerank_norm).
int ref_pr_norm_run(void* hv, double damping, int64_t iters, double* out_rank,
                    double* algo_seconds) {
  return guarded([&] {
    auto* h = static_cast<RefPrGraph*>(hv);
    auto& g = h->g;
    const uint64_t n = g.num_vertices();
    EngineConfig cfg;
    cfg.thread_count = h->threads;
    Engine eng(cfg);
    const auto deg = degree_vector(eng, g, DegreeKind::OUT);
    auto& props = g.properties();
    const double nd = static_cast<double>(n);
    for (VertexId v = 0; v < n; ++v) props[v] = {1.0 / nd, deg[v]};
    const double t0 = now_s();
    for (int64_t it = 1; it <= iters; ++it) {
      double dangling = 0.0;
      for (VertexId v = 0; v < n; ++v)
        if (props[v].out_degree == 0) dangling += props[v].rank;
      NormalizedPageRank prog;
      prog.damping = damping;
      prog.base = (1.0 - damping) / nd + damping * dangling / nd;
      props.set_all_active(true);
      auto x = eng.generate_messages(g, prog);
      auto y = eng.generalized_spmv(g, x, prog);
      eng.apply_and_activate(g, y, prog);
      for (VertexId v = 0; v < n; ++v)
        if (!y.valid(v)) props[v] = prog.apply(0.0, props[v]);
    }
    if (algo_seconds) *algo_seconds = now_s() - t0;
    if (out_rank)
      for (VertexId v = 0; v < n; ++v) out_rank[v] = props[v].rank;
  });
}

// Semiring (+, x) over int64 like tests/acceptance.cpp:97-116: x valid where
// xvalid[j]; y written where valid.
int ref_semiring_spmv(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                      const int64_t* vals, const int64_t* x, const uint8_t* xvalid,
                      unsigned threads, unsigned parts, int64_t* y, uint8_t* yvalid) {
  return guarded([&] {
    struct Cell {
      long long x = 0, y = 0;
      bool has_x = false, has_y = false;
      bool operator==(const Cell& o) const {
        return x == o.x && y == o.y && has_x == o.has_x && has_y == o.has_y;
      }
    };
    struct Prog {
      using vertex_t = Cell;
      using edge_t = long long;
      using message_t = long long;
      using reduced_t = long long;
      ScatterDirection direction() const { return ScatterDirection::OUT; }
      std::optional<message_t> send_message(const vertex_t& v, VertexId) const {
        if (!v.has_x) return std::nullopt;
        return v.x;
      }
      reduced_t process_message(const message_t& mm, const edge_t& ee, const vertex_t&) const {
        return mm * ee;
      }
      reduced_t reduce(const reduced_t& a, const reduced_t& b) const { return a + b; }
      reduced_t reduce_identity() const { return 0; }
      vertex_t apply(const reduced_t& s, const vertex_t& o) const { return {o.x, s, o.has_x, true}; }
    };
    threads = resolve_threads(threads);
    std::vector<EdgeTriple<long long>> e(static_cast<std::size_t>(m));
    for (int64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i], vals[i]};
    auto g = build_graph<Cell, long long>(e, n, parts ? parts : 1);
    EngineConfig cfg;
    cfg.thread_count = threads;
    Engine eng(cfg);
    auto& props = g.properties();
    for (VertexId j = 0; j < n; ++j) {
      if (!xvalid[j]) continue;
      props[j].x = x[j];
      props[j].has_x = true;
      props.set_active(j, true);
    }
    Prog prog;
    auto xs = eng.generate_messages(g, prog);
    auto ys = eng.generalized_spmv(g, xs, prog);
    for (VertexId k2 = 0; k2 < n; ++k2) {
      yvalid[k2] = ys.valid(k2) ? 1 : 0;
      y[k2] = ys.valid(k2) ? ys.value(k2) : 0;
    }
  });
}

// io::preprocess(mode 0..3); returns the new count (arrays need 2m room) or -1
// (InputError, message in ref_last_error).
int64_t ref_preprocess(int64_t m, uint32_t* src, uint32_t* dst, double* vals, int mode) {
  int64_t out = -1;
  const int rc = guarded([&] {
    auto e = triples(m, src, dst, vals);
    const io::PreprocessMode md = mode == 1   ? io::PreprocessMode::SYMMETRIZE
                                  : mode == 2 ? io::PreprocessMode::DAGIFY
                                  : mode == 3 ? io::PreprocessMode::BIPARTITE_CHECK
                                              : io::PreprocessMode::NONE;
    auto r = io::preprocess(std::move(e), md);
    for (std::size_t i = 0; i < r.size(); ++i) {
      src[i] = static_cast<uint32_t>(r[i].src);
      dst[i] = static_cast<uint32_t>(r[i].dst);
      if (vals) vals[i] = r[i].value;
    }
    out = static_cast<int64_t>(r.size());
  });
  return rc == 0 ? out : -1;
}

// algo::triangle_count on a DAG-form edge list; local = TriangleState::local_count.
int ref_triangle_count(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                       unsigned threads, unsigned parts, uint64_t* total, uint64_t* local,
                       double* algo_seconds) {
  return guarded([&] {
    auto e = triples(m, src, dst, nullptr);
    auto g = build_graph<algo::TriangleState, double>(e, n, parts ? parts : 1);
    EngineConfig cfg;
    cfg.thread_count = resolve_threads(threads);
    cfg.max_iterations = 4;
    Engine eng(cfg);
    const double t0 = now_s();
    *total = algo::triangle_count(g, eng);
    if (algo_seconds) *algo_seconds = now_s() - t0;
    if (local) {
      auto& props = g.properties();
      for (VertexId v = 0; v < n; ++v) local[v] = props[v].local_count;
    }
  });
}

// ---- files: run the reference's loader (kind 0 text, 1 text weighted,
// 2 Matrix Market, 3 GMB1) and re-emit what it parsed as GMB1 with the
// reference's own writer, so tests compare parsed edge lists exactly.
int ref_io_load_to_binary(int kind, const char* path, const char* out_gmb1) {
  return guarded([&] {
    io::EdgeList e = kind == 0   ? io::load_edge_list(path, false)
                     : kind == 1 ? io::load_edge_list(path, true)
                     : kind == 2 ? io::load_matrix_market(path)
                                 : io::read_binary(path);
    io::write_binary(out_gmb1, e.edges, e.num_vertices);
  });
}

// io::write_edge_list of a GMB1 file's edges.
int ref_io_write_edge_list(const char* in_gmb1, const char* out_path) {
  return guarded([&] { io::write_edge_list(out_path, io::read_binary(in_gmb1).edges); });
}

int ref_io_write_results(const char* path, const double* values, uint64_t n) {
  return guarded([&] { bench::write_results(path, std::vector<double>(values, values + n)); });
}

int ref_io_write_vector_results(const char* path, const double* rows, uint64_t n, uint64_t k) {
  return guarded([&] {
    std::vector<std::vector<double>> r(n);
    for (uint64_t v = 0; v < n; ++v) r[v].assign(rows + v * k, rows + (v + 1) * k);
    bench::write_vector_results(path, r);
  });
}

int ref_io_write_report(const char* path, const char* algorithm, const char* graph,
                        unsigned threads, uint64_t partitions, const double* iter_seconds,
                        uint64_t n_iter, double total_seconds, uint64_t checksum,
                        const char* const* keys, const char* const* values, uint64_t n_extras) {
  return guarded([&] {
    bench::RunReport r;
    r.algorithm = algorithm;
    r.graph = graph;
    r.threads = threads;
    r.partitions = partitions;
    r.iterations.resize(n_iter);
    for (uint64_t i = 0; i < n_iter; ++i) r.iterations[i].total_seconds = iter_seconds[i];
    r.total_seconds = total_seconds;
    r.checksum = checksum;
    for (uint64_t i = 0; i < n_extras; ++i) r.extras.emplace_back(keys[i], values[i]);
    bench::write_report(path, r);
  });
}

int ref_io_fnv1a64_file(const char* path, uint64_t* out) {
  return guarded([&] { *out = bench::fnv1a64_file(path); });
}

// The reference CLI's "run" composition (tools/sgraph.cpp:104-183) over the
// reference library API -- the CLI binary itself needs the absent CLI11.  Writes
// the results file and returns its FNV-1a checksum (report.checksum).
int ref_run_one(const char* algorithm, const char* graph_path, const char* format, int weighted,
                uint64_t source, int64_t max_iters, double damping, unsigned threads,
                const char* out_path, uint64_t* checksum, double* total_out) {
  return guarded([&] {
    const std::string algo_name = algorithm, fmt = format;
    io::EdgeList input = fmt == "mtx"   ? io::load_matrix_market(graph_path)
                         : fmt == "bin" ? io::read_binary(graph_path)
                                        : io::load_edge_list(graph_path, weighted != 0);
    const io::PreprocessMode mode = algo_name == "bfs"  ? io::PreprocessMode::SYMMETRIZE
                                    : algo_name == "tc" ? io::PreprocessMode::DAGIFY
                                                        : io::PreprocessMode::NONE;
    auto edges = io::preprocess(std::move(input.edges), mode);
    const std::size_t n = input.num_vertices;
    threads = resolve_threads(threads);
    const std::size_t parts = std::size_t(threads) * 8;
    EngineConfig ec;
    ec.thread_count = threads;
    if (algo_name == "pagerank") {
      auto g = build_graph<algo::PageRankState, double>(edges, n, parts);
      Engine eng(ec);
      algo::PageRankConfig pc;
      pc.r = damping;
      pc.max_iterations = max_iters < 0 ? 100 : std::size_t(max_iters);
      bench::write_results(out_path, algo::pagerank(g, eng, pc));
    } else if (algo_name == "bfs" || algo_name == "sssp") {
      auto g = build_graph<algo::DistanceState, double>(edges, n, parts);
      const std::size_t budget = max_iters < 0 ? std::max<std::size_t>(n, 1) : std::size_t(max_iters);
      ec.max_iterations = budget == 0 ? 1 : budget;
      Engine eng(ec);
      const VertexId root = source - 1;
      bench::write_results(out_path, algo_name == "bfs" ? algo::bfs(g, eng, root)
                                                        : algo::sssp(g, eng, root));
    } else if (algo_name == "tc") {
      auto g = build_graph<algo::TriangleState, double>(edges, n, parts);
      Engine eng(ec);
      const std::uint64_t total = algo::triangle_count(g, eng);
      std::vector<double> per(n);
      for (VertexId v = 0; v < n; ++v) per[v] = static_cast<double>(g.properties()[v].local_count);
      bench::write_results(out_path, per);
      if (total_out) *total_out = static_cast<double>(total);
    } else {
      throw InputError("ref_run_one: unsupported algorithm " + algo_name);
    }
    *checksum = bench::fnv1a64_file(out_path);
  });
}

}  // extern "C"
