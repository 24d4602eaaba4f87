// generic_programs.cu -- built-in VertexProgram instantiations of the generic engine.
//
// Each struct restates a reference program (or test probe) as a device
// functor; the generic engine (engine.cuh) runs it with the reference's exact
// superstep semantics.  Compiled with --fmad=false so fp64 folds round like the
// reference build (no FMA contraction).
#include <cub/device/device_scan.cuh>

#include "api_internal.cuh"
#include "engine.cuh"

namespace gm {

__global__ void k_row_lens(const uint32_t* rows, uint64_t nrows, const uint64_t* ptr,
                           uint32_t* lens) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nrows;
       i += uint64_t(gridDim.x) * blockDim.x)
    lens[i] = uint32_t(min(ptr[rows[i] + 1] - ptr[rows[i]], uint64_t(0xFFFFFFFFu)));
}

__global__ void k_long_rows(uint64_t n, const uint64_t* ptr, uint32_t* rows,
                            unsigned long long* cnt) {
  for (uint64_t v0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); v0 < n;
       v0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t v = v0 + lane_id();
    const bool is_long = v < n && ptr[v + 1] - ptr[v] > kLongRow;
    const unsigned m = __ballot_sync(0xffffffffu, is_long);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(cnt, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (is_long) rows[base + __popc(m & ((1u << lane_id()) - 1u))] = uint32_t(v);
  }
}

// The valid messages (set bits of xbits) as a queue, warp-aggregated, with
// the sum of their out-degrees: ctr[0] = count, ctr[1] = edges.
__global__ void k_msg_queue(uint64_t n, const uint32_t* xbits, const uint64_t* out_ptr,
                            uint32_t* q, unsigned long long* ctr) {
  // 32 consecutive words per warp step: their popcounts scanned across the
  // warp, one queue reservation per step (an atomic per word had serialised
  // a dense frontier's 262 K words on the counter: ~0.2 ms at scale 23), then
  // the nonzero words lane = vertex
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long edges = 0;
  for (uint64_t w0 = warp * 32; w0 < words; w0 += nwarps * 32) {
    const uint64_t wl = w0 + lane;
    const uint32_t mybits = wl < words ? xbits[wl] : 0u;
    const unsigned c = __popc(mybits);
    unsigned incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= unsigned(o)) incl += t;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) continue;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(&ctr[0], (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 31);
    const unsigned excl = incl - c;
    unsigned todo = __ballot_sync(0xffffffffu, mybits != 0u);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t bits = __shfl_sync(0xffffffffu, mybits, j);
      const unsigned off = __shfl_sync(0xffffffffu, excl, j);
      const uint64_t v = (w0 + uint64_t(j)) * 32 + lane;
      if ((bits >> lane) & 1u) {
        edges += out_ptr[v + 1] - out_ptr[v];
        q[base + off + __popc(bits & ((1u << lane) - 1u))] = uint32_t(v);
      }
    }
  }
  warp_add_u64(&ctr[1], edges);
}

__global__ void k_queue_degrees(const uint32_t* q, const unsigned long long* qn,
                                const uint64_t* out_ptr, uint64_t* deg) {
  const uint64_t nq = qn[0];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i <= nq;
       i += uint64_t(gridDim.x) * blockDim.x)
    deg[i] = i < nq ? out_ptr[q[i] + 1] - out_ptr[q[i]] : 0;
}

__global__ void k_piece_counts(const uint32_t* rows, uint64_t nrows, const uint64_t* ptr,
                               uint64_t* cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i <= nrows;
       i += uint64_t(gridDim.x) * blockDim.x)
    cnt[i] = i < nrows ? (ptr[rows[i] + 1] - ptr[rows[i]] + kPiece - 1) / kPiece : 0;
}

__global__ void k_piece_fill(const uint32_t* rows, uint64_t nrows, const uint64_t* ptr,
                             const uint64_t* off, uint32_t* prow, uint64_t* pbeg) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nrows;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t k = rows[i];
    uint64_t o = off[i];
    for (uint64_t b = ptr[k]; b < ptr[k + 1]; b += kPiece, ++o) {
      prow[o] = k;
      pbeg[o] = b;
    }
  }
}

void exclusive_scan_u64(uint64_t* data, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  size_t tmp = 0;
  GM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, data, data, int64_t(n), s));
  DevBuf<uint8_t> t(tmp, s);
  GM_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, data, data, int64_t(n), s));
}

__global__ void k_bytes_to_bits(const uint8_t* bytes, uint64_t n, uint32_t* bits) {
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint64_t v = w * 32 + lane_id();
    const unsigned b = __ballot_sync(0xffffffffu, v < n && bytes[v] != 0);
    if (lane_id() == 0) bits[w] = b;
  }
}

__global__ void k_bits_to_bytes(const uint32_t* bits, uint64_t n, uint8_t* bytes) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    bytes[v] = bit_test(bits, uint32_t(v)) ? 1 : 0;
}

namespace {

__device__ __forceinline__ bool bits_eq(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);  // core.hpp:63-65
}

// ---- PageRankProgram, algorithms/pagerank.hpp:24-63 ----------------------
struct PageRankState {
  double rank;
  uint64_t out_degree;
};
struct PageRankRef {
  using vertex_t = PageRankState;
  using edge_t = NoEdge;
  using message_t = double;
  using reduced_t = double;
  static constexpr gm_value_type kEdgeType = GM_VAL_NONE;
  double r = 0.15;
  __host__ __device__ Direction direction() const { return Direction::OUT; }
  __device__ bool send_message(const vertex_t& v, uint64_t, message_t* out) const {
    if (v.out_degree == 0) return false;
    *out = v.rank / static_cast<double>(v.out_degree);
    return true;
  }
  __device__ reduced_t process_message(const message_t& m, const edge_t&, const vertex_t&) const { return m; }
  __device__ reduced_t reduce(const reduced_t& a, const reduced_t& b) const { return a + b; }
  __device__ reduced_t reduce_identity() const { return 0.0; }
  __device__ vertex_t apply(const reduced_t& sum, const vertex_t& old) const {
    return {r + (1.0 - r) * sum, old.out_degree};
  }
  __device__ bool equal(const vertex_t& a, const vertex_t& b) const {
    return bits_eq(a.rank, b.rank) && a.out_degree == b.out_degree;
  }
  static const char* error_message(int) { return "pagerank failure"; }
};

// BASELINE normalised PageRank as a generic program (params: damping, base).
struct NormPageRank : PageRankRef {
  double damping = 0.85, base = 0.0;
  __device__ vertex_t apply(const reduced_t& sum, const vertex_t& old) const {
    return {base + damping * sum, old.out_degree};
  }
};

// ---- BfsProgram / SsspProgram, algorithms/traversal.hpp:39-91 ----------------
struct BfsRef {
  // min of doubles (no NaN, no -0 from the reference's non-negative
  // distances): any fold order gives the sequential result
  static constexpr bool kExactReorder = true;
  using vertex_t = double;  // DistanceState{distance}
  using edge_t = NoEdge;
  using message_t = double;
  using reduced_t = double;
  static constexpr gm_value_type kEdgeType = GM_VAL_NONE;
  __host__ __device__ Direction direction() const { return Direction::OUT; }
  __device__ bool send_message(const vertex_t& v, uint64_t, message_t* out) const {
    *out = v;
    return true;
  }
  __device__ reduced_t process_message(const message_t& m, const edge_t&, const vertex_t&) const { return m + 1.0; }
  __device__ reduced_t reduce(const reduced_t& a, const reduced_t& b) const { return a < b ? a : b; }
  __device__ reduced_t reduce_identity() const { return __longlong_as_double(0x7FF0000000000000ll); }
  __device__ vertex_t apply(const reduced_t& d, const vertex_t& old) const { return d < old ? d : old; }
  __device__ bool equal(const vertex_t& a, const vertex_t& b) const { return bits_eq(a, b); }
  static const char* error_message(int) { return "bfs failure"; }
};

struct SsspRef : BfsRef {
  using edge_t = double;
  static constexpr gm_value_type kEdgeType = GM_VAL_F64;
  __device__ reduced_t process_message(const message_t& m, const edge_t& w, const vertex_t&) const {
    return m + w;
  }
};

// ---- semiring probe, tests/acceptance.cpp:94-116 -----------------------------
struct SemiringCell {
  int64_t x, y;
  uint8_t has_x, has_y;
  uint8_t pad[6];
};
struct SemiringI64 {
  using vertex_t = SemiringCell;
  using edge_t = int64_t;
  using message_t = int64_t;
  using reduced_t = int64_t;
  static constexpr bool kExactReorder = true;  // integer sums (wrapping) are order-free
  static constexpr gm_value_type kEdgeType = GM_VAL_I64;
  __host__ __device__ Direction direction() const { return Direction::OUT; }
  __device__ bool send_message(const vertex_t& v, uint64_t, message_t* out) const {
    if (!v.has_x) return false;
    *out = v.x;
    return true;
  }
  __device__ reduced_t process_message(const message_t& m, const edge_t& e, const vertex_t&) const { return m * e; }
  __device__ reduced_t reduce(const reduced_t& a, const reduced_t& b) const { return a + b; }
  __device__ reduced_t reduce_identity() const { return 0; }
  __device__ vertex_t apply(const reduced_t& s, const vertex_t& o) const {
    vertex_t r = o;
    r.y = s;
    r.has_y = 1;
    return r;
  }
  __device__ bool equal(const vertex_t& a, const vertex_t& b) const {
    return a.x == b.x && a.y == b.y && a.has_x == b.has_x && a.has_y == b.has_y;
  }
  static const char* error_message(int) { return "semiring failure"; }
};

// ---- engine probes, tests/test_engine.cpp:31-80, 133-223 ---------------------
struct AddProbe {
  using vertex_t = double;
  using edge_t = NoEdge;
  using message_t = double;
  using reduced_t = double;
  static constexpr gm_value_type kEdgeType = GM_VAL_NONE;
  __host__ __device__ Direction direction() const { return Direction::OUT; }
  __device__ bool send_message(const vertex_t& v, uint64_t, message_t* out) const {
    *out = v;
    return true;
  }
  __device__ reduced_t process_message(const message_t& m, const edge_t&, const vertex_t&) const { return m; }
  __device__ reduced_t reduce(const reduced_t& a, const reduced_t& b) const { return a + b; }
  __device__ reduced_t reduce_identity() const { return 0.0; }
  __device__ vertex_t apply(const reduced_t& s, const vertex_t& old) const { return old + s; }
  __device__ bool equal(const vertex_t& a, const vertex_t& b) const { return a == b; }
  static const char* error_message(int) { return "probe failure"; }
};

struct InAddProbe : AddProbe {
  __host__ __device__ Direction direction() const { return Direction::IN; }
};

struct SelectiveProbe : AddProbe {
  __device__ bool send_message(const vertex_t& v, uint64_t id, message_t* out) const {
    if (id == 0) return false;
    *out = v;
    return true;
  }
};

struct FixedProbe : AddProbe {
  __device__ vertex_t apply(const reduced_t&, const vertex_t& old) const { return old; }
};

struct ThrowingApply : AddProbe {
  static constexpr bool kCanFail = true;
  __device__ bool send_message(const vertex_t& v, uint64_t, message_t* out, int&) const {
    *out = v;
    return true;
  }
  __device__ reduced_t process_message(const message_t& m, const edge_t&, const vertex_t&, int&) const { return m; }
  __device__ vertex_t apply(const reduced_t&, const vertex_t& old, int& err) const {
    err = 1;  // throw std::runtime_error("boom")
    return old;
  }
  static const char* error_message(int) { return "boom"; }
};

struct OrderList {  // reduced_t of BothOrderProbe: a short ordered list
  double v[4];
  int32_t n;
  int32_t pad;
};
struct BothOrderProbe {
  using vertex_t = double;
  using edge_t = double;
  using message_t = double;
  using reduced_t = OrderList;
  static constexpr gm_value_type kEdgeType = GM_VAL_F64;
  __host__ __device__ Direction direction() const { return Direction::BOTH; }
  __device__ bool send_message(const vertex_t& v, uint64_t, message_t* out) const {
    *out = v;
    return true;
  }
  __device__ reduced_t process_message(const message_t& m, const edge_t& e, const vertex_t&) const {
    reduced_t r{};
    r.v[0] = m * 100.0 + e;
    r.n = 1;
    return r;
  }
  __device__ reduced_t reduce(const reduced_t& a, const reduced_t& b) const {
    reduced_t out = a;
    for (int i = 0; i < b.n && out.n < 4; ++i) out.v[out.n++] = b.v[i];
    return out;
  }
  __device__ reduced_t reduce_identity() const { return reduced_t{}; }
  __device__ vertex_t apply(const reduced_t&, const vertex_t& old) const { return old; }
  __device__ bool equal(const vertex_t& a, const vertex_t& b) const { return a == b; }
  static const char* error_message(int) { return "probe failure"; }
};

template <typename P>
void sizes_of(size_t* v, size_t* m, size_t* r) {
  if (v) *v = sizeof(typename P::vertex_t);
  if (m) *m = sizeof(typename P::message_t);
  if (r) *r = sizeof(typename P::reduced_t);
}

template <typename F>
void dispatch(int prog, const double* params, F&& f) {
  switch (prog) {
    case GM_PROG_PAGERANK_REF: {
      PageRankRef p;
      if (params) p.r = params[0];
      if (!(p.r >= 0.0 && p.r <= 1.0)) fail(GM_EINPUT, "pagerank: r must be in [0, 1]");
      f(p);
      break;
    }
    case GM_PROG_NORM_PAGERANK: {
      NormPageRank p;
      if (params) {
        p.damping = params[0];
        p.base = params[1];
      }
      f(p);
      break;
    }
    case GM_PROG_BFS_REF: f(BfsRef{}); break;
    case GM_PROG_SSSP_REF: f(SsspRef{}); break;
    case GM_PROG_SEMIRING_I64: f(SemiringI64{}); break;
    case GM_PROG_ADD_PROBE: f(AddProbe{}); break;
    case GM_PROG_IN_ADD_PROBE: f(InAddProbe{}); break;
    case GM_PROG_SELECTIVE_PROBE: f(SelectiveProbe{}); break;
    case GM_PROG_THROWING_APPLY: f(ThrowingApply{}); break;
    case GM_PROG_BOTH_ORDER_PROBE: f(BothOrderProbe{}); break;
    case GM_PROG_FIXED_PROBE: f(FixedProbe{}); break;
    default: fail(GM_EUSAGE, "unknown program id " + std::to_string(prog));
  }
}

__global__ void k_count_nan_f64(const double* v, uint64_t n, unsigned long long* bad) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    c += v[i] != v[i];
  if (c) atomicAdd(bad, c);
}

// BfsRef / SsspRef fold min lane-parallel (kExactReorder); that equals the
// reference's sequential `a < b ? a : b` fold only without NaN (and without
// -0 ties).  algo::sssp rejects such inputs in its wrapper (traversal.hpp:
// 125-133); the raw programs get the same guard here.
void check_min_fold_inputs(Graph& g, int prog, const void* props) {
  if (prog != GM_PROG_BFS_REF && prog != GM_PROG_SSSP_REF) return;
  const double* p = static_cast<const double*>(props);
  for (uint64_t v = 0; v < g.n; ++v) {
    uint64_t b;
    std::memcpy(&b, &p[v], 8);
    if (p[v] != p[v] || b == 0x8000000000000000ull)
      fail(GM_EINPUT, "distance of vertex " + std::to_string(v + 1) +
                          " is NaN or -0; the min fold needs ordered distances");
  }
  if (prog == GM_PROG_SSSP_REF && g.value_type == GM_VAL_F64 && g.m) {
    DevBuf<unsigned long long> bad(1, g.stream);
    bad.zero(g.stream);
    k_count_nan_f64<<<grid_for(g.m, 256), 256, 0, g.stream>>>(
        reinterpret_cast<const double*>(g.in.val.get()), g.m, bad.get());
    GM_LAUNCH_CHECK();
    unsigned long long h = 0;
    GM_CUDA(cudaMemcpyAsync(&h, bad.get(), 8, cudaMemcpyDeviceToHost, g.stream));
    GM_CUDA(cudaStreamSynchronize(g.stream));
    if (h) fail(GM_EINPUT, "sssp: edge weights must be non-negative and not NaN");
  }
}

}  // namespace

void program_sizes(int prog, size_t* v, size_t* m, size_t* r) {
  dispatch(prog, nullptr, [&](auto p) { sizes_of<decltype(p)>(v, m, r); });
}

std::vector<gm_iteration_stats> run_program(Graph& g, int prog, const double* params, void* props,
                                            uint8_t* active, int64_t max_iters) {
  std::vector<gm_iteration_stats> st;
  dispatch(prog, params, [&](auto p) {
    using P = decltype(p);
    if (max_iters <= 0) return;  // zero budget is a no-op (engine.hpp:197)
    check_min_fold_inputs(g, prog, props);
    Engine<P> eng(g, p);
    eng.load(props, active);
    st = eng.run(max_iters);
    eng.store(props, active);
  });
  return st;
}

void superstep_phases(Graph& g, int prog, const double* params, const void* props,
                      const uint8_t* active, void* x, uint8_t* x_valid, int run_spmv, void* y,
                      uint8_t* y_valid) {
  dispatch(prog, params, [&](auto p) {
    using P = decltype(p);
    check_min_fold_inputs(g, prog, props);
    Engine<P> eng(g, p);
    eng.load(props, active);
    const uint64_t n = g.n;
    if (!n) return;
    DevBuf<unsigned long long> dummy;
    eng.send();
    eng.check_error();
    auto out_vals = [&](auto& buf, void* host) {
      using T = typename std::remove_reference_t<decltype(buf)>::value_type;
      DevBuf<T> e(n, eng.stream());
      to_external(g, buf.get(), e.get(), sizeof(T));
      GM_CUDA(cudaMemcpyAsync(host, e.get(), n * sizeof(T), cudaMemcpyDeviceToHost, eng.stream()));
      GM_CUDA(cudaStreamSynchronize(eng.stream()));
    };
    if (x) out_vals(eng.x(), x);
    if (x_valid) eng.bits_out(eng.xbits().get(), x_valid);
    if (run_spmv) {
      eng.spmv();
      eng.check_error();
      if (y) out_vals(eng.y(), y);
      if (y_valid) eng.bits_out(eng.ybits().get(), y_valid);
    }
  });
}

}  // namespace gm
