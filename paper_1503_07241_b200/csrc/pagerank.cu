// pagerank.cu -- normalised PageRank superstep: fused pull SpMV + apply + send.
//
// One superstep of the reference engine (include/semigraph/engine.hpp:176-189)
// for the BASELINE configs[0] program: every vertex active, a non-dangling u
// sends rank(u)/outdeg(u) (PageRankProgram shape, algorithms/pagerank.hpp:46-49),
// receivers fold Σ (engine.hpp:224-260), apply writes base + d·Σ with
// base = (1-d)/N + d·D/N (D = dangling mass), un-messaged vertices take the
// empty sum (collaborative_filtering.hpp:192-193 pattern).
//
// Device layout per superstep (internal ids, relabeled by out-degree so
// dangling vertices form the tail [nonzero_outdeg, n)):
//   x_cur[N]  f32  message vector (rank * inv_outdeg; 0 for dangling)   gathered
//   in.ptr    u64  CSR(G^T) offsets                                      streamed
//   in.idx    u32  CSR(G^T) sources                                      streamed
//   inv[N]    f32  1/outdeg                                              streamed
//   rank[N]   f32  written in place (only the row owner touches it)
//   x_next[N] f32  written: the next superstep's message vector (the send phase
//                  is fused into this superstep's apply epilogue)
// Algorithmic bytes/superstep = 4·nnz + 8·(N+1) + 16·N.
//
// SpMV = merge-path over row-aligned tiles (Merrill & Garland's CSR merge
// SpMV, specialised): the row sequence is cut once (cached per graph) into
// tiles of at most kTile path items (rows + nonzeros).  A 256-thread CTA
// stages the tile's row ends and the gathered x[col] values in shared memory
// (every gather of the tile in flight at once), each thread takes exactly
// kIPT path items found by a merge-path search in shared memory, and a block
// segmented scan hands partial row sums across threads.  Load balance is
// perfect whatever the degree mix (54% empty rows, hubs of 10^5 entries), and
// every reduction is a fixed tree, so results are bitwise reproducible.
// Rows longer than a tile get a CTA each (k_pr_long_rows).
// The dangling mass for the NEXT superstep is reduced deterministically by
// k_dangling (fixed grid, per-block partials, last-block final), which also
// computes base on device, so the supersteps run without a host round trip.
#include <vector>

#include "api_internal.cuh"

namespace gm {

constexpr int kPrThreads = 256;
constexpr int kIPT = 8;
constexpr int kTile = kPrThreads * kIPT;  // path items per tile
constexpr unsigned kDangBlocks = 296;

struct PrCache {
  uint64_t n = 0;
  uint64_t row_lo = 0, row_hi = 0;  // rows of G^T this process computes
  DevBuf<float> inv, rank, x0, x1;
  DevBuf<uint32_t> tile_b, tile_e, long_rows;
  uint64_t ntiles = 0, n_long = 0;
  DevBuf<float> scalars;       // [0] = base for the current superstep
  DevBuf<float> dang_partial;  // kDangBlocks
  DevBuf<unsigned long long> ctr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~PrCache() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

namespace {

__global__ void k_pr_init(uint64_t n, const uint32_t* outdeg, float* inv, float* rank, float* x) {
  const float r0 = 1.0f / float(n);
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t d = outdeg[v];
    const float iv = d ? 1.0f / float(d) : 0.0f;
    inv[v] = iv;
    rank[v] = r0;
    x[v] = r0 * iv;
  }
}

// D = Σ rank over dangling vertices (inv == 0) in [lo, n); base on device.
__global__ void k_dangling(uint64_t lo, uint64_t n, const float* rank, const float* inv,
                           float* partial, float* scalars, double damping, unsigned* ticket) {
  __shared__ float red[256];
  __shared__ bool last;
  float s = 0.0f;
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    if (inv[v] == 0.0f) s += rank[v];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = red[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  float t = 0.0f;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) t += ((volatile float*)partial)[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float nf = float(n);
    const float d = float(damping);
    scalars[0] = (1.0f - d) / nf + d * red[0] / nf;
    *ticket = 0;
  }
}

// Next superstep's base from the per-CTA dangling partials, summed in a fixed
// order (one CTA): base = (1-d)/N + d*D/N.
__global__ void __launch_bounds__(1024) k_pr_base(const float* partial, uint32_t np, uint64_t n,
                                                  double damping, float* scalars) {
  __shared__ float red[1024];
  float s = 0.0f;
  for (uint32_t i = threadIdx.x; i < np; i += 1024) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float nf = float(n), d = float(damping);
    scalars[0] = (1.0f - d) / nf + d * red[0] / nf;
  }
}

// Block-wide fixed-tree sum (all threads call; result valid in thread 0).
template <int kThreadsT>
__device__ __forceinline__ float block_sum(float v, float* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31u) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.0f;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kThreadsT / 32 ? scratch[threadIdx.x] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;
}

template <bool kCount>
__device__ __forceinline__ void pr_write(uint64_t row, float sum, float base, float damping,
                                         const float* __restrict__ inv, float* rank,
                                         float* __restrict__ x_next, bool nonempty,
                                         unsigned long long& changed, float& dangling) {
  const float r = base + damping * sum;
  if (kCount) changed += nonempty && (__float_as_uint(r) != __float_as_uint(rank[row]));
  rank[row] = r;
  const float iv = inv[row];
  x_next[row] = r * iv;
  if (iv == 0.0f) dangling += r;
}

template <bool kCount>
__global__ void __launch_bounds__(kPrThreads) k_pr_tiles(
    const uint32_t* __restrict__ tile_b, const uint32_t* __restrict__ tile_e,
    const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
    const float* __restrict__ x_cur, const float* __restrict__ inv, float* rank,
    float* __restrict__ x_next, const float* __restrict__ scalars, float damping,
    unsigned long long* ctr, float* __restrict__ dang_partial) {
  __shared__ uint32_t s_end[kTile + 1];
  __shared__ float s_red[kPrThreads / 32];
  float dangling = 0.0f;
  __shared__ float s_val[kTile];
  __shared__ uint32_t s_wk[kPrThreads / 32];
  __shared__ float s_wv[kPrThreads / 32];
  const unsigned tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  const uint32_t r0 = tile_b[blockIdx.x], r1 = tile_e[blockIdx.x];
  const uint64_t j0 = ptr[r0];
  const uint32_t nrows = r1 - r0;
  const uint32_t nnz = uint32_t(ptr[r1] - j0);
  const uint32_t items = nrows + nnz;
  const float base = scalars[0];
  // Stage row ends and gathered messages; all gathers of the tile in flight.
  for (uint32_t k = tid; k < nrows; k += kPrThreads) s_end[k] = uint32_t(ptr[r0 + k + 1] - j0);
  if (tid == 0) s_end[nrows] = 0xFFFFFFFFu;
#pragma unroll
  for (int u = 0; u < kIPT; ++u) {
    const uint32_t k = tid + u * kPrThreads;
    if (k < nnz) s_val[k] = __ldg(&x_cur[__ldg(&idx[j0 + k])]);
  }
  __syncthreads();
  // Merge-path search for this thread's diagonal.
  const uint32_t d0 = min(tid * kIPT, items), d1 = min(d0 + kIPT, items);
  uint32_t lo = d0 > nnz ? d0 - nnz : 0, hi = min(d0, nrows);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s_end[mid] <= d0 - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  uint32_t ti = lo, tj = d0 - lo;
  const uint32_t start_row = ti;
  float run = 0.0f, first_val = 0.0f;
  bool has_first = false;
  unsigned long long changed = 0;
  for (uint32_t k = d0; k < d1; ++k) {
    if (tj < s_end[ti]) {
      run += s_val[tj];
      ++tj;
    } else {
      if (!has_first) {
        has_first = true;
        first_val = run;
      } else {
        const uint32_t row_len = s_end[ti] - (ti ? s_end[ti - 1] : 0);
        pr_write<kCount>(r0 + ti, run, base, damping, inv, rank, x_next, row_len != 0, changed,
                         dangling);
      }
      run = 0.0f;
      ++ti;
    }
  }
  // Block segmented inclusive scan of the carries (key = open row, val = partial).
  uint32_t key = ti;
  float val = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t k2 = __shfl_up_sync(0xffffffffu, key, o);
    const float v2 = __shfl_up_sync(0xffffffffu, val, o);
    if (lane >= unsigned(o) && k2 == key) val += v2;
  }
  if (lane == 31) {
    s_wk[wid] = key;
    s_wv[wid] = val;
  }
  __syncthreads();
  if (wid == 0) {
    uint32_t wk = lane < kPrThreads / 32 ? s_wk[lane] : 0xFFFFFFFFu;
    float wv = lane < kPrThreads / 32 ? s_wv[lane] : 0.0f;
#pragma unroll
    for (int o = 1; o < kPrThreads / 32; o <<= 1) {
      const uint32_t k2 = __shfl_up_sync(0xffffffffu, wk, o);
      const float v2 = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= unsigned(o) && k2 == wk) wv += v2;
    }
    if (lane < kPrThreads / 32) {
      s_wk[lane] = wk;
      s_wv[lane] = wv;
    }
  }
  __syncthreads();
  if (wid > 0 && s_wk[wid - 1] == key) val += s_wv[wid - 1];
  // carry-in of this thread = inclusive carry of the previous thread
  uint32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
  float pv = __shfl_up_sync(0xffffffffu, val, 1);
  if (lane == 0) {
    pk = wid > 0 ? s_wk[wid - 1] : 0xFFFFFFFFu;
    pv = wid > 0 ? s_wv[wid - 1] : 0.0f;
  }
  if (has_first) {
    const float carry = (tid > 0 && pk == start_row) ? pv : 0.0f;
    const uint32_t row_len = s_end[start_row] - (start_row ? s_end[start_row - 1] : 0);
    pr_write<kCount>(r0 + start_row, carry + first_val, base, damping, inv, rank, x_next,
                     row_len != 0, changed, dangling);
  }
  if (kCount) warp_add_u64(ctr, changed);
  // Dangling mass of this tile's rows, for the next superstep's base.
  const float dsum = block_sum<kPrThreads>(dangling, s_red);
  if (tid == 0) dang_partial[blockIdx.x] = dsum;
}

template <bool kCount>
__global__ void __launch_bounds__(256) k_pr_long_rows(const uint32_t* rows, const uint64_t* ptr,
                                                      const uint32_t* __restrict__ idx,
                                                      const float* __restrict__ x_cur,
                                                      const float* inv, float* rank, float* x_next,
                                                      const float* scalars, float damping,
                                                      unsigned long long* ctr,
                                                      float* dang_partial) {
  __shared__ float red[256];
  const uint32_t row = rows[blockIdx.x];
  const uint64_t beg = ptr[row], end = ptr[row + 1];
  float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
  uint64_t e = beg + threadIdx.x;
  for (; e + 3 * 256 < end; e += 4 * 256) {
    a0 += __ldg(&x_cur[__ldg(&idx[e])]);
    a1 += __ldg(&x_cur[__ldg(&idx[e + 256])]);
    a2 += __ldg(&x_cur[__ldg(&idx[e + 512])]);
    a3 += __ldg(&x_cur[__ldg(&idx[e + 768])]);
  }
  for (; e < end; e += 256) a0 += __ldg(&x_cur[__ldg(&idx[e])]);
  red[threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float r = scalars[0] + damping * red[0];
    if (kCount && __float_as_uint(r) != __float_as_uint(rank[row])) atomicAdd(ctr, 1ull);
    rank[row] = r;
    const float iv = inv[row];
    x_next[row] = r * iv;
    dang_partial[blockIdx.x] = iv == 0.0f ? r : 0.0f;
  }
}

// Row-aligned tiles of <= kTile path items; rows needing more than a tile go
// to the long-row list.  One-time host pass over the offsets (cached).
void build_tiles(Graph& g, PrCache& c, cudaStream_t s, uint64_t lo, uint64_t n) {
  std::vector<uint64_t> ptr(g.n + 1);
  GM_CUDA(cudaMemcpyAsync(ptr.data(), g.in.ptr.get(), (g.n + 1) * 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  std::vector<uint32_t> tb, te, lr;
  uint64_t r = lo;
  while (r < n) {
    const uint64_t deg = ptr[r + 1] - ptr[r];
    if (deg + 1 > uint64_t(kTile)) {
      lr.push_back(uint32_t(r));
      ++r;
      continue;
    }
    const uint64_t start = r;
    uint64_t items = 0;
    while (r < n) {
      const uint64_t d = ptr[r + 1] - ptr[r];
      if (d + 1 > uint64_t(kTile) || items + d + 1 > uint64_t(kTile)) break;
      items += d + 1;
      ++r;
    }
    tb.push_back(uint32_t(start));
    te.push_back(uint32_t(r));
  }
  c.ntiles = tb.size();
  c.n_long = lr.size();
  c.tile_b.alloc(c.ntiles + 1, s);
  c.tile_e.alloc(c.ntiles + 1, s);
  c.long_rows.alloc(c.n_long + 1, s);
  if (c.ntiles) {
    GM_CUDA(cudaMemcpyAsync(c.tile_b.get(), tb.data(), c.ntiles * 4, cudaMemcpyHostToDevice, s));
    GM_CUDA(cudaMemcpyAsync(c.tile_e.get(), te.data(), c.ntiles * 4, cudaMemcpyHostToDevice, s));
  }
  if (c.n_long)
    GM_CUDA(cudaMemcpyAsync(c.long_rows.get(), lr.data(), c.n_long * 4, cudaMemcpyHostToDevice, s));
  GM_CUDA(cudaStreamSynchronize(s));
}

// Per-graph state for the rows [lo, hi) this process computes (all rows on
// one GPU; one row block of G^T per rank when sharded).
PrCache& cache(Graph& g, uint64_t lo, uint64_t hi) {
  if (!g.pr || g.pr->row_lo != lo || g.pr->row_hi != hi) {
    g.pr = std::unique_ptr<PrCache, void (*)(PrCache*)>(new PrCache(), [](PrCache* p) { delete p; });
    PrCache& c = *g.pr;
    cudaStream_t s = g.stream;
    const uint64_t n = g.n;
    c.n = n;
    c.row_lo = lo;
    c.row_hi = hi;
    c.inv.alloc(n, s);
    c.rank.alloc(n, s);
    c.x0.alloc(n, s);
    c.x1.alloc(n, s);
    c.scalars.alloc(4, s);
    c.ctr.alloc(4, s);
    c.ctr.zero(s);
    GM_CUDA(cudaEventCreate(&c.e0));
    GM_CUDA(cudaEventCreate(&c.e1));
    build_tiles(g, c, s, lo, hi);
    c.dang_partial.alloc(std::max<uint64_t>(kDangBlocks, c.ntiles + c.n_long) + 1, s);
    k_pr_init<<<grid_for(n, 256), 256, 0, s>>>(n, g.outdeg.get(), c.inv.get(), c.rank.get(),
                                               c.x0.get());
    GM_LAUNCH_CHECK();
    GM_CUDA(cudaStreamSynchronize(s));
  }
  return *g.pr;
}

PrCache& cache(Graph& g) { return cache(g, 0, g.n); }

}  // namespace

std::vector<gm_iteration_stats> pagerank(Graph& g, double damping, int64_t iters, float* out,
                                         bool out_on_device, bool collect) {
  if (!(damping >= 0.0 && damping <= 1.0)) fail(GM_EINPUT, "pagerank: damping must be in [0, 1]");
  if (iters < 0) fail(GM_EUSAGE, "pagerank: negative iteration count");
  std::vector<gm_iteration_stats> stats;
  const uint64_t n = g.n;
  if (n == 0) return stats;
  PrCache& c = cache(g);
  cudaStream_t s = g.stream;
  const uint64_t dang_lo = (g.relabeled && g.shards == 1) ? g.nonzero_outdeg : 0;
  k_pr_init<<<grid_for(n, 256), 256, 0, s>>>(n, g.outdeg.get(), c.inv.get(), c.rank.get(), c.x0.get());
  GM_LAUNCH_CHECK();
  unsigned* ticket = reinterpret_cast<unsigned*>(c.ctr.get() + 3);
  GM_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  float* xc = c.x0.get();
  float* xn = c.x1.get();
  const float d = float(damping);
  // Base of the first superstep (initial ranks); later bases come from the
  // dangling partials the SpMV kernels emit (k_pr_base).
  k_dangling<<<kDangBlocks, 256, 0, s>>>(dang_lo, n, c.rank.get(), c.inv.get(),
                                         c.dang_partial.get(), c.scalars.get(), damping, ticket);
  GM_LAUNCH_CHECK();
  float* part = c.dang_partial.get();
  for (int64_t it = 1; it <= iters; ++it) {
    if (collect) GM_CUDA(cudaEventRecord(c.e0, s));
    if (collect) GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
    if (c.ntiles) {
      if (collect)
        k_pr_tiles<true><<<unsigned(c.ntiles), kPrThreads, 0, s>>>(
            c.tile_b.get(), c.tile_e.get(), g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(),
            c.rank.get(), xn, c.scalars.get(), d, c.ctr.get(), part);
      else
        k_pr_tiles<false><<<unsigned(c.ntiles), kPrThreads, 0, s>>>(
            c.tile_b.get(), c.tile_e.get(), g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(),
            c.rank.get(), xn, c.scalars.get(), d, c.ctr.get(), part);
      GM_LAUNCH_CHECK();
    }
    if (c.n_long) {
      if (collect)
        k_pr_long_rows<true><<<unsigned(c.n_long), 256, 0, s>>>(
            c.long_rows.get(), g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(), c.rank.get(), xn,
            c.scalars.get(), d, c.ctr.get(), part + c.ntiles);
      else
        k_pr_long_rows<false><<<unsigned(c.n_long), 256, 0, s>>>(
            c.long_rows.get(), g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(), c.rank.get(), xn,
            c.scalars.get(), d, c.ctr.get(), part + c.ntiles);
      GM_LAUNCH_CHECK();
    }
    k_pr_base<<<1, 1024, 0, s>>>(part, uint32_t(c.ntiles + c.n_long), n, damping, c.scalars.get());
    GM_LAUNCH_CHECK();
    std::swap(xc, xn);
    if (!collect) continue;
    GM_CUDA(cudaEventRecord(c.e1, s));
    unsigned long long upd = 0;
    GM_CUDA(cudaMemcpyAsync(&upd, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    GM_CUDA(cudaEventElapsedTime(&ms, c.e0, c.e1));
    gm_iteration_stats st{};
    st.iteration = it;
    st.active_before = int64_t(n);
    st.messages_generated = int64_t(g.nonzero_outdeg);
    st.vertices_updated = int64_t(upd);
    st.spmv_seconds = ms * 1e-3;
    st.total_seconds = ms * 1e-3;
    st.edges_processed = int64_t(g.in.nnz);
    st.bytes_algorithmic = int64_t(4 * g.in.nnz + 8 * (n + 1) + 16 * n);
    st.direction = 0;
    stats.push_back(st);
  }
  if (out) {
    if (out_on_device) {
      to_external(g, c.rank.get(), out, 4);
    } else {
      DevBuf<float> ext(n, s);
      to_external(g, c.rank.get(), ext.get(), 4);
      GM_CUDA(cudaMemcpyAsync(out, ext.get(), n * 4, cudaMemcpyDeviceToHost, s));
    }
  }
  GM_CUDA(cudaStreamSynchronize(s));
  return stats;
}

// ---- 1-D row sharding: this process owns rows [lo, hi) of G^T --------------
// (the reference's row partitions, dcsc.hpp:77-105, one per GPU).  The caller
// all-gathers the message blocks of every rank into x_full between supersteps
// and all-reduces the dangling masses into the next base.

namespace {

__global__ void k_count_dangling(const float* inv, uint64_t lo, uint64_t hi,
                                 unsigned long long* cnt) {
  unsigned long long c = 0;
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x)
    c += inv[v] == 0.0f;
  warp_add_u64(cnt, c);
}

// Fixed-order sum of the per-tile dangling partials (one CTA) into a double.
__global__ void __launch_bounds__(1024) k_sum_partials(const float* partial, uint32_t np,
                                                       double* out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < np; i += 1024) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

void check_block(Graph& g, uint64_t lo, uint64_t hi) {
  if (lo > hi || hi > g.n) fail(GM_EUSAGE, "pagerank shard: bad row block");
}

}  // namespace

double pagerank_shard_init(Graph& g, uint64_t lo, uint64_t hi, float* x_block) {
  check_block(g, lo, hi);
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  k_pr_init<<<grid_for(g.n, 256), 256, 0, s>>>(g.n, g.outdeg.get(), c.inv.get(), c.rank.get(),
                                               c.x0.get());
  GM_LAUNCH_CHECK();
  if (hi > lo)
    GM_CUDA(cudaMemcpyAsync(x_block, c.x0.get() + lo, (hi - lo) * 4, cudaMemcpyDeviceToDevice, s));
  GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
  if (hi > lo) {
    k_count_dangling<<<grid_for(hi - lo, 256), 256, 0, s>>>(c.inv.get(), lo, hi, c.ctr.get());
    GM_LAUNCH_CHECK();
  }
  unsigned long long cnt = 0;
  GM_CUDA(cudaMemcpyAsync(&cnt, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return double(cnt) / double(g.n);
}

double pagerank_shard_step(Graph& g, uint64_t lo, uint64_t hi, const float* x_full, double base,
                           double damping, float* x_block) {
  check_block(g, lo, hi);
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  const float b = float(base);
  const float d = float(damping);
  GM_CUDA(cudaMemcpyAsync(c.scalars.get(), &b, 4, cudaMemcpyHostToDevice, s));
  float* part = c.dang_partial.get();
  float* xn = x_block - lo;  // the kernels write x_next[row] for rows in [lo, hi)
  if (c.ntiles) {
    k_pr_tiles<false><<<unsigned(c.ntiles), kPrThreads, 0, s>>>(
        c.tile_b.get(), c.tile_e.get(), g.in.ptr.get(), g.in.idx.get(), x_full, c.inv.get(),
        c.rank.get(), xn, c.scalars.get(), d, c.ctr.get(), part);
    GM_LAUNCH_CHECK();
  }
  if (c.n_long) {
    k_pr_long_rows<false><<<unsigned(c.n_long), 256, 0, s>>>(
        c.long_rows.get(), g.in.ptr.get(), g.in.idx.get(), x_full, c.inv.get(), c.rank.get(), xn,
        c.scalars.get(), d, c.ctr.get(), part + c.ntiles);
    GM_LAUNCH_CHECK();
  }
  double* dsum = reinterpret_cast<double*>(c.ctr.get() + 2);
  k_sum_partials<<<1, 1024, 0, s>>>(part, uint32_t(c.ntiles + c.n_long), dsum);
  GM_LAUNCH_CHECK();
  double h = 0.0;
  GM_CUDA(cudaMemcpyAsync(&h, dsum, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

void pagerank_shard_ranks(Graph& g, uint64_t lo, uint64_t hi, float* out_host) {
  check_block(g, lo, hi);
  PrCache& c = cache(g, lo, hi);
  if (hi > lo)
    GM_CUDA(cudaMemcpyAsync(out_host, c.rank.get() + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost,
                            g.stream));
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

}  // namespace gm
