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
//   x_cur[N]  f32  message vector (rank * inv_outdeg; 0 for dangling)   read by gather
//   in.ptr    u64  CSR(G^T) offsets                                      streamed
//   in.idx    u32  CSR(G^T) sources                                      streamed (128-bit)
//   inv[N]    f32  1/outdeg                                              streamed
//   rank[N]   f32  written in place (only the row owner touches it)
//   x_next[N] f32  written (the next superstep's message vector: the send
//                  phase is fused into this superstep's apply epilogue)
// Algorithmic bytes/superstep = 4·nnz + 8·(N+1) + 16·N.
//
// Kernels: rows with in-degree <= kLongRow go to k_pr_rows (8-lane groups, one
// row per group, shuffle tree reduce); longer rows get a CTA each
// (k_pr_long_rows).  Both reductions are fixed trees -> bitwise reproducible.
// The dangling mass for the NEXT superstep is reduced deterministically by
// k_dangling (fixed grid, per-block partials, single-block final), which also
// computes base on device, so 20 supersteps run without a host round trip.
#include <vector>

#include "api_internal.cuh"

namespace gm {

constexpr uint32_t kLongRow = 1024;
constexpr unsigned kDangBlocks = 296;

struct PrCache {
  uint64_t n = 0;
  DevBuf<float> inv, rank, x0, x1;
  DevBuf<uint32_t> long_rows;
  uint64_t n_long = 0;
  DevBuf<float> scalars;       // [0] = base for the current superstep
  DevBuf<float> dang_partial;  // kDangBlocks
  DevBuf<unsigned long long> ctr;
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

__global__ void k_long_rows(const uint64_t* ptr, uint64_t n, uint32_t thresh, uint32_t* list,
                            unsigned long long* cnt) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    if (ptr[v + 1] - ptr[v] > thresh) {
      const unsigned long long at = atomicAdd(cnt, 1ull);
      list[at] = uint32_t(v);
    }
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
  // Final fixed-order reduction by the last block to arrive.
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

template <bool kCount>
__global__ void __launch_bounds__(256) k_pr_rows(uint64_t n, const uint64_t* __restrict__ ptr,
                                                 const uint32_t* __restrict__ idx,
                                                 const float* __restrict__ x_cur,
                                                 const float* __restrict__ inv, float* rank,
                                                 float* __restrict__ x_next,
                                                 const float* __restrict__ scalars, float damping,
                                                 unsigned long long* ctr) {
  const unsigned lane8 = threadIdx.x & 7u;
  const unsigned gmask = 0xFFu << (threadIdx.x & 24u);
  const uint64_t group = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 3;
  const uint64_t ngroups = (uint64_t(gridDim.x) * blockDim.x) >> 3;
  const float base = scalars[0];
  unsigned long long changed = 0;
  for (uint64_t row = group; row < n; row += ngroups) {
    const uint64_t beg = ptr[row], end = ptr[row + 1];
    if (end - beg > kLongRow) continue;
    float s = 0.0f;
    for (uint64_t e = beg + lane8; e < end; e += 8) s += __ldg(&x_cur[__ldg(&idx[e])]);
    s += __shfl_xor_sync(gmask, s, 4, 8);
    s += __shfl_xor_sync(gmask, s, 2, 8);
    s += __shfl_xor_sync(gmask, s, 1, 8);
    if (lane8 == 0) {
      const float r = base + damping * s;
      if (kCount) changed += (end > beg) && (__float_as_uint(r) != __float_as_uint(rank[row]));
      rank[row] = r;
      x_next[row] = r * inv[row];
    }
  }
  if (kCount) warp_add_u64(ctr, changed);
}

template <bool kCount>
__global__ void __launch_bounds__(256) k_pr_long_rows(const uint32_t* rows, const uint64_t* ptr,
                                                      const uint32_t* __restrict__ idx,
                                                      const float* __restrict__ x_cur,
                                                      const float* inv, float* rank, float* x_next,
                                                      const float* scalars, float damping,
                                                      unsigned long long* ctr) {
  __shared__ float red[256];
  const uint32_t row = rows[blockIdx.x];
  const uint64_t beg = ptr[row], end = ptr[row + 1];
  float s = 0.0f;
  for (uint64_t e = beg + threadIdx.x; e < end; e += blockDim.x) s += __ldg(&x_cur[__ldg(&idx[e])]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float r = scalars[0] + damping * red[0];
    if (kCount && __float_as_uint(r) != __float_as_uint(rank[row])) atomicAdd(ctr, 1ull);
    rank[row] = r;
    x_next[row] = r * inv[row];
  }
}

PrCache& cache(Graph& g) {
  if (!g.pr) {
    g.pr = std::unique_ptr<PrCache, void (*)(PrCache*)>(new PrCache(), [](PrCache* p) { delete p; });
    PrCache& c = *g.pr;
    cudaStream_t s = g.stream;
    const uint64_t n = g.n;
    c.n = n;
    c.inv.alloc(n, s);
    c.rank.alloc(n, s);
    c.x0.alloc(n, s);
    c.x1.alloc(n, s);
    c.scalars.alloc(4, s);
    c.dang_partial.alloc(kDangBlocks + 1, s);
    c.ctr.alloc(4, s);
    c.ctr.zero(s);
    // long-row list
    DevBuf<unsigned long long> cnt(1, s);
    cnt.zero(s);
    c.long_rows.alloc(n ? n : 1, s);
    if (n)
      k_long_rows<<<grid_for(n, 256), 256, 0, s>>>(g.in.ptr.get(), n, kLongRow, c.long_rows.get(),
                                                   cnt.get());
    GM_LAUNCH_CHECK();
    unsigned long long h = 0;
    GM_CUDA(cudaMemcpyAsync(&h, cnt.get(), 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    c.n_long = h;
  }
  return *g.pr;
}

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
  const unsigned grid_rows = 148 * 8;
  const uint64_t dang_lo = g.relabeled ? g.nonzero_outdeg : 0;
  k_pr_init<<<grid_for(n, 256), 256, 0, s>>>(n, g.outdeg.get(), c.inv.get(), c.rank.get(), c.x0.get());
  GM_LAUNCH_CHECK();
  unsigned* ticket = reinterpret_cast<unsigned*>(c.ctr.get() + 3);
  GM_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  float* xc = c.x0.get();
  float* xn = c.x1.get();
  const float d = float(damping);
  cudaEvent_t e0, e1;
  GM_CUDA(cudaEventCreate(&e0));
  GM_CUDA(cudaEventCreate(&e1));
  for (int64_t it = 1; it <= iters; ++it) {
    if (collect) GM_CUDA(cudaEventRecord(e0, s));
    k_dangling<<<kDangBlocks, 256, 0, s>>>(dang_lo, n, c.rank.get(), c.inv.get(),
                                           c.dang_partial.get(), c.scalars.get(), damping, ticket);
    GM_LAUNCH_CHECK();
    if (collect) {
      GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
      k_pr_rows<true><<<grid_rows, 256, 0, s>>>(n, g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(),
                                                c.rank.get(), xn, c.scalars.get(), d, c.ctr.get());
    } else {
      k_pr_rows<false><<<grid_rows, 256, 0, s>>>(n, g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(),
                                                 c.rank.get(), xn, c.scalars.get(), d, c.ctr.get());
    }
    GM_LAUNCH_CHECK();
    if (c.n_long) {
      if (collect)
        k_pr_long_rows<true><<<unsigned(c.n_long), 256, 0, s>>>(
            c.long_rows.get(), g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(), c.rank.get(), xn,
            c.scalars.get(), d, c.ctr.get());
      else
        k_pr_long_rows<false><<<unsigned(c.n_long), 256, 0, s>>>(
            c.long_rows.get(), g.in.ptr.get(), g.in.idx.get(), xc, c.inv.get(), c.rank.get(), xn,
            c.scalars.get(), d, c.ctr.get());
      GM_LAUNCH_CHECK();
    }
    std::swap(xc, xn);
    if (!collect) continue;
    GM_CUDA(cudaEventRecord(e1, s));
    unsigned long long upd = 0;
    GM_CUDA(cudaMemcpyAsync(&upd, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    GM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
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
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
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

}  // namespace gm
