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
//   x_cur[N]   f32  message vector (rank * inv_outdeg; 0 for dangling)   gathered
//   in.ptr     u64  CSR(G^T) offsets                                      streamed
//   in.idx     u32  CSR(G^T) sources                                      streamed
//   inv[N]     f32  1/outdeg                                              streamed
//   rank_n[N]  f32  written (double-buffered: the previous superstep's ranks stay
//                   readable for the stats pass, the SpMV never reads ranks)
//   x_next[N]  f32  written: the next superstep's message vector (the send phase
//                   is fused into this superstep's apply epilogue)
// Algorithmic bytes/superstep = 4·nnz + 8·(N+1) + 16·N.
//
// SpMV = merge-path over row-aligned tiles (Merrill & Garland's CSR merge
// SpMV, specialised): the row sequence is cut once (cached per graph) into
// tiles of at most kTile path items (rows + nonzeros).  A 256-thread CTA
// stages the tile's row ends (16-bit, tile-local) and the gathered x[col]
// values in shared memory (every gather of the tile in flight at once), each
// thread takes exactly kIPT path items found by a merge-path search in shared
// memory, and a block segmented scan hands partial row sums across threads.
// Rows longer than a tile are cut into tile-sized chunks, one CTA each, in the
// same launch; the last chunk of a row to finish folds the chunk sums in order.
// Every reduction is a fixed tree, so results are bitwise reproducible.
//
// Shared memory is kept small on purpose (12.3 KB per CTA): the L1 that the
// carveout leaves is what caches the hub entries of x (relabeling puts them at
// the low ids), and the kernel time tracks that hit rate.
//
// The dangling mass for the NEXT superstep's base is reduced from per-CTA
// partials in a fixed order by k_pr_base, on device: the supersteps run without
// a host round trip.  The updated-vertex count of a stats superstep is a
// separate streaming pass over the two rank buffers (k_pr_count).
#include <vector>

#include "api_internal.cuh"

namespace gm {

constexpr int kPrThreads = 256;
constexpr int kIPT = 8;
constexpr int kTile = kPrThreads * kIPT;  // path items per tile
static_assert(kTile < 0xFFFF, "tile-local row ends are 16-bit");
constexpr unsigned kDangBlocks = 296;

struct PrCache {
  uint64_t n = 0;
  uint64_t row_lo = 0, row_hi = 0;  // rows of G^T this process computes
  DevBuf<float> inv, rank0, rank1, x0, x1;
  int cur = 0;  // rank buffer holding the latest ranks
  DevBuf<uint32_t> tile_b, tile_e;
  DevBuf<uint32_t> chunk_row, chunk_slot, slot_first;  // long rows, kTile nnz per chunk
  DevBuf<float> chunk_sum;
  DevBuf<unsigned> slot_ticket;
  uint64_t ntiles = 0, n_long = 0, nchunks = 0;
  // Sharded exchange of only the non-dangling prefix of every block: the
  // owned rows' column ids remapped to the packed layout (block b's entry o
  // at b * pack_lmax + o), see pagerank_shard_pack.
  DevBuf<uint32_t> idx_packed;
  uint64_t pack_lmax = 0, pack_stride = 0, ptr_lo = 0;
  DevBuf<float> scalars;       // [0] = base for the current superstep
  DevBuf<float> dang_partial;  // per SpMV CTA (and kDangBlocks for the first base)
  DevBuf<unsigned long long> ctr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  float* rank() { return cur ? rank1.get() : rank0.get(); }
  float* rank_other() { return cur ? rank0.get() : rank1.get(); }
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

// vertices_updated of a stats superstep (rule S7): rows with at least one
// in-edge (a valid y) whose rank changed bitwise.  Streams ptr and both rank
// buffers once; one atomic per warp.
__global__ void k_pr_count(uint64_t lo, uint64_t hi, const uint64_t* ptr, const float* old_rank,
                           const float* new_rank, unsigned long long* ctr) {
  unsigned long long c = 0;
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x)
    c += ptr[v + 1] != ptr[v] && __float_as_uint(old_rank[v]) != __float_as_uint(new_rank[v]);
  warp_add_u64(ctr, c);
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

// Fused all-gather (multi-GPU shards): the epilogue stores each message
// straight into every rank's full message vector over NVLink peer memory
// (CUDA IPC mappings; the local buffer is one of them), at row + off, for
// the rows of the block's gathered prefix (row - lo < lim).  n == 0: the
// message goes to x_next only.
constexpr int kMaxPeers = 8;
struct PeerOut {
  float* p[kMaxPeers];
  uint32_t n;
  int64_t off;
  uint64_t lo, lim;
};

// Apply + send for one row: stores only, plus the inv read.
__device__ __forceinline__ void pr_write(uint64_t row, float sum, float base, float damping,
                                         const float* __restrict__ inv, float* __restrict__ rank,
                                         float* __restrict__ x_next, const PeerOut& po,
                                         float& dangling) {
  const float r = base + damping * sum;
  rank[row] = r;
  const float iv = __ldg(&inv[row]);
  const float x = r * iv;
  if (po.n == 0) {
    x_next[row] = x;
  } else if (row - po.lo < po.lim) {
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q < int(po.n)) po.p[q][int64_t(row) + po.off] = x;
  }
  if (iv == 0.0f) dangling += r;
}

// One superstep's SpMV launch: blocks [0, nchunks) take one kTile-nnz chunk of
// a long row each (the heaviest work first), blocks [nchunks, nchunks+ntiles)
// one merge-path tile each.  Dangling partials: tiles at [0, ntiles), long row
// `slot` at ntiles + slot.
struct PrArgs {
  const uint32_t* tile_b;
  const uint32_t* tile_e;
  const uint64_t* ptr;
  const uint32_t* idx;
  const float* x_cur;
  const float* inv;
  float* rank;  // this superstep's output buffer
  float* x_next;
  const float* scalars;
  float damping;
  uint32_t ntiles, nchunks;
  const uint32_t* chunk_row;   // [nchunks] row of G^T
  const uint32_t* chunk_slot;  // [nchunks] long-row slot
  const uint32_t* slot_first;  // [n_long + 1] first chunk of each long row
  float* chunk_sum;            // [nchunks]
  unsigned* slot_ticket;       // [n_long] arrivals this superstep (reset by the last)
  float* dang_partial;
  PeerOut peers;
};

// A long row is cut into chunks of kTile nonzeros, one CTA each (all gathers
// in flight, fixed-tree block sum).  The CTA that completes a row last (ticket)
// folds the row's chunk sums in chunk order, so the result does not depend on
// which CTA finishes last, and runs the apply + send epilogue.
__device__ __forceinline__ void pr_chunk(const PrArgs& a, float* s_red) {
  const unsigned tid = threadIdx.x;
  const uint32_t ci = blockIdx.x;
  const uint32_t row = a.chunk_row[ci], slot = a.chunk_slot[ci];
  const uint32_t f = a.slot_first[slot], nch = a.slot_first[slot + 1] - f;
  const uint64_t re = a.ptr[row + 1];
  const uint64_t beg = a.ptr[row] + uint64_t(ci - f) * kTile;
  const uint32_t len = uint32_t(min(uint64_t(kTile), re - beg));
  float v[kIPT];
#pragma unroll
  for (int u = 0; u < kIPT; ++u) {
    const uint32_t k = tid + u * kPrThreads;
    v[u] = k < len ? __ldg(&a.x_cur[__ldg(&a.idx[beg + k])]) : 0.0f;
  }
  float acc = 0.0f;
#pragma unroll
  for (int u = 0; u < kIPT; ++u) acc += v[u];
  acc = block_sum<kPrThreads>(acc, s_red);
  if (tid != 0) return;
  a.chunk_sum[ci] = acc;
  __threadfence();
  if (atomicAdd(&a.slot_ticket[slot], 1u) != nch - 1) return;
  __threadfence();
  float sum = 0.0f;
  for (uint32_t i = 0; i < nch; ++i) sum += __ldcg(&a.chunk_sum[f + i]);
  a.slot_ticket[slot] = 0;
  float dangling = 0.0f;
  pr_write(row, sum, a.scalars[0], a.damping, a.inv, a.rank, a.x_next, a.peers, dangling);
  a.dang_partial[a.ntiles + slot] = dangling;
}

__global__ void __launch_bounds__(kPrThreads) k_pr_spmv(const PrArgs a) {
  __shared__ uint16_t s_end[kTile + 1];  // tile-local row ends (exclusive nnz offsets)
  __shared__ float s_val[kTile];         // gathered x[col] of the tile's nonzeros
  __shared__ float s_red[kPrThreads / 32];
  __shared__ uint32_t s_wk[kPrThreads / 32];
  __shared__ float s_wv[kPrThreads / 32];
  if (blockIdx.x < a.nchunks) {
    pr_chunk(a, s_red);
    return;
  }
  const uint64_t* __restrict__ ptr = a.ptr;
  const float damping = a.damping;
  const uint32_t tile = blockIdx.x - a.nchunks;
  float dangling = 0.0f;
  const unsigned tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  const uint32_t r0 = a.tile_b[tile], r1 = a.tile_e[tile];
  const uint64_t j0 = ptr[r0];
  const uint32_t nrows = r1 - r0;
  const uint32_t nnz = uint32_t(ptr[r1] - j0);
  const uint32_t items = nrows + nnz;
  const float base = a.scalars[0];
  // Stage row ends and gathered messages; all gathers of the tile in flight.
  for (uint32_t k = tid; k < nrows; k += kPrThreads) s_end[k] = uint16_t(ptr[r0 + k + 1] - j0);
  if (tid == 0) s_end[nrows] = 0xFFFFu;
#pragma unroll
  for (int u = 0; u < kIPT; ++u) {
    const uint32_t k = tid + u * kPrThreads;
    if (k < nnz) s_val[k] = __ldg(&a.x_cur[__ldg(&a.idx[j0 + k])]);
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
  for (uint32_t k = d0; k < d1; ++k) {
    if (tj < s_end[ti]) {
      run += s_val[tj];
      ++tj;
    } else {
      if (!has_first) {
        has_first = true;
        first_val = run;
      } else {
        pr_write(r0 + ti, run, base, damping, a.inv, a.rank, a.x_next, a.peers, dangling);
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
    pr_write(r0 + start_row, carry + first_val, base, damping, a.inv, a.rank, a.x_next, a.peers,
             dangling);
  }
  // Dangling mass of this tile's rows, for the next superstep's base.
  const float dsum = block_sum<kPrThreads>(dangling, s_red);
  if (tid == 0) a.dang_partial[tile] = dsum;
}

// Row-aligned tiles of <= kTile path items; rows needing more than a tile are
// long rows, cut into chunks of kTile nonzeros.  One-time host pass over the
// offsets (cached with the graph).
void build_tiles(Graph& g, PrCache& c, cudaStream_t s, uint64_t lo, uint64_t n) {
  std::vector<uint64_t> ptr(g.n + 1);
  GM_CUDA(cudaMemcpyAsync(ptr.data(), g.in.ptr.get(), (g.n + 1) * 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  std::vector<uint32_t> tb, te, crow, cslot, sfirst;
  uint64_t r = lo;
  while (r < n) {
    const uint64_t deg = ptr[r + 1] - ptr[r];
    if (deg + 1 > uint64_t(kTile)) {
      sfirst.push_back(uint32_t(crow.size()));
      for (uint64_t k = 0; k < deg; k += kTile) {
        crow.push_back(uint32_t(r));
        cslot.push_back(uint32_t(sfirst.size() - 1));
      }
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
  c.n_long = sfirst.size();
  c.nchunks = crow.size();
  sfirst.push_back(uint32_t(crow.size()));
  if (c.ntiles + c.nchunks > 0x7FFFFFFFull) fail(GM_EENGINE, "pagerank: graph too large for one grid");
  auto up = [&](DevBuf<uint32_t>& d, const std::vector<uint32_t>& h) {
    d.alloc(h.size() + 1, s);
    if (!h.empty())
      GM_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * 4, cudaMemcpyHostToDevice, s));
  };
  up(c.tile_b, tb);
  up(c.tile_e, te);
  up(c.chunk_row, crow);
  up(c.chunk_slot, cslot);
  up(c.slot_first, sfirst);
  c.chunk_sum.alloc(c.nchunks + 1, s);
  c.slot_ticket.alloc(c.n_long + 1, s);
  c.slot_ticket.zero(s);
  GM_CUDA(cudaStreamSynchronize(s));
}

// Run one superstep's SpMV: reads x_cur, writes the other rank buffer and x_next.
void launch_spmv(Graph& g, PrCache& c, const float* x_cur, float* x_next, float damping,
                 cudaStream_t s, const PeerOut* peers = nullptr) {
  PrArgs a;
  if (peers)
    a.peers = *peers;
  else
    a.peers.n = 0;
  a.tile_b = c.tile_b.get();
  a.tile_e = c.tile_e.get();
  a.ptr = g.in.ptr.get();
  a.idx = c.pack_lmax ? c.idx_packed.get() - c.ptr_lo : g.in.idx.get();
  a.x_cur = x_cur;
  a.inv = c.inv.get();
  a.rank = c.rank_other();
  a.x_next = x_next;
  a.scalars = c.scalars.get();
  a.damping = damping;
  a.ntiles = uint32_t(c.ntiles);
  a.nchunks = uint32_t(c.nchunks);
  a.chunk_row = c.chunk_row.get();
  a.chunk_slot = c.chunk_slot.get();
  a.slot_first = c.slot_first.get();
  a.chunk_sum = c.chunk_sum.get();
  a.slot_ticket = c.slot_ticket.get();
  a.dang_partial = c.dang_partial.get();
  const unsigned grid = a.ntiles + a.nchunks;
  if (grid) {
    g.ktimer.begin(s, "k_pr_spmv");
    k_pr_spmv<<<grid, kPrThreads, 0, s>>>(a);
    g.ktimer.end(s);
    GM_LAUNCH_CHECK();
  }
  c.cur ^= 1;
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
    c.rank0.alloc(n, s);
    c.rank1.alloc(n, s);
    c.x0.alloc(n, s);
    c.x1.alloc(n, s);
    c.scalars.alloc(4, s);
    c.ctr.alloc(4, s);
    c.ctr.zero(s);
    GM_CUDA(cudaEventCreate(&c.e0));
    GM_CUDA(cudaEventCreate(&c.e1));
    build_tiles(g, c, s, lo, hi);
    c.dang_partial.alloc(std::max<uint64_t>(kDangBlocks, c.ntiles + c.n_long) + 1, s);
    GM_CUDA(cudaStreamSynchronize(s));
  }
  return *g.pr;
}

PrCache& cache(Graph& g) { return cache(g, 0, g.n); }

// Initial state: ranks 1/N in buffer 0, x = rank * inv.
void init_state(Graph& g, PrCache& c) {
  c.cur = 0;
  k_pr_init<<<grid_for(g.n, 256), 256, 0, g.stream>>>(g.n, g.outdeg.get(), c.inv.get(),
                                                       c.rank0.get(), c.x0.get());
  GM_LAUNCH_CHECK();
}

}  // namespace

std::vector<gm_iteration_stats> pagerank(Graph& g, double damping, int64_t iters, float* out,
                                         bool out_on_device, bool collect, bool async) {
  if (!(damping >= 0.0 && damping <= 1.0)) fail(GM_EINPUT, "pagerank: damping must be in [0, 1]");
  if (iters < 0) fail(GM_EUSAGE, "pagerank: negative iteration count");
  std::vector<gm_iteration_stats> stats;
  const uint64_t n = g.n;
  if (n == 0) return stats;
  if (pagerank_hub_enabled(g))
    return pagerank_hub(g, damping, iters, out, out_on_device, collect, async);
  if (g.pr && g.pr->pack_lmax) g.pr.reset();  // a packed shard layout is not the full vector
  PrCache& c = cache(g);
  cudaStream_t s = g.stream;
  const uint64_t dang_lo = (g.relabeled && g.shards == 1) ? g.nonzero_outdeg : 0;
  init_state(g, c);
  unsigned* ticket = reinterpret_cast<unsigned*>(c.ctr.get() + 3);
  GM_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  float* xc = c.x0.get();
  float* xn = c.x1.get();
  const float d = float(damping);
  // Base of the first superstep (initial ranks); later bases come from the
  // dangling partials the SpMV kernel emits (k_pr_base).
  k_dangling<<<kDangBlocks, 256, 0, s>>>(dang_lo, n, c.rank(), c.inv.get(), c.dang_partial.get(),
                                         c.scalars.get(), damping, ticket);
  GM_LAUNCH_CHECK();
  for (int64_t it = 1; it <= iters; ++it) {
    if (collect) GM_CUDA(cudaEventRecord(c.e0, s));
    launch_spmv(g, c, xc, xn, d, s);
    k_pr_base<<<1, 1024, 0, s>>>(c.dang_partial.get(), uint32_t(c.ntiles + c.n_long), n, damping,
                                 c.scalars.get());
    GM_LAUNCH_CHECK();
    std::swap(xc, xn);
    if (!collect) continue;
    GM_CUDA(cudaEventRecord(c.e1, s));
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
    k_pr_count<<<grid_for(n, 256), 256, 0, s>>>(0, n, g.in.ptr.get(), c.rank_other(), c.rank(),
                                                c.ctr.get());
    GM_LAUNCH_CHECK();
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
      to_external(g, c.rank(), out, 4);
    } else {
      DevBuf<float> ext(n, s);
      to_external(g, c.rank(), ext.get(), 4);
      GM_CUDA(cudaMemcpyAsync(out, ext.get(), n * 4, cudaMemcpyDeviceToHost, s));
    }
  }
  if (!async) GM_CUDA(cudaStreamSynchronize(s));
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

__global__ void k_pack_cols(const uint32_t* idx, uint64_t m, uint64_t stride, uint64_t lmax,
                            uint32_t* out, unsigned long long* bad) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < m;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = idx[j], b = c / stride, o = c % stride;
    if (o >= lmax) atomicAdd(bad, 1ull);
    out[j] = uint32_t(b * lmax + o);
  }
}

// Last non-dangling offset + 1 inside [lo, hi): every gathered column of a
// block lies below it (dangling sources have no out-edges).
__global__ void k_last_active(const float* inv, uint64_t lo, uint64_t hi, unsigned long long* last) {
  unsigned long long m = 0;
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x)
    if (inv[v] != 0.0f) m = max(m, (unsigned long long)(v - lo + 1));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31u) == 0 && m) atomicMax(last, m);
}

void check_block(Graph& g, uint64_t lo, uint64_t hi) {
  if (lo > hi || hi > g.n) fail(GM_EUSAGE, "pagerank shard: bad row block");
}

}  // namespace

double pagerank_shard_init(Graph& g, uint64_t lo, uint64_t hi, float* x_block) {
  check_block(g, lo, hi);
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  init_state(g, c);
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
  GM_CUDA(cudaMemcpyAsync(c.scalars.get(), &b, 4, cudaMemcpyHostToDevice, s));
  // the kernel writes x_next[row] for rows in [lo, hi) only
  launch_spmv(g, c, x_full, x_block - lo, float(damping), s);
  double* dsum = reinterpret_cast<double*>(c.ctr.get() + 2);
  k_sum_partials<<<1, 1024, 0, s>>>(c.dang_partial.get(), uint32_t(c.ntiles + c.n_long), dsum);
  GM_LAUNCH_CHECK();
  double h = 0.0;
  GM_CUDA(cudaMemcpyAsync(&h, dsum, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

namespace {
__global__ void k_push_block(const float* x, uint64_t lo, uint64_t cnt, PeerOut po) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t row = lo + i;
    const float v = x[row];
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q < int(po.n)) po.p[q][int64_t(row) + po.off] = v;
  }
}

PeerOut make_peers(float* const* peers, int npeers, int64_t offset, uint64_t lo, uint64_t limit) {
  if (npeers < 1 || npeers > kMaxPeers)
    fail(GM_EUSAGE, "pagerank shard: 1 to " + std::to_string(kMaxPeers) + " peer buffers");
  PeerOut po{};
  for (int q = 0; q < npeers; ++q) {
    if (!peers[q]) fail(GM_EUSAGE, "pagerank shard: null peer buffer");
    po.p[q] = peers[q];
  }
  po.n = uint32_t(npeers);
  po.off = offset;
  po.lo = lo;
  po.lim = limit;
  return po;
}
}  // namespace

// Initial messages of the block's gathered prefix into every peer buffer.
double pagerank_shard_init_peers(Graph& g, uint64_t lo, uint64_t hi, float* const* peers,
                                 int npeers, int64_t offset, uint64_t limit) {
  check_block(g, lo, hi);
  const PeerOut po = make_peers(peers, npeers, offset, lo, limit);
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  init_state(g, c);
  const uint64_t cnt = std::min<uint64_t>(hi - lo, limit);
  if (cnt) {
    k_push_block<<<grid_for(cnt, 256), 256, 0, s>>>(c.x0.get(), lo, cnt, po);
    GM_LAUNCH_CHECK();
  }
  GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
  if (hi > lo) {
    k_count_dangling<<<grid_for(hi - lo, 256), 256, 0, s>>>(c.inv.get(), lo, hi, c.ctr.get());
    GM_LAUNCH_CHECK();
  }
  unsigned long long dn = 0;
  GM_CUDA(cudaMemcpyAsync(&dn, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return double(dn) / double(g.n);
}

// The fused variant: no x_block; the messages go to the peers' buffers.
double pagerank_shard_step_peers(Graph& g, uint64_t lo, uint64_t hi, const float* x_full,
                                 double base, double damping, float* const* peers, int npeers,
                                 int64_t offset, uint64_t limit) {
  check_block(g, lo, hi);
  const PeerOut po = make_peers(peers, npeers, offset, lo, limit);
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  const float b = float(base);
  GM_CUDA(cudaMemcpyAsync(c.scalars.get(), &b, 4, cudaMemcpyHostToDevice, s));
  launch_spmv(g, c, x_full, nullptr, float(damping), s, &po);
  double* dsum = reinterpret_cast<double*>(c.ctr.get() + 2);
  k_sum_partials<<<1, 1024, 0, s>>>(c.dang_partial.get(), uint32_t(c.ntiles + c.n_long), dsum);
  GM_LAUNCH_CHECK();
  double h = 0.0;
  GM_CUDA(cudaMemcpyAsync(&h, dsum, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t pagerank_shard_active(Graph& g, uint64_t lo, uint64_t hi) {
  check_block(g, lo, hi);
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  init_state(g, c);
  GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
  if (hi > lo) {
    k_last_active<<<grid_for(hi - lo, 256), 256, 0, s>>>(c.inv.get(), lo, hi, c.ctr.get());
    GM_LAUNCH_CHECK();
  }
  unsigned long long h = 0;
  GM_CUDA(cudaMemcpyAsync(&h, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

void pagerank_shard_pack(Graph& g, uint64_t lo, uint64_t hi, uint64_t stride, uint64_t lmax) {
  check_block(g, lo, hi);
  if (stride == 0 || g.n % stride != 0) fail(GM_EUSAGE, "pagerank shard pack: bad block stride");
  if (lmax == 0 || lmax > stride) fail(GM_EUSAGE, "pagerank shard pack: bad prefix length");
  PrCache& c = cache(g, lo, hi);
  cudaStream_t s = g.stream;
  uint64_t pl = 0, ph = 0;
  GM_CUDA(cudaMemcpyAsync(&pl, g.in.ptr.get() + lo, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaMemcpyAsync(&ph, g.in.ptr.get() + hi, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  c.idx_packed.alloc(ph - pl + 1, s);
  GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
  if (ph > pl) {
    k_pack_cols<<<grid_for(ph - pl, 256), 256, 0, s>>>(g.in.idx.get() + pl, ph - pl, stride, lmax,
                                                       c.idx_packed.get(), c.ctr.get());
    GM_LAUNCH_CHECK();
  }
  unsigned long long bad = 0;
  GM_CUDA(cudaMemcpyAsync(&bad, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (bad) fail(GM_EUSAGE, "pagerank shard pack: a gathered column lies past the packed prefix");
  c.ptr_lo = pl;
  c.pack_stride = stride;
  c.pack_lmax = lmax;
}

void pagerank_shard_ranks(Graph& g, uint64_t lo, uint64_t hi, float* out_host) {
  check_block(g, lo, hi);
  PrCache& c = cache(g, lo, hi);
  if (hi > lo)
    GM_CUDA(cudaMemcpyAsync(out_host, c.rank() + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost,
                            g.stream));
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

}  // namespace gm
