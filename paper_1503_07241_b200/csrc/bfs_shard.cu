// bfs_shard.cu -- multi-GPU BFS superstep on one rank's row block.
//
// 1-D row sharding of the symmetric graph, like the reference's row
// partitions (include/semigraph/dcsc.hpp:77-105): rank r owns the vertices
// [lo, hi) (GM_SHARDS(P) makes those blocks nnz-balanced) and is the only
// writer of their levels and next-frontier bits.  Per superstep every rank
// holds the same full frontier bitmap and visited bitmap; the caller
// all-gathers the next-frontier blocks (N/8/P bytes per rank) and ORs them into
// visited, and all-reduces two scalars (vertices found, their edges) that drive
// the push/pull decision identically on every rank -- the single-GPU rule of
// k_bfs_coop: pull once frontier edges exceed 5% of m, back to push once the
// frontier drops below n/24.
//
//   push: every frontier vertex u (a queue built from the frontier bitmap) is
//         expanded over the part of its sorted adjacency that lies inside
//         [lo, hi) (two binary searches), so the ranks split the frontier's
//         edges by destination without replicating work;
//   pull: every unvisited owned row scans its in-neighbours until one is in
//         the frontier (early exit).
// Levels equal the reference's: a vertex gets the superstep that first reaches
// it (traversal.hpp:39-63 under engine.hpp:193-213).
#include "api_internal.cuh"

namespace gm {

struct BfsShardCache {
  uint64_t lo = 0, hi = 0;
  DevBuf<int32_t> level;           // [hi - lo]
  DevBuf<uint32_t> queue;          // frontier vertices (push)
  DevBuf<unsigned long long> ctr;  // [0] queue length, [1] found, [2] found edges
};

namespace {

constexpr unsigned kSbThreads = 256;

__global__ void k_sb_init(int32_t* level, uint64_t lo, uint64_t hi, uint64_t root) {
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x)
    level[v - lo] = v == root ? 0 : -1;
}

// Frontier bitmap -> queue (order irrelevant: pushes only set bits / levels).
__global__ void k_sb_queue(const uint32_t* fb, uint64_t words, uint32_t* q,
                           unsigned long long* qn) {
  for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < words;
       w += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t bits = fb[w];
    if (!bits) continue;
    const unsigned long long base = atomicAdd(qn, (unsigned long long)__popc(bits));
    unsigned k = 0;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      q[base + k++] = uint32_t(w * 32 + b);
    }
  }
}

__device__ __forceinline__ uint64_t lower_bound64(const uint32_t* a, uint64_t lo, uint64_t hi,
                                                  uint64_t x) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Claim v (owned) for the next frontier: the next-frontier block bit is the
// claim, so each vertex is counted and labelled once.
__device__ __forceinline__ bool claim(uint32_t v, uint64_t lo, uint32_t* next_blk) {
  const uint64_t o = v - lo;
  const uint32_t bit = 1u << (o & 31u);
  return !(atomicOr(&next_blk[o >> 5], bit) & bit);
}

__global__ void __launch_bounds__(kSbThreads) k_sb_push(
    const uint32_t* __restrict__ q, const unsigned long long* qn, const uint64_t* __restrict__ ptr,
    const uint32_t* __restrict__ idx, const uint32_t* __restrict__ vis, uint64_t lo, uint64_t hi,
    int32_t lvl, int32_t* level, uint32_t* next_blk, unsigned long long* found) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t nq = *qn;
  unsigned long long f = 0, fe = 0;
  for (uint64_t i = warp; i < nq; i += nwarps) {
    const uint32_t u = q[i];
    const uint64_t b = ptr[u], e = ptr[u + 1];
    // the slice of u's sorted adjacency inside [lo, hi)
    const uint64_t s0 = lower_bound64(idx, b, e, lo), s1 = lower_bound64(idx, s0, e, hi);
    for (uint64_t k = s0 + lane; k < s1; k += 32) {
      const uint32_t v = idx[k];
      if ((__ldcg(&vis[v >> 5]) >> (v & 31u)) & 1u) continue;
      if (claim(v, lo, next_blk)) {
        level[v - lo] = lvl;
        ++f;
        fe += ptr[v + 1] - ptr[v];
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    fe += __shfl_xor_sync(0xffffffffu, fe, o);
  }
  if (lane == 0 && f) {
    atomicAdd(&found[0], f);
    atomicAdd(&found[1], fe);
  }
}

__global__ void __launch_bounds__(kSbThreads) k_sb_pull(
    const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ fb, const uint32_t* __restrict__ vis, uint64_t lo, uint64_t hi,
    int32_t lvl, int32_t* level, uint32_t* next_blk, unsigned long long* found) {
  unsigned long long f = 0, fe = 0;
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x) {
    if ((vis[v >> 5] >> (v & 31u)) & 1u) continue;
    const uint64_t b = ptr[v], e = ptr[v + 1];
    for (uint64_t k = b; k < e; ++k) {
      const uint32_t u = __ldg(&idx[k]);
      if ((__ldg(&fb[u >> 5]) >> (u & 31u)) & 1u) {
        if (claim(uint32_t(v), lo, next_blk)) {
          level[v - lo] = lvl;
          ++f;
          fe += e - b;
        }
        break;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    fe += __shfl_xor_sync(0xffffffffu, fe, o);
  }
  if ((threadIdx.x & 31u) == 0 && f) {
    atomicAdd(&found[0], f);
    atomicAdd(&found[1], fe);
  }
}

// The block's next-frontier words stored into every rank's frontier bitmap
// for the next superstep (CUDA IPC peer mappings, the local one included):
// the all-gather as NVLink stores.  Whole words are stored, zeros included,
// so a target buffer never needs clearing (each word has one writer).
constexpr int kMaxPeerBufs = 8;
struct PeerWords {
  uint32_t* p[kMaxPeerBufs];
  int n;
};

__global__ void k_sb_peer_store(const uint32_t* next_blk, uint64_t w0, uint64_t nw, PeerWords pw) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nw;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = next_blk[i];
#pragma unroll
    for (int q = 0; q < kMaxPeerBufs; ++q)
      if (q < pw.n) pw.p[q][w0 + i] = v;
  }
}

void check_sb(Graph& g, uint64_t lo, uint64_t hi) {
  if (!g.symmetric) fail(GM_EUSAGE, "bfs shard: needs a symmetric graph (GM_SYMMETRIZE)");
  if (lo > hi || hi > g.n || (lo & 31u) || ((hi & 31u) && hi != g.n))
    fail(GM_EUSAGE, "bfs shard: row block must be 32-vertex aligned");
}

BfsShardCache& sb_cache(Graph& g, uint64_t lo, uint64_t hi) {
  if (!g.bfs_shard || g.bfs_shard->lo != lo || g.bfs_shard->hi != hi) {
    g.bfs_shard = std::unique_ptr<BfsShardCache, void (*)(BfsShardCache*)>(
        new BfsShardCache(), [](BfsShardCache* p) { delete p; });
    BfsShardCache& c = *g.bfs_shard;
    c.lo = lo;
    c.hi = hi;
    c.level.alloc(hi - lo + 1, g.stream);
    c.queue.alloc(g.n + 1, g.stream);
    c.ctr.alloc(4, g.stream);
  }
  return *g.bfs_shard;
}

}  // namespace

void bfs_shard_init(Graph& g, uint64_t lo, uint64_t hi, uint64_t root_internal) {
  check_sb(g, lo, hi);
  if (root_internal >= g.n) fail(GM_EINPUT, "bfs shard: root out of range");
  BfsShardCache& c = sb_cache(g, lo, hi);
  if (hi > lo) {
    k_sb_init<<<grid_for(hi - lo, 256), 256, 0, g.stream>>>(c.level.get(), lo, hi, root_internal);
    GM_LAUNCH_CHECK();
  }
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

void bfs_shard_step(Graph& g, uint64_t lo, uint64_t hi, const uint32_t* frontier,
                    const uint32_t* visited, int32_t lvl, int32_t pull, uint32_t* next_block,
                    uint64_t* found, uint64_t* found_edges) {
  check_sb(g, lo, hi);
  BfsShardCache& c = sb_cache(g, lo, hi);
  cudaStream_t s = g.stream;
  const uint64_t words_blk = (hi - lo + 31) / 32;
  if (words_blk) GM_CUDA(cudaMemsetAsync(next_block, 0, words_blk * 4, s));
  GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 4 * 8, s));
  const Csr& a = g.in;  // symmetric: CSR(G^T) == CSR(G)
  if (pull) {
    if (hi > lo) {
      k_sb_pull<<<grid_for(hi - lo, kSbThreads), kSbThreads, 0, s>>>(
          a.ptr.get(), a.idx.get(), frontier, visited, lo, hi, lvl, c.level.get(), next_block,
          c.ctr.get() + 1);
      GM_LAUNCH_CHECK();
    }
  } else {
    const uint64_t words = (g.n + 31) / 32;
    k_sb_queue<<<grid_for(words, 256), 256, 0, s>>>(frontier, words, c.queue.get(), c.ctr.get());
    GM_LAUNCH_CHECK();
    k_sb_push<<<148u * 8u, kSbThreads, 0, s>>>(c.queue.get(), c.ctr.get(), a.ptr.get(), a.idx.get(),
                                               visited, lo, hi, lvl, c.level.get(), next_block,
                                               c.ctr.get() + 1);
    GM_LAUNCH_CHECK();
  }
  unsigned long long h[2] = {0, 0};
  GM_CUDA(cudaMemcpyAsync(h, c.ctr.get() + 1, 16, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (found) *found = h[0];
  if (found_edges) *found_edges = h[1];
}

void bfs_shard_push(Graph& g, uint64_t lo, uint64_t hi, const uint32_t* next_block,
                    uint32_t* const* peers, int npeers) {
  check_sb(g, lo, hi);
  if (npeers < 1 || npeers > kMaxPeerBufs)
    fail(GM_EUSAGE, "bfs shard: 1 to " + std::to_string(kMaxPeerBufs) + " peer bitmaps");
  PeerWords pw{};
  for (int q = 0; q < npeers; ++q) {
    if (!peers[q]) fail(GM_EUSAGE, "bfs shard: null peer bitmap");
    pw.p[q] = peers[q];
  }
  pw.n = npeers;
  const uint64_t nw = (hi - lo + 31) / 32;
  if (nw) {
    k_sb_peer_store<<<grid_for(nw, 256), 256, 0, g.stream>>>(next_block, lo / 32, nw, pw);
    GM_LAUNCH_CHECK();
  }
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

namespace {
__global__ void k_bits_or(uint32_t* dst, const uint32_t* src, uint64_t words) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] |= src[i];
}
}  // namespace

void bitmap_or(Graph& g, uint32_t* dst, const uint32_t* src, uint64_t words) {
  if (words) {
    k_bits_or<<<grid_for(words, 256), 256, 0, g.stream>>>(dst, src, words);
    GM_LAUNCH_CHECK();
  }
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

// A device block stored into every peer buffer at the same byte offset (the
// exchange of the SSSP / CF shards as NVLink peer copies instead of an
// all-gather); copies on the graph's stream, then a sync.
void push_block(Graph& g, const void* src, uint64_t bytes, void* const* peers, int npeers,
                uint64_t dst_offset) {
  if (npeers < 1 || npeers > kMaxPeerBufs)
    fail(GM_EUSAGE, "push block: 1 to " + std::to_string(kMaxPeerBufs) + " peer buffers");
  for (int q = 0; q < npeers; ++q) {
    if (!peers[q]) fail(GM_EUSAGE, "push block: null peer buffer");
    if (bytes)
      GM_CUDA(cudaMemcpyAsync(static_cast<char*>(peers[q]) + dst_offset, src, bytes,
                              cudaMemcpyDeviceToDevice, g.stream));
  }
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

void bfs_shard_levels(Graph& g, uint64_t lo, uint64_t hi, int32_t* out_host) {
  check_sb(g, lo, hi);
  BfsShardCache& c = sb_cache(g, lo, hi);
  if (hi > lo)
    GM_CUDA(cudaMemcpyAsync(out_host, c.level.get(), (hi - lo) * 4, cudaMemcpyDeviceToHost,
                            g.stream));
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

}  // namespace gm
