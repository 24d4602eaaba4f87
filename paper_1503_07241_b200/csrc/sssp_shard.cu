// sssp_shard.cu -- multi-GPU SSSP superstep on one rank's row block.
//
// Bulk-synchronous Bellman-Ford (SsspProgram, traversal.hpp:67-91, driven by
// run_distance_program :95-115 under engine.hpp:193-213) with 1-D row
// sharding like the reference's row partitions (dcsc.hpp:77-105): rank r owns
// the vertices [lo, hi) and is the only writer of their distances.  Every rank
// holds the same full message vector msg (uint32, the superstep-start
// distance of every frontier vertex, UINT32_MAX elsewhere -- the snapshot rule
// S3); per superstep the ranks all-gather their blocks of the next msg and
// sum-reduce (changed, changed out-edges), which drive the single-GPU
// direction rule (pull once frontier out-edges exceed m/6) and termination.
//
//   push: the frontier (a queue built from msg) is relaxed over the slice of
//         each vertex's sorted out-adjacency inside [lo, hi) (two binary
//         searches: the ranks split the frontier's edges by destination);
//         atomicMin on the owned distance, a changed bit on improvement;
//   pull: every owned row takes min over its in-neighbours u of msg[u] + w.
// Both compute min(dist[v], min over frontier u of snapshot(u) + w(u, v)), so
// distances and per-superstep counts equal the reference's.
#include "api_internal.cuh"

namespace gm {

struct SsspShardCache {
  uint64_t lo = 0, hi = 0;
  DevBuf<uint32_t> dist;           // [hi - lo]
  DevBuf<uint32_t> changed;        // block bitmap
  DevBuf<uint32_t> queue;          // frontier vertices (push)
  DevBuf<unsigned long long> ctr;  // [0] queue length, [1] changed, [2] changed out-edges
};

namespace {

constexpr unsigned kSsThreads = 256;
constexpr uint32_t kInf = 0xFFFFFFFFu;

__global__ void k_ss_init(uint32_t* dist, uint64_t lo, uint64_t hi, uint64_t root) {
  for (uint64_t v = lo + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x)
    dist[v - lo] = v == root ? 0u : kInf;
}

// Frontier = vertices with a message (order irrelevant: relaxations are mins).
__global__ void k_ss_queue(const uint32_t* msg, uint64_t n, uint32_t* q, unsigned long long* qn) {
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t v0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); v0 < n;
       v0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t v = v0 + lane;
    const bool in = v < n && msg[v] != kInf;
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(qn, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (in) q[base + __popc(m & ((1u << lane) - 1u))] = uint32_t(v);
  }
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t lo, uint64_t hi,
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

template <typename W>
__global__ void __launch_bounds__(kSsThreads) k_ss_push(
    const uint32_t* __restrict__ q, const unsigned long long* qn, const uint64_t* __restrict__ ptr,
    const uint32_t* __restrict__ idx, const W* __restrict__ wt, const uint32_t* __restrict__ msg,
    uint64_t lo, uint64_t hi, uint32_t* dist, uint32_t* changed) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t nq = *qn;
  for (uint64_t i = warp; i < nq; i += nwarps) {
    const uint32_t u = q[i];
    const uint32_t du = msg[u];
    const uint64_t b = ptr[u], e = ptr[u + 1];
    const uint64_t s0 = lower_bound_u32(idx, b, e, lo), s1 = lower_bound_u32(idx, s0, e, hi);
    for (uint64_t k = s0 + lane; k < s1; k += 32) {
      const uint32_t v = idx[k];
      const uint32_t nd = du + uint32_t(wt[k]);
      if (nd < du) continue;  // beyond uint32: unreachable as a distance
      const uint64_t o = v - lo;
      if (nd < atomicMin(&dist[o], nd)) atomicOr(&changed[o >> 5], 1u << (o & 31u));
    }
  }
}

// a warp per owned row: lane-strided min over the row's in-neighbours
template <typename W>
__global__ void __launch_bounds__(kSsThreads) k_ss_pull(
    const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx, const W* __restrict__ wt,
    const uint32_t* __restrict__ msg, uint64_t lo, uint64_t hi, uint32_t* dist, uint32_t* changed) {
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t v = lo + (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / 32; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x / 32) {
    const uint64_t b = ptr[v], e = ptr[v + 1];
    uint32_t best = kInf;
    for (uint64_t k = b + lane; k < e; k += 32) {
      const uint32_t du = __ldg(&msg[idx[k]]);
      if (du == kInf) continue;
      const uint32_t nd = du + uint32_t(wt[k]);
      if (nd >= du) best = min(best, nd);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    const uint64_t o = v - lo;
    if (lane == 0 && best < dist[o]) {
      dist[o] = best;  // the row's only writer
      atomicOr(&changed[o >> 5], 1u << (o & 31u));  // 32 rows (warps) share a word
    }
  }
}

// next messages of the block: the new distance of every changed vertex
// (its snapshot for the next superstep), INF elsewhere; counts for the rule
__global__ void k_ss_emit(uint64_t lo, uint64_t hi, const uint32_t* dist, uint32_t* changed,
                          const uint64_t* __restrict__ out_ptr, uint32_t* msg_block,
                          unsigned long long* ctr) {
  unsigned long long c = 0, ce = 0;
  for (uint64_t o = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; o < hi - lo;
       o += uint64_t(gridDim.x) * blockDim.x) {
    const bool ch = (changed[o >> 5] >> (o & 31u)) & 1u;
    msg_block[o] = ch ? dist[o] : kInf;
    if (ch) {
      ++c;
      ce += out_ptr[lo + o + 1] - out_ptr[lo + o];
    }
  }
  warp_add_u64(&ctr[1], c);
  warp_add_u64(&ctr[2], ce);
}

void check_ss(Graph& g, uint64_t lo, uint64_t hi) {
  if (g.value_type != GM_VAL_U8 && g.value_type != GM_VAL_U32)
    fail(GM_EUSAGE, std::string("sssp shard: needs u8 or u32 edge weights, graph stores ") +
                        value_name(g.value_type));
  if (lo > hi || hi > g.n || (lo & 31u) || ((hi & 31u) && hi != g.n))
    fail(GM_EUSAGE, "sssp shard: row block must be 32-vertex aligned");
}

SsspShardCache& ss_cache(Graph& g, uint64_t lo, uint64_t hi) {
  if (!g.sssp_shard || g.sssp_shard->lo != lo || g.sssp_shard->hi != hi) {
    g.sssp_shard = std::unique_ptr<SsspShardCache, void (*)(SsspShardCache*)>(
        new SsspShardCache(), [](SsspShardCache* p) { delete p; });
    SsspShardCache& c = *g.sssp_shard;
    c.lo = lo;
    c.hi = hi;
    c.dist.alloc(hi - lo + 1, g.stream);
    c.changed.alloc((hi - lo + 31) / 32 + 1, g.stream);
    c.queue.alloc(g.n + 1, g.stream);
    c.ctr.alloc(4, g.stream);
  }
  return *g.sssp_shard;
}

template <typename W>
void ss_step(Graph& g, SsspShardCache& c, const uint32_t* msg, bool pull, cudaStream_t s) {
  const uint64_t lo = c.lo, hi = c.hi;
  if (pull) {
    const W* wt = reinterpret_cast<const W*>(g.in.val.get());
    if (hi > lo) {
      k_ss_pull<W><<<grid_for((hi - lo) * 32, kSsThreads), kSsThreads, 0, s>>>(
          g.in.ptr.get(), g.in.idx.get(), wt, msg, lo, hi, c.dist.get(), c.changed.get());
      GM_LAUNCH_CHECK();
    }
  } else {
    const Csr& fw = g.fwd();
    k_ss_queue<<<grid_for(g.n, 256), 256, 0, s>>>(msg, g.n, c.queue.get(), c.ctr.get());
    GM_LAUNCH_CHECK();
    k_ss_push<W><<<148u * 8u, kSsThreads, 0, s>>>(c.queue.get(), c.ctr.get(), fw.ptr.get(),
                                                  fw.idx.get(), reinterpret_cast<const W*>(fw.val.get()),
                                                  msg, lo, hi, c.dist.get(), c.changed.get());
    GM_LAUNCH_CHECK();
  }
}

}  // namespace

void sssp_shard_init(Graph& g, uint64_t lo, uint64_t hi, uint64_t root_internal) {
  check_ss(g, lo, hi);
  if (root_internal >= g.n) fail(GM_EINPUT, "sssp shard: root out of range");
  ensure_forward(g);
  SsspShardCache& c = ss_cache(g, lo, hi);
  if (hi > lo) {
    k_ss_init<<<grid_for(hi - lo, 256), 256, 0, g.stream>>>(c.dist.get(), lo, hi, root_internal);
    GM_LAUNCH_CHECK();
  }
  c.changed.zero(g.stream);
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

void sssp_shard_step(Graph& g, uint64_t lo, uint64_t hi, const uint32_t* msg, int32_t pull,
                     uint32_t* msg_block, uint64_t* changed, uint64_t* changed_edges) {
  check_ss(g, lo, hi);
  ensure_forward(g);
  SsspShardCache& c = ss_cache(g, lo, hi);
  cudaStream_t s = g.stream;
  GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 4 * 8, s));
  if (g.value_type == GM_VAL_U8)
    ss_step<uint8_t>(g, c, msg, pull != 0, s);
  else
    ss_step<uint32_t>(g, c, msg, pull != 0, s);
  if (hi > lo) {
    k_ss_emit<<<grid_for(hi - lo, 256), 256, 0, s>>>(lo, hi, c.dist.get(), c.changed.get(),
                                                    g.fwd().ptr.get(), msg_block, c.ctr.get());
    GM_LAUNCH_CHECK();
  }
  c.changed.zero(s);
  unsigned long long h[2] = {0, 0};
  GM_CUDA(cudaMemcpyAsync(h, c.ctr.get() + 1, 16, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (changed) *changed = h[0];
  if (changed_edges) *changed_edges = h[1];
}

void sssp_shard_dists(Graph& g, uint64_t lo, uint64_t hi, uint32_t* out_host) {
  check_ss(g, lo, hi);
  SsspShardCache& c = ss_cache(g, lo, hi);
  if (hi > lo)
    GM_CUDA(cudaMemcpyAsync(out_host, c.dist.get(), (hi - lo) * 4, cudaMemcpyDeviceToHost,
                            g.stream));
  GM_CUDA(cudaStreamSynchronize(g.stream));
}

}  // namespace gm
