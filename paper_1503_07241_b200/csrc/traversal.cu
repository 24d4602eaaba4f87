// traversal.cu -- BFS and SSSP supersteps: push SpMSpV / pull SpMV with a
// direction switch, bitmap frontiers, exact bulk-synchronous semantics.
//
// Reference: BfsProgram / SsspProgram (include/semigraph/algorithms/traversal.hpp:39-91)
// run by run_distance_program (:95-115) through Engine::run_graph_program
// (include/semigraph/engine.hpp:193-213).  The reference scans every stored
// column of every partition each superstep (engine.hpp:234-236); here a
// superstep touches only the frontier (push) or only unvisited vertices (pull).
//
// BFS (min over level+1): results and per-superstep stats (active_before =
// messages_generated = |frontier|, vertices_updated = |next frontier|) equal the
// reference's exactly, because a vertex's level is written once, in the
// superstep that first reaches it, whichever direction runs.
//   push  (frontier queue -> CSR(G) out-edges): one warp per frontier vertex,
//         visited bitmap claimed with atomicOr (each vertex enqueued once).
//   pull  (unvisited vertices -> CSR(G^T) in-edges): one thread per vertex,
//         early exit at the first in-neighbour in the frontier bitmap; with
//         GM_RELABEL the adjacency is ordered hub-first so the exit is early.
//   switch: pull while frontier edges > kPullFraction * m (BASELINE configs[1]).
// SSSP (min over dist+w, uint32, UINT32_MAX = unreached): push with the
// frontier's superstep-start distances carried in the queue (the message
// snapshot, S3), atomicMin into dist; a vertex whose distance dropped is
// claimed once in a changed-bitmap and becomes the next frontier.  Per-
// superstep stats equal the reference's.
#include <vector>

#include "api_internal.cuh"

namespace gm {

struct TravCache {
  uint64_t n = 0;
  DevBuf<int32_t> level;
  DevBuf<uint32_t> dist;
  DevBuf<uint32_t> q0, q1;        // frontier queues (vertex ids)
  DevBuf<uint32_t> d0, d1;        // SSSP message snapshots parallel to the queues
  DevBuf<uint32_t> vis, fb, nbm;  // visited / frontier / next-frontier bitmaps
  DevBuf<unsigned long long> ctr; // [0] next count [1] next edges [2] examined
};

namespace {

constexpr double kPullFraction = 0.05;

TravCache& cache(Graph& g) {
  if (!g.trav) {
    g.trav = std::unique_ptr<TravCache, void (*)(TravCache*)>(new TravCache(),
                                                              [](TravCache* p) { delete p; });
    TravCache& c = *g.trav;
    cudaStream_t s = g.stream;
    const uint64_t n = g.n, words = (n + 31) / 32 + 1;
    c.n = n;
    c.q0.alloc(n + 1, s);
    c.q1.alloc(n + 1, s);
    c.vis.alloc(words, s);
    c.fb.alloc(words, s);
    c.nbm.alloc(words, s);
    c.ctr.alloc(8, s);
  }
  return *g.trav;
}

// ------------------------------------------------------------------- BFS
__global__ void k_bfs_init(int32_t* level, uint32_t* vis, uint64_t n, uint32_t root,
                           uint32_t* queue) {
  const uint64_t words = (n + 31) / 32 + 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n || i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (i < n) level[i] = i == root ? 0 : -1;
    if (i < words) vis[i] = (i == (root >> 5)) ? (1u << (root & 31u)) : 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) queue[0] = root;
}

// Push: one warp per frontier vertex, lanes stride its out-edges.
__global__ void __launch_bounds__(256) k_bfs_push(const uint32_t* __restrict__ q, uint32_t nq,
                                                  const uint64_t* __restrict__ ptr,
                                                  const uint32_t* __restrict__ idx,
                                                  const uint32_t* __restrict__ deg, int32_t* level,
                                                  uint32_t* vis, int32_t next_level,
                                                  uint32_t* qn, unsigned long long* ctr) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long my_edges = 0;
  for (uint64_t i = warp; i < nq; i += nwarps) {
    const uint32_t u = q[i];
    const uint64_t beg = ptr[u], end = ptr[u + 1];
    for (uint64_t base = beg; base < end; base += 32) {
      const uint64_t e = base + lane;
      bool won = false;
      uint32_t v = 0;
      if (e < end) {
        v = idx[e];
        const uint32_t bit = 1u << (v & 31u);
        if (!(vis[v >> 5] & bit)) {
          const uint32_t old = atomicOr(&vis[v >> 5], bit);
          won = !(old & bit);
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, won);
      if (b) {
        uint32_t at = 0;
        if (lane == 0) at = uint32_t(atomicAdd(&ctr[0], (unsigned long long)__popc(b)));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (won) {
          level[v] = next_level;
          qn[at + __popc(b & ((1u << lane) - 1u))] = v;
          my_edges += deg[v];
        }
      }
    }
  }
  warp_add_u64(&ctr[1], my_edges);
}

// Pull: thread per vertex in [0, nv); unvisited vertices look for a frontier
// in-neighbour and stop at the first one.
__global__ void __launch_bounds__(256) k_bfs_pull(uint64_t nv, const uint64_t* __restrict__ ptr,
                                                  const uint32_t* __restrict__ idx,
                                                  const uint32_t* __restrict__ fb, uint32_t* vis,
                                                  uint32_t* nbm, int32_t* level,
                                                  int32_t next_level, unsigned long long* ctr) {
  const uint64_t words = (nv + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint32_t vw = vis[w];
    const uint64_t v = w * 32 + lane;
    bool found = false;
    if (v < nv && !((vw >> lane) & 1u)) {
      const uint64_t beg = ptr[v], end = ptr[v + 1];
      for (uint64_t e = beg; e < end; ++e) {
        const uint32_t u = idx[e];
        ++examined;
        if (bit_test(fb, u)) {
          found = true;
          break;
        }
      }
      if (found) {
        level[v] = next_level;
        found_e += end - beg;
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, found);
    if (lane == 0) {
      nbm[w] = b;
      if (b) vis[w] = vw | b;
    }
    found_n += found;
  }
  warp_add_u64(&ctr[0], found_n);
  warp_add_u64(&ctr[1], found_e);
  warp_add_u64(&ctr[2], examined);
}

__global__ void k_queue_to_bitmap(const uint32_t* q, uint32_t nq, uint32_t* bm) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x) {
    const uint32_t v = q[i];
    atomicOr(&bm[v >> 5], 1u << (v & 31u));
  }
}

__global__ void k_bitmap_to_queue(const uint32_t* bm, uint64_t words, uint32_t* q,
                                  unsigned long long* cnt) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t w0 = warp * 32; w0 < words; w0 += nwarps * 32) {
    const uint64_t w = w0 + lane;
    const uint32_t word = w < words ? bm[w] : 0u;
    const uint32_t c = __popc(word);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t base = 0;
    if (lane == 31 && total) base = uint32_t(atomicAdd(cnt, (unsigned long long)total));
    base = __shfl_sync(0xffffffffu, base, 31);
    uint32_t at = base + incl - c;
    uint32_t bits = word;
    while (bits) {
      const uint32_t b = __ffs(bits) - 1;
      bits &= bits - 1;
      q[at++] = uint32_t(w * 32 + b);
    }
  }
}

// ------------------------------------------------------------------- SSSP
template <typename W>
__global__ void __launch_bounds__(256) k_sssp_push(const uint32_t* __restrict__ q,
                                                   const uint32_t* __restrict__ dq, uint32_t nq,
                                                   const uint64_t* __restrict__ ptr,
                                                   const uint32_t* __restrict__ idx,
                                                   const W* __restrict__ wt, uint32_t* dist,
                                                   uint32_t* changed, uint32_t* qn,
                                                   unsigned long long* ctr) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long edges = 0;
  for (uint64_t i = warp; i < nq; i += nwarps) {
    const uint32_t u = q[i];
    const uint64_t du = dq[i];
    const uint64_t beg = ptr[u], end = ptr[u + 1];
    edges += end - beg;
    for (uint64_t base = beg; base < end; base += 32) {
      const uint64_t e = base + lane;
      bool won = false;
      uint32_t v = 0;
      if (e < end) {
        v = idx[e];
        const uint64_t cand64 = du + uint64_t(wt[e]);
        const uint32_t cand = cand64 >= 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(cand64);
        if (cand < dist[v]) {
          const uint32_t old = atomicMin(&dist[v], cand);
          if (cand < old) {
            const uint32_t bit = 1u << (v & 31u);
            won = !(atomicOr(&changed[v >> 5], bit) & bit);
          }
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, won);
      if (b) {
        uint32_t at = 0;
        if (lane == 0) at = uint32_t(atomicAdd(&ctr[0], (unsigned long long)__popc(b)));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (won) qn[at + __popc(b & ((1u << lane) - 1u))] = v;
      }
    }
  }
  if (lane == 0 && edges) atomicAdd(&ctr[2], edges);
}

__global__ void k_sssp_snapshot(const uint32_t* q, uint32_t nq, const uint32_t* dist, uint32_t* dq,
                                uint32_t* changed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x) {
    const uint32_t v = q[i];
    dq[i] = dist[v];
    changed[v >> 5] = 0u;  // reset for the next superstep (benign duplicate writes)
  }
}

__global__ void k_sssp_init(uint32_t* dist, uint64_t n, uint32_t root, uint32_t* q, uint32_t* dq) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dist[i] = i == root ? 0u : 0xFFFFFFFFu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q[0] = root;
    dq[0] = 0;
  }
}

uint32_t to_internal_id(Graph& g, uint64_t v) {
  if (!g.relabeled) return uint32_t(v);
  uint32_t h = 0;
  GM_CUDA(cudaMemcpy(&h, g.perm.get() + v, 4, cudaMemcpyDeviceToHost));
  return h;
}

template <typename T>
void write_out(Graph& g, const T* internal, T* out, bool out_on_device) {
  cudaStream_t s = g.stream;
  if (out_on_device) {
    to_external(g, internal, out, sizeof(T));
  } else {
    DevBuf<T> ext(g.n, s);
    to_external(g, internal, ext.get(), sizeof(T));
    GM_CUDA(cudaMemcpyAsync(out, ext.get(), g.n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

std::vector<gm_iteration_stats> bfs(Graph& g, uint64_t root, int64_t max_iters, int32_t* out,
                                    bool out_on_device, bool collect) {
  const uint64_t n = g.n;
  if (root >= n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(n));
  std::vector<gm_iteration_stats> stats;
  TravCache& c = cache(g);
  cudaStream_t s = g.stream;
  if (!c.level) c.level.alloc(n, s);
  ensure_forward(g);
  const Csr& fw = g.fwd();
  const uint64_t words = (n + 31) / 32;
  // Pull range: with a relabeled symmetric graph the vertices that can be
  // reached are exactly the prefix with nonzero degree.
  const uint64_t nv = (g.relabeled && g.symmetric) ? g.nonzero_outdeg : n;
  const uint32_t r = to_internal_id(g, root);
  k_bfs_init<<<grid_for(std::max<uint64_t>(n, words + 1), 256), 256, 0, s>>>(c.level.get(), c.vis.get(), n, r,
                                                                       c.q0.get());
  GM_LAUNCH_CHECK();
  uint32_t deg_root = 0;
  GM_CUDA(cudaMemcpyAsync(&deg_root, g.outdeg.get() + r, 4, cudaMemcpyDeviceToHost, s));
  HostPinned<unsigned long long> h(4);
  GM_CUDA(cudaStreamSynchronize(s));
  uint64_t nf = 1, mf = deg_root;
  bool frontier_is_queue = true;  // else: frontier in c.fb bitmap
  uint32_t* q = c.q0.get();
  uint32_t* qn = c.q1.get();
  cudaEvent_t e0, e1;
  GM_CUDA(cudaEventCreate(&e0));
  GM_CUDA(cudaEventCreate(&e1));
  for (int64_t it = 1; it <= max_iters; ++it) {
    const bool pull = double(mf) > kPullFraction * double(g.m) && nf > 0;
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 4 * 8, s));
    if (collect) GM_CUDA(cudaEventRecord(e0, s));
    if (pull) {
      if (frontier_is_queue) {
        c.fb.zero(s);
        k_queue_to_bitmap<<<grid_for(nf, 256), 256, 0, s>>>(q, uint32_t(nf), c.fb.get());
        GM_LAUNCH_CHECK();
      }
      k_bfs_pull<<<grid_for((nv + 31) / 32 * 32, 256), 256, 0, s>>>(
          nv, g.in.ptr.get(), g.in.idx.get(), c.fb.get(), c.vis.get(), c.nbm.get(),
          c.level.get(), int32_t(it), c.ctr.get());
      GM_LAUNCH_CHECK();
      // next frontier lives in nbm (words beyond nv stay zero: clear the tail)
      if (nv < n) {
        const uint64_t w0 = (nv + 31) / 32;
        if (w0 < words + 1)
          GM_CUDA(cudaMemsetAsync(c.nbm.get() + w0, 0, (words + 1 - w0) * 4, s));
      }
      c.fb.swap(c.nbm);
      frontier_is_queue = false;
    } else {
      if (!frontier_is_queue) {
        // compact bitmap frontier to a queue
        GM_CUDA(cudaMemsetAsync(c.ctr.get() + 3, 0, 8, s));
        k_bitmap_to_queue<<<grid_for(words + 32, 256), 256, 0, s>>>(c.fb.get(), words, q,
                                                                              c.ctr.get() + 3);
        GM_LAUNCH_CHECK();
      }
      if (nf)
        k_bfs_push<<<grid_for(nf * 32, 256), 256, 0, s>>>(q, uint32_t(nf), fw.ptr.get(), fw.idx.get(),
                                                          g.outdeg.get(), c.level.get(), c.vis.get(),
                                                          int32_t(it), qn, c.ctr.get());
      GM_LAUNCH_CHECK();
      std::swap(q, qn);
      frontier_is_queue = true;
    }
    if (collect) GM_CUDA(cudaEventRecord(e1, s));
    GM_CUDA(cudaMemcpyAsync(h.get(), c.ctr.get(), 3 * 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const uint64_t nn = h[0], mn = h[1];
    if (collect) {
      float ms = 0;
      GM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      gm_iteration_stats st{};
      st.iteration = it;
      st.active_before = int64_t(nf);
      st.messages_generated = int64_t(nf);
      st.vertices_updated = int64_t(nn);
      st.spmv_seconds = ms * 1e-3;
      st.total_seconds = ms * 1e-3;
      st.edges_processed = int64_t(pull ? h[2] : mf);
      st.bytes_algorithmic = pull ? int64_t(16 * nv + 4 * h[2] + 4 * nn + 2 * n / 8)
                                  : int64_t(16 * nf + 4 * mf + 4 * nn + 2 * n / 8);
      st.direction = pull ? 0 : 1;
      stats.push_back(st);
    }
    nf = nn;
    mf = mn;
    if (nn == 0) break;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (out) write_out(g, c.level.get(), out, out_on_device);
  return stats;
}

std::vector<gm_iteration_stats> sssp(Graph& g, uint64_t root, int64_t max_iters, uint32_t* out,
                                     bool out_on_device, bool collect) {
  const uint64_t n = g.n;
  if (root >= n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(n));
  if (g.value_type != GM_VAL_U8 && g.value_type != GM_VAL_U32)
    fail(GM_EUSAGE, std::string("sssp: needs u8 or u32 edge weights, graph stores ") +
                        value_name(g.value_type) + " (use GM_PROG_SSSP_REF for real weights)");
  std::vector<gm_iteration_stats> stats;
  TravCache& c = cache(g);
  cudaStream_t s = g.stream;
  if (!c.dist) {
    c.dist.alloc(n, s);
    c.d0.alloc(n + 1, s);
    c.d1.alloc(n + 1, s);
  }
  ensure_forward(g);
  const Csr& fw = g.fwd();
  const uint32_t r = to_internal_id(g, root);
  k_sssp_init<<<grid_for(n, 256), 256, 0, s>>>(c.dist.get(), n, r, c.q0.get(), c.d0.get());
  GM_LAUNCH_CHECK();
  c.nbm.zero(s);  // changed bitmap
  HostPinned<unsigned long long> h(4);
  uint32_t *q = c.q0.get(), *qn = c.q1.get(), *dq = c.d0.get(), *dqn = c.d1.get();
  uint64_t nf = 1;
  cudaEvent_t e0, e1;
  GM_CUDA(cudaEventCreate(&e0));
  GM_CUDA(cudaEventCreate(&e1));
  for (int64_t it = 1; it <= max_iters; ++it) {
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 4 * 8, s));
    if (collect) GM_CUDA(cudaEventRecord(e0, s));
    if (g.value_type == GM_VAL_U8)
      k_sssp_push<uint8_t><<<grid_for(nf * 32, 256), 256, 0, s>>>(
          q, dq, uint32_t(nf), fw.ptr.get(), fw.idx.get(), fw.val.get(), c.dist.get(), c.nbm.get(),
          qn, c.ctr.get());
    else
      k_sssp_push<uint32_t><<<grid_for(nf * 32, 256), 256, 0, s>>>(
          q, dq, uint32_t(nf), fw.ptr.get(), fw.idx.get(),
          reinterpret_cast<const uint32_t*>(fw.val.get()), c.dist.get(), c.nbm.get(), qn,
          c.ctr.get());
    GM_LAUNCH_CHECK();
    if (collect) GM_CUDA(cudaEventRecord(e1, s));
    GM_CUDA(cudaMemcpyAsync(h.get(), c.ctr.get(), 3 * 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const uint64_t nn = h[0];
    if (nn) {
      k_sssp_snapshot<<<grid_for(nn, 256), 256, 0, s>>>(qn, uint32_t(nn), c.dist.get(), dqn,
                                                        c.nbm.get());
      GM_LAUNCH_CHECK();
    }
    if (collect) {
      float ms = 0;
      GM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      gm_iteration_stats st{};
      st.iteration = it;
      st.active_before = int64_t(nf);
      st.messages_generated = int64_t(nf);
      st.vertices_updated = int64_t(nn);
      st.spmv_seconds = ms * 1e-3;
      st.total_seconds = ms * 1e-3;
      st.edges_processed = int64_t(h[2]);
      st.bytes_algorithmic = int64_t(20 * nf + 5 * h[2] + 4 * nn + 2 * n / 8);
      st.direction = 1;
      stats.push_back(st);
    }
    std::swap(q, qn);
    std::swap(dq, dqn);
    nf = nn;
    if (nn == 0) break;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (out) write_out(g, c.dist.get(), out, out_on_device);
  return stats;
}

}  // namespace gm
