// traversal.cu -- BFS and SSSP supersteps: push SpMSpV / pull SpMV with a
// direction switch, bitmap frontiers, exact bulk-synchronous semantics.
//
// Reference: BfsProgram / SsspProgram (include/semigraph/algorithms/traversal.hpp:39-91)
// run by run_distance_program (:95-115) through Engine::run_graph_program
// (include/semigraph/engine.hpp:193-213).  The reference scans every stored
// column of every partition each superstep (engine.hpp:234-236); here a
// superstep touches only the frontier's edges (push) or only unvisited
// vertices (pull).
//
// BFS (min over level+1): levels and per-superstep stats (active_before =
// messages_generated = |frontier|, vertices_updated = |next frontier|) equal the
// reference's exactly, because a vertex's level is written once, in the
// superstep that first reaches it, whichever direction runs.
//   push (SpMSpV over CSR(G)): edge-balanced.  The frontier queue carries each
//        vertex's degree; an exclusive scan gives edge offsets and every thread
//        expands kEPT consecutive frontier edges (one binary search per thread),
//        so a single hub and a million leaves cost the same per edge.  A vertex
//        is claimed once through the visited bitmap (atomicOr) and appended to
//        the next queue with a warp-aggregated atomic.
//   pull (SpMV over CSR(G^T), unvisited rows only): with GM_RELABEL the ids are
//        sorted by degree, so rows [0, hub_end) (degree >= 32) are probed a warp
//        at a time (32 neighbours per ballot) and the rest a thread per row;
//        adjacency is hub-first, so the first frontier neighbour comes early.
//   switch: push -> pull when frontier edges > 5% of m (BASELINE configs[1]);
//        pull -> push when the frontier falls below n/24 (Beamer et al.).
// SSSP (min over dist+w, uint32, UINT32_MAX = unreached): the same edge-balanced
// push, carrying the frontier's superstep-start distances in the queue (the
// message snapshot, rule S3); atomicMin into dist; a vertex whose distance
// dropped is claimed once through a changed-bitmap and forms the next frontier.
#include <cub/device/device_scan.cuh>

#include <vector>

#include "api_internal.cuh"

namespace gm {

struct TravCache {
  uint64_t n = 0;
  DevBuf<int32_t> level;
  DevBuf<uint32_t> dist;
  DevBuf<uint32_t> q0, q1;        // frontier queues (internal ids)
  DevBuf<uint32_t> g0, g1;        // degree of each queued vertex (scan input)
  DevBuf<uint32_t> d0, d1;        // SSSP message snapshots parallel to the queues
  DevBuf<uint64_t> offs;          // exclusive scan of queued degrees (n + 1)
  DevBuf<uint8_t> scan_tmp;
  size_t scan_tmp_bytes = 0;
  DevBuf<uint32_t> vis, fb, nbm;  // visited / frontier / next-frontier bitmaps
  DevBuf<unsigned long long> ctr; // [0] next count [1] next edges [2] examined [3] scratch
  DevBuf<int32_t> ext_out;        // caller-order staging for host outputs
  std::unique_ptr<HostPinned<unsigned long long>> h;
  uint64_t hub_end = 0;           // rows [0, hub_end) have degree >= 32 (relabeled, symmetric)
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~TravCache() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

namespace {

constexpr double kPullFraction = 0.05;
constexpr uint64_t kBeta = 24;
constexpr int kEPT = 4;  // edges per thread in the edge-balanced push

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
    c.g0.alloc(n + 1, s);
    c.g1.alloc(n + 1, s);
    c.offs.alloc(n + 2, s);
    c.vis.alloc(words, s);
    c.fb.alloc(words, s);
    c.nbm.alloc(words, s);
    c.ctr.alloc(8, s);
    c.ctr.zero(s);
    c.h = std::make_unique<HostPinned<unsigned long long>>(8);
    GM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, c.scan_tmp_bytes, (const uint32_t*)nullptr,
                                          (uint64_t*)nullptr, int64_t(n + 1), s));
    c.scan_tmp.alloc(c.scan_tmp_bytes + 16, s);
    GM_CUDA(cudaEventCreate(&c.e0));
    GM_CUDA(cudaEventCreate(&c.e1));
    // hub_end: first internal id with degree < 32 (degrees sorted descending).
    if (g.relabeled && g.symmetric && n) {
      std::vector<uint32_t> deg(n);
      GM_CUDA(cudaMemcpyAsync(deg.data(), g.outdeg.get(), n * 4, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
      uint64_t lo = 0, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (deg[mid] >= 32)
          lo = mid + 1;
        else
          hi = mid;
      }
      c.hub_end = lo;
    }
    GM_CUDA(cudaStreamSynchronize(s));
  }
  return *g.trav;
}

// Frontier-degree scan: offs[i] = sum of deg of queue entries before i; offs[nq]
// = total frontier edges (read by the expansion kernel on device).
void scan_degrees(TravCache& c, const uint32_t* qdeg, uint64_t nq, cudaStream_t s) {
  size_t bytes = c.scan_tmp_bytes;
  GM_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.get(), bytes, qdeg, c.offs.get(),
                                        int64_t(nq + 1), s));
}

// Binary search: last i in [0, nq) with offs[i] <= t.
__device__ __forceinline__ uint32_t find_source(const uint64_t* offs, uint32_t nq, uint64_t t) {
  uint32_t lo = 0, hi = nq;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (offs[mid] <= t)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// ------------------------------------------------------------------- BFS
__global__ void k_bfs_init(uint32_t* vis, uint64_t words, uint64_t root_ext, const uint32_t* perm,
                           uint32_t* queue, uint32_t* qdeg, const uint32_t* deg, int32_t* level) {
  const uint32_t root = perm ? perm[root_ext] : uint32_t(root_ext);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x)
    vis[i] = (i == (root >> 5)) ? (1u << (root & 31u)) : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    queue[0] = root;
    qdeg[0] = deg[root];
    qdeg[1] = 0;
    level[root] = 0;
  }
}

// Edge-balanced push.  Each lane owns kEPT consecutive frontier edges.
__global__ void __launch_bounds__(256) k_bfs_push(const uint32_t* __restrict__ q,
                                                  const uint64_t* __restrict__ offs, uint32_t nq,
                                                  const uint64_t* __restrict__ ptr,
                                                  const uint32_t* __restrict__ idx,
                                                  const uint32_t* __restrict__ deg, int32_t* level,
                                                  uint32_t* vis, int32_t next_level, uint32_t* qn,
                                                  uint32_t* qdeg_n, unsigned long long* ctr) {
  const uint64_t total = offs[nq];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long my_edges = 0;
  for (uint64_t wb = warp * 32 * kEPT; wb < total; wb += nwarps * 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    uint32_t i = 0, u = 0;
    uint64_t e = 0, rem = 0;
    if (t0 < total) {
      i = find_source(offs, nq, t0);
      u = q[i];
      e = ptr[u] + (t0 - offs[i]);
      rem = offs[i + 1] - t0;
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      const uint64_t t = t0 + k;
      bool won = false;
      uint32_t v = 0;
      if (t < total) {
        while (rem == 0) {  // next queue entry with edges
          ++i;
          u = q[i];
          e = ptr[u];
          rem = offs[i + 1] - offs[i];
        }
        v = idx[e];
        ++e;
        --rem;
        const uint32_t bit = 1u << (v & 31u);
        if (!(vis[v >> 5] & bit)) won = !(atomicOr(&vis[v >> 5], bit) & bit);
      }
      const unsigned b = __ballot_sync(0xffffffffu, won);
      if (b) {
        uint32_t at = 0;
        if (lane == 0) at = uint32_t(atomicAdd(&ctr[0], (unsigned long long)__popc(b)));
        at = __shfl_sync(0xffffffffu, at, 0) + __popc(b & ((1u << lane) - 1u));
        if (won) {
          const uint32_t dv = deg[v];
          level[v] = next_level;
          qn[at] = v;
          qdeg_n[at] = dv;
          my_edges += dv;
        }
      }
    }
  }
  warp_add_u64(&ctr[1], my_edges);
}

// Frontier-bitmap probe: the hot prefix [0, 32*s_words) lives in shared memory
// (with GM_RELABEL the low ids are the hubs every adjacency list starts with).
__device__ __forceinline__ bool fb_probe(const uint32_t* s_fb, uint32_t s_words,
                                         const uint32_t* __restrict__ fb, uint32_t u) {
  const uint32_t w = u >> 5;
  const uint32_t word = w < s_words ? s_fb[w] : __ldg(&fb[w]);
  return (word >> (u & 31u)) & 1u;
}

constexpr int kPullProbes = 8;        // pass 1 probes at most this many in-neighbours
constexpr uint32_t kSmemFbWords = 24 * 1024;  // 96 KB of frontier bitmap per CTA

// Pull pass 1: thread per unvisited row, at most kPullProbes probes (loads
// issued 4 at a time); rows still unresolved with more in-edges are deferred
// (queue + remaining-degree) to the edge-balanced pass 2.
__global__ void __launch_bounds__(1024, 2) k_bfs_pull1(
    uint64_t nv, const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ fb, uint32_t s_words, uint32_t* vis, uint32_t* nbm,
    int32_t* level, int32_t next_level, const uint32_t* __restrict__ outdeg, uint32_t* defq,
    uint32_t* defdeg, unsigned long long* ctr) {
  extern __shared__ uint32_t s_fb[];
  for (uint32_t i = threadIdx.x; i < s_words; i += blockDim.x) s_fb[i] = fb[i];
  __syncthreads();
  const uint64_t words = (nv + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint32_t vw = vis[w];
    const uint64_t v = w * 32 + lane;
    bool found = false, defer = false;
    uint32_t rest = 0;
    if (v < nv && !((vw >> lane) & 1u)) {
      const uint64_t beg = ptr[v], end = ptr[v + 1];
      const uint64_t d = end - beg;
      const uint32_t lim = d < kPullProbes ? uint32_t(d) : kPullProbes;
      for (uint32_t p = 0; p < lim && !found; p += 4) {
        uint32_t u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = p + k < lim ? __ldg(&idx[beg + p + k]) : 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!found && u[k] != 0xFFFFFFFFu) {
            ++examined;
            found = fb_probe(s_fb, s_words, fb, u[k]);
          }
        }
      }
      if (found) {
        level[v] = next_level;
        found_e += outdeg[v];
      } else if (d > kPullProbes) {
        defer = true;
        rest = uint32_t(d - kPullProbes);
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, found);
    const unsigned db = __ballot_sync(0xffffffffu, defer);
    if (lane == 0) {
      nbm[w] = b;
      if (b) vis[w] = vw | b;
    }
    if (db) {
      uint32_t at = 0;
      if (lane == 0) at = uint32_t(atomicAdd(&ctr[4], (unsigned long long)__popc(db)));
      at = __shfl_sync(0xffffffffu, at, 0) + __popc(db & ((1u << lane) - 1u));
      if (defer) {
        defq[at] = uint32_t(v);
        defdeg[at] = rest;
      }
    }
    found_n += found;
  }
  warp_add_u64(&ctr[0], found_n);
  warp_add_u64(&ctr[1], found_e);
  warp_add_u64(&ctr[2], examined);
}

// Pull pass 2: edge-balanced over the deferred rows' remaining in-edges; a row
// is claimed once through its next-frontier bit.
__global__ void __launch_bounds__(1024, 2) k_bfs_pull2(
    const uint32_t* __restrict__ defq, const uint64_t* __restrict__ offs, uint32_t ndef,
    const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ fb, uint32_t s_words, uint32_t* vis, uint32_t* nbm,
    int32_t* level, int32_t next_level, const uint32_t* __restrict__ outdeg,
    unsigned long long* ctr) {
  extern __shared__ uint32_t s_fb[];
  for (uint32_t i = threadIdx.x; i < s_words; i += blockDim.x) s_fb[i] = fb[i];
  __syncthreads();
  const uint64_t total = offs[ndef];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t wb = warp * 32 * kEPT; wb < total; wb += nwarps * 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    if (t0 >= total) continue;
    uint32_t i = find_source(offs, ndef, t0);
    uint32_t v = defq[i];
    uint64_t e = ptr[v] + kPullProbes + (t0 - offs[i]);
    uint64_t rem = offs[i + 1] - t0;
    for (int k = 0; k < kEPT && t0 + k < total; ++k) {
      while (rem == 0) {
        ++i;
        v = defq[i];
        e = ptr[v] + kPullProbes;
        rem = offs[i + 1] - offs[i];
      }
      const uint32_t bit = 1u << (v & 31u);
      if (!(nbm[v >> 5] & bit)) {
        ++examined;
        if (fb_probe(s_fb, s_words, fb, __ldg(&idx[e])) && !(atomicOr(&nbm[v >> 5], bit) & bit)) {
          level[v] = next_level;
          atomicOr(&vis[v >> 5], bit);
          ++found_n;
          found_e += outdeg[v];
        }
      }
      ++e;
      --rem;
    }
  }
  warp_add_u64(&ctr[0], found_n);
  warp_add_u64(&ctr[1], found_e);
  warp_add_u64(&ctr[2], examined);
}

// Pull, warp per hub row [0, hub_end): 32 in-neighbours per probe.
__global__ void __launch_bounds__(256) k_bfs_pull_hubs(uint64_t hub_end,
                                                       const uint64_t* __restrict__ ptr,
                                                       const uint32_t* __restrict__ idx,
                                                       const uint32_t* __restrict__ fb, uint32_t* vis,
                                                       uint32_t* nbm, int32_t* level,
                                                       int32_t next_level, unsigned long long* ctr) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t v = warp; v < hub_end; v += nwarps) {
    const uint32_t bit = 1u << (v & 31u);
    if (vis[v >> 5] & bit) continue;
    const uint64_t beg = ptr[v], end = ptr[v + 1];
    bool found = false;
    for (uint64_t base = beg; base < end && !found; base += 32) {
      const uint64_t e = base + lane;
      const bool hit = e < end && bit_test(fb, idx[e]);
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      examined += (lane == 0) ? (b ? uint64_t(__ffs(b)) : (end - base < 32 ? end - base : 32)) : 0;
      found = b != 0;
    }
    if (found && lane == 0) {
      level[v] = next_level;
      atomicOr(&vis[v >> 5], bit);
      atomicOr(&nbm[v >> 5], bit);
      ++found_n;
      found_e += end - beg;
    }
  }
  warp_add_u64(&ctr[0], found_n);
  warp_add_u64(&ctr[1], found_e);
  warp_add_u64(&ctr[2], examined);
}

// Pull, thread per row in [lo, nv); rows come in whole 32-row words.
__global__ void __launch_bounds__(256) k_bfs_pull(uint64_t w_lo, uint64_t nv,
                                                  const uint64_t* __restrict__ ptr,
                                                  const uint32_t* __restrict__ idx,
                                                  const uint32_t* __restrict__ fb, uint32_t* vis,
                                                  uint32_t* nbm, int32_t* level,
                                                  int32_t next_level, unsigned long long* ctr) {
  const uint64_t words = (nv + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t w = w_lo + warp; w < words; w += nwarps) {
    const uint32_t vw = vis[w];
    const uint64_t v = w * 32 + lane;
    bool found = false;
    if (v < nv && !((vw >> lane) & 1u)) {
      const uint64_t beg = ptr[v], end = ptr[v + 1];
      for (uint64_t e = beg; e < end; ++e) {
        ++examined;
        if (bit_test(fb, __ldg(&idx[e]))) {
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
      nbm[w] = b;  // this word holds no hub rows: plain store
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

// Bitmap -> queue (+ degrees), warp-aggregated; queue order is irrelevant to the results.
__global__ void k_bitmap_to_queue(const uint32_t* bm, uint64_t words, const uint32_t* deg,
                                  uint32_t* q, uint32_t* qdeg, unsigned long long* cnt) {
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
      const uint32_t v = uint32_t(w * 32 + b);
      q[at] = v;
      qdeg[at] = deg[v];
      ++at;
    }
  }
}

// Caller-order output: out[v] = visited(p) ? level[p] : -1, p = perm[v].
__global__ void k_bfs_output(uint64_t n, const uint32_t* perm, const uint32_t* vis,
                             const int32_t* level, int32_t* out) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = perm ? perm[v] : uint32_t(v);
    out[v] = bit_test(vis, p) ? level[p] : -1;
  }
}

// ------------------------------------------------------------------- SSSP
template <typename W>
__global__ void __launch_bounds__(256) k_sssp_push(const uint32_t* __restrict__ q,
                                                   const uint32_t* __restrict__ dq,
                                                   const uint64_t* __restrict__ offs, uint32_t nq,
                                                   const uint64_t* __restrict__ ptr,
                                                   const uint32_t* __restrict__ idx,
                                                   const W* __restrict__ wt,
                                                   const uint32_t* __restrict__ deg, uint32_t* dist,
                                                   uint32_t* changed, uint32_t* qn,
                                                   uint32_t* qdeg_n, unsigned long long* ctr) {
  const uint64_t total = offs[nq];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t wb = warp * 32 * kEPT; wb < total; wb += nwarps * 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    uint32_t i = 0, u = 0;
    uint64_t e = 0, rem = 0, du = 0;
    if (t0 < total) {
      i = find_source(offs, nq, t0);
      u = q[i];
      du = dq[i];
      e = ptr[u] + (t0 - offs[i]);
      rem = offs[i + 1] - t0;
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      const uint64_t t = t0 + k;
      bool won = false;
      uint32_t v = 0;
      if (t < total) {
        while (rem == 0) {
          ++i;
          u = q[i];
          du = dq[i];
          e = ptr[u];
          rem = offs[i + 1] - offs[i];
        }
        v = idx[e];
        const uint64_t c64 = du + uint64_t(wt[e]);
        ++e;
        --rem;
        const uint32_t cand = c64 >= 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(c64);
        if (cand < dist[v] && cand < atomicMin(&dist[v], cand)) {
          const uint32_t bit = 1u << (v & 31u);
          won = !(atomicOr(&changed[v >> 5], bit) & bit);
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, won);
      if (b) {
        uint32_t at = 0;
        if (lane == 0) at = uint32_t(atomicAdd(&ctr[0], (unsigned long long)__popc(b)));
        at = __shfl_sync(0xffffffffu, at, 0) + __popc(b & ((1u << lane) - 1u));
        if (won) {
          qn[at] = v;
          qdeg_n[at] = deg[v];
        }
      }
    }
  }
}

// Next frontier's message snapshot; resets its changed-bits for the next superstep.
__global__ void k_sssp_snapshot(const uint32_t* q, uint32_t nq, const uint32_t* dist, uint32_t* dq,
                                uint32_t* changed, unsigned long long* edges,
                                const uint32_t* qdeg) {
  unsigned long long m = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x) {
    const uint32_t v = q[i];
    dq[i] = dist[v];
    changed[v >> 5] = 0u;
    m += qdeg[i];
  }
  warp_add_u64(edges, m);
}

__global__ void k_sssp_init(uint32_t* dist, uint64_t n, uint64_t root_ext, const uint32_t* perm,
                            uint32_t* q, uint32_t* dq, uint32_t* qdeg, const uint32_t* deg) {
  const uint32_t root = perm ? perm[root_ext] : uint32_t(root_ext);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dist[i] = i == root ? 0u : 0xFFFFFFFFu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q[0] = root;
    dq[0] = 0;
    qdeg[0] = deg[root];
    qdeg[1] = 0;
  }
}

template <typename T>
__global__ void k_gather_out(uint64_t n, const uint32_t* perm, const T* in, T* out) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    out[v] = in[perm ? perm[v] : v];
}

unsigned push_grid(uint64_t edges) {
  const uint64_t threads = (edges + kEPT - 1) / kEPT;
  return grid_for(threads, 256, 148 * 8);
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
  if (!c.level) {
    c.level.alloc(n, s);
    GM_CUDA(cudaFuncSetAttribute(k_bfs_pull1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kSmemFbWords * 4)));
    GM_CUDA(cudaFuncSetAttribute(k_bfs_pull2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kSmemFbWords * 4)));
  }
  ensure_forward(g);
  const Csr& fw = g.fwd();
  const uint64_t words = (n + 31) / 32;
  // Pull rows: with a relabeled symmetric graph only the nonzero-degree prefix
  // can ever be reached.
  const uint64_t nv = (g.relabeled && g.symmetric) ? g.nonzero_outdeg : n;
  // Hub rows (warp per row) are [0, hub_end) rounded up to whole bitmap words;
  // the thread-per-row pass owns every later word exclusively.
  const uint64_t hub_words = (c.hub_end + 31) / 32;
  const uint64_t hub_end = std::min<uint64_t>(nv, hub_words * 32);
  const uint32_t* perm = g.relabeled ? g.perm.get() : nullptr;
  k_bfs_init<<<grid_for(words + 1, 256), 256, 0, s>>>(c.vis.get(), words + 1, root, perm,
                                                      c.q0.get(), c.g0.get(), g.outdeg.get(),
                                                      c.level.get());
  GM_LAUNCH_CHECK();
  uint64_t nf = 1, mf = 0;
  bool frontier_is_queue = true, prev_pull = false;
  uint32_t *q = c.q0.get(), *qn = c.q1.get(), *qd = c.g0.get(), *qdn = c.g1.get();
  unsigned long long* h = c.h->get();
  for (int64_t it = 1; it <= max_iters; ++it) {
    bool pull = prev_pull ? (nf * kBeta >= n) : (double(mf) > kPullFraction * double(g.m));
    if (it == 1) pull = false;
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 4 * 8, s));
    if (collect) GM_CUDA(cudaEventRecord(c.e0, s));
    if (pull) {
      if (frontier_is_queue) {
        c.fb.zero(s);
        k_queue_to_bitmap<<<grid_for(nf, 256), 256, 0, s>>>(q, uint32_t(nf), c.fb.get());
        GM_LAUNCH_CHECK();
      }
      c.nbm.zero(s);
      const uint32_t s_words = uint32_t(std::min<uint64_t>(kSmemFbWords, (nv + 31) / 32));
      const size_t smem = size_t(s_words) * 4;
      k_bfs_pull1<<<148 * 2, 1024, smem, s>>>(nv, g.in.ptr.get(), g.in.idx.get(), c.fb.get(),
                                              s_words, c.vis.get(), c.nbm.get(), c.level.get(),
                                              int32_t(it), g.outdeg.get(), qn, qdn, c.ctr.get());
      GM_LAUNCH_CHECK();
      GM_CUDA(cudaMemcpyAsync(h + 4, c.ctr.get() + 4, 8, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
      const uint64_t ndef = h[4];
      if (ndef) {
        GM_CUDA(cudaMemsetAsync(qdn + ndef, 0, 4, s));
        scan_degrees(c, qdn, ndef, s);
        k_bfs_pull2<<<148 * 2, 1024, smem, s>>>(qn, c.offs.get(), uint32_t(ndef), g.in.ptr.get(),
                                                g.in.idx.get(), c.fb.get(), s_words, c.vis.get(),
                                                c.nbm.get(), c.level.get(), int32_t(it),
                                                g.outdeg.get(), c.ctr.get());
        GM_LAUNCH_CHECK();
      }
      (void)hub_end;
      c.fb.swap(c.nbm);
      frontier_is_queue = false;
    } else {
      if (!frontier_is_queue) {
        k_bitmap_to_queue<<<grid_for(words + 32, 256), 256, 0, s>>>(c.fb.get(), words, g.outdeg.get(),
                                                                    q, qd, c.ctr.get() + 3);
        GM_LAUNCH_CHECK();
      }
      GM_CUDA(cudaMemsetAsync(qd + nf, 0, 4, s));
      scan_degrees(c, qd, nf, s);
      k_bfs_push<<<push_grid(it == 1 ? 65536 : mf), 256, 0, s>>>(
          q, c.offs.get(), uint32_t(nf), fw.ptr.get(), fw.idx.get(), g.outdeg.get(), c.level.get(),
          c.vis.get(), int32_t(it), qn, qdn, c.ctr.get());
      GM_LAUNCH_CHECK();
      std::swap(q, qn);
      std::swap(qd, qdn);
      frontier_is_queue = true;
    }
    if (collect) GM_CUDA(cudaEventRecord(c.e1, s));
    GM_CUDA(cudaMemcpyAsync(h, c.ctr.get(), 3 * 8, cudaMemcpyDeviceToHost, s));
    if (!pull) GM_CUDA(cudaMemcpyAsync(h + 3, c.offs.get() + nf, 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const uint64_t nn = h[0], mn = h[1], examined = h[2];
    if (!pull) mf = h[3];  // exact frontier edges (the first superstep only had a hint)
    if (collect) {
      float ms = 0;
      GM_CUDA(cudaEventElapsedTime(&ms, c.e0, c.e1));
      gm_iteration_stats st{};
      st.iteration = it;
      st.active_before = int64_t(nf);
      st.messages_generated = int64_t(nf);
      st.vertices_updated = int64_t(nn);
      st.spmv_seconds = ms * 1e-3;
      st.total_seconds = ms * 1e-3;
      st.edges_processed = int64_t(pull ? examined : mf);
      // pull: ptr + vis per candidate row, examined col ids, level + bitmap writes
      // push: queue + offsets + ptr per frontier vertex, col id per edge, queue writes
      st.bytes_algorithmic = pull ? int64_t(16 * nv + 4 * examined + 4 * nn + 2 * n / 8)
                                  : int64_t(16 * nf + 4 * mf + 8 * nn + n / 8);
      st.direction = pull ? 0 : 1;
      stats.push_back(st);
    }
    nf = nn;
    mf = mn;
    prev_pull = pull;
    if (nn == 0) break;
  }
  if (out) {
    int32_t* dst = out;
    if (!out_on_device) {
      if (!c.ext_out) c.ext_out.alloc(n, s);
      dst = c.ext_out.get();
    }
    k_bfs_output<<<grid_for(n, 256), 256, 0, s>>>(n, perm, c.vis.get(), c.level.get(), dst);
    GM_LAUNCH_CHECK();
    if (!out_on_device) GM_CUDA(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
  }
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
  const uint32_t* perm = g.relabeled ? g.perm.get() : nullptr;
  k_sssp_init<<<grid_for(n, 256), 256, 0, s>>>(c.dist.get(), n, root, perm, c.q0.get(), c.d0.get(),
                                               c.g0.get(), g.outdeg.get());
  GM_LAUNCH_CHECK();
  c.nbm.zero(s);  // changed bitmap
  unsigned long long* h = c.h->get();
  uint32_t *q = c.q0.get(), *qn = c.q1.get(), *dq = c.d0.get(), *dqn = c.d1.get();
  uint32_t *qd = c.g0.get(), *qdn = c.g1.get();
  uint64_t nf = 1, mf = 65536;  // grid hint only for the first superstep
  for (int64_t it = 1; it <= max_iters; ++it) {
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 4 * 8, s));
    if (collect) GM_CUDA(cudaEventRecord(c.e0, s));
    GM_CUDA(cudaMemsetAsync(qd + nf, 0, 4, s));
    scan_degrees(c, qd, nf, s);
    if (g.value_type == GM_VAL_U8)
      k_sssp_push<uint8_t><<<push_grid(mf), 256, 0, s>>>(
          q, dq, c.offs.get(), uint32_t(nf), fw.ptr.get(), fw.idx.get(), fw.val.get(),
          g.outdeg.get(), c.dist.get(), c.nbm.get(), qn, qdn, c.ctr.get());
    else
      k_sssp_push<uint32_t><<<push_grid(mf), 256, 0, s>>>(
          q, dq, c.offs.get(), uint32_t(nf), fw.ptr.get(), fw.idx.get(),
          reinterpret_cast<const uint32_t*>(fw.val.get()), g.outdeg.get(), c.dist.get(),
          c.nbm.get(), qn, qdn, c.ctr.get());
    GM_LAUNCH_CHECK();
    if (collect) GM_CUDA(cudaEventRecord(c.e1, s));
    GM_CUDA(cudaMemcpyAsync(h, c.ctr.get(), 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaMemcpyAsync(h + 3, c.offs.get() + nf, 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const uint64_t nn = h[0];
    mf = h[3];  // exact edges of this frontier
    if (nn) {
      k_sssp_snapshot<<<grid_for(nn, 256), 256, 0, s>>>(qn, uint32_t(nn), c.dist.get(), dqn,
                                                        c.nbm.get(), c.ctr.get() + 1, qdn);
      GM_LAUNCH_CHECK();
      GM_CUDA(cudaMemcpyAsync(h + 1, c.ctr.get() + 1, 8, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
    }
    const uint64_t mn = nn ? h[1] : 0;
    if (collect) {
      float ms = 0;
      GM_CUDA(cudaEventElapsedTime(&ms, c.e0, c.e1));
      gm_iteration_stats st{};
      st.iteration = it;
      st.active_before = int64_t(nf);
      st.messages_generated = int64_t(nf);
      st.vertices_updated = int64_t(nn);
      st.spmv_seconds = ms * 1e-3;
      st.total_seconds = ms * 1e-3;
      st.edges_processed = int64_t(mf);
      st.bytes_algorithmic = int64_t(24 * nf + 5 * mf + 8 * nn + n / 8);
      st.direction = 1;
      stats.push_back(st);
    }
    std::swap(q, qn);
    std::swap(dq, dqn);
    std::swap(qd, qdn);
    nf = nn;
    mf = mn;
    if (nn == 0) break;
  }
  if (out) {
    uint32_t* dst = out;
    if (!out_on_device) {
      if (!c.ext_out) c.ext_out.alloc(n, s);
      dst = reinterpret_cast<uint32_t*>(c.ext_out.get());
    }
    k_gather_out<uint32_t><<<grid_for(n, 256), 256, 0, s>>>(n, perm, c.dist.get(), dst);
    GM_LAUNCH_CHECK();
    if (!out_on_device) GM_CUDA(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
  }
  return stats;
}

}  // namespace gm
