// traversal.cu -- BFS and SSSP supersteps: push SpMSpV / pull SpMV with a
// direction switch, bitmap frontiers, exact bulk-synchronous semantics.
//
// Reference: BfsProgram / SsspProgram (include/semigraph/algorithms/traversal.hpp:39-91)
// run by run_distance_program (:95-115) through Engine::run_graph_program
// (include/semigraph/engine.hpp:193-213).  The reference scans every stored
// column of every partition each superstep (engine.hpp:234-236); here a
// superstep touches only the frontier's edges (push) or only unvisited rows
// (pull), and the whole superstep loop runs on the device: the host enqueues
// supersteps in batches and reads one flag per batch.
//
// BFS (min over level+1): levels and per-superstep stats (active_before =
// messages_generated = |frontier|, vertices_updated = |next frontier|) equal the
// reference's exactly, because a vertex's level is written once, in the
// superstep that first reaches it, whichever direction runs.
//   frontier: a queue whose entries carry exclusive edge offsets (queue order
//        = offset order) plus a bitmap.  Both are produced at enqueue time: a
//        warp reserves its slots and its edge range with ONE 64-bit atomicAdd
//        on a packed (count << 36 | edges) counter, so no scan pass is needed.
//   push (SpMSpV over CSR(G)): edge-balanced; each thread expands kEPT
//        consecutive frontier edges found by one binary search over the
//        offsets, so one hub and a million leaves cost the same per edge.
//        A vertex is claimed once through the visited bitmap (atomicOr).
//   pull (SpMV over CSR(G^T), unvisited rows only): pass 1 probes at most
//        kPullProbes in-neighbours per row (thread per row); rows still open
//        are deferred to pass 2, edge-balanced over their remaining in-edges.
//        The hot prefix of the frontier bitmap is staged in shared memory
//        (with GM_RELABEL low ids are the hubs every adjacency list starts
//        with, so most probes hit it).
//   switch (decided on device): push -> pull when frontier edges > 5% of m
//        (BASELINE configs[1]); pull -> push when the frontier drops below n/24
//        (Beamer et al.).
// SSSP (min over dist+w, uint32, UINT32_MAX = unreached): the same edge-
// balanced push, carrying the frontier's superstep-start distances (the
// message snapshot, rule S3); atomicMin into dist; a vertex whose distance
// dropped is claimed once through a changed-bitmap and forms the next frontier.
#include <vector>

#include "api_internal.cuh"

namespace gm {

namespace {

constexpr int kMaxRecorded = 4096;  // per-superstep records kept on device
constexpr int kBatch = 4;           // supersteps enqueued per host check
constexpr int kEPT = 4;             // edges per thread, edge-balanced passes
constexpr int kPullProbes = 8;      // pull pass 1 probes at most this many in-neighbours
constexpr uint32_t kSmemFbWords = 24 * 1024;  // 96 KB of frontier bitmap per CTA
constexpr unsigned kGrid = 148 * 2;           // persistent grid (2 CTAs of 1024 per SM)
constexpr unsigned kThreads = 1024;
constexpr int kCountShift = 36;  // packed counter: count << 36 | edges
constexpr unsigned long long kEdgeMask = (1ull << kCountShift) - 1;

enum Dir : int32_t { kPush = 1, kPull = 0 };

struct StepRec {
  int64_t active, updated, edges, examined;
  int32_t dir, pad;
};

// Device-resident superstep state.
struct Ctl {
  unsigned long long qpack;     // next queue (count << 36 | edges)
  unsigned long long dpack;     // deferred rows (count << 36 | remaining edges)
  unsigned long long found_n, found_e, examined;
  unsigned long long nf, mf;    // current frontier: vertices, edges
  int32_t it, dir, prev_pull, cur_is_queue, done, max_it;
  uint64_t n_total, m_total, nv;
  StepRec rec[kMaxRecorded];
};

}  // namespace

struct TravCache {
  uint64_t n = 0;
  DevBuf<int32_t> level;
  DevBuf<uint32_t> dist;
  DevBuf<uint32_t> q[2];        // frontier queues (internal ids)
  DevBuf<uint64_t> offs[2];     // exclusive edge offsets, parallel to q (+1 total)
  DevBuf<uint32_t> dq[2];       // SSSP message snapshots parallel to q
  DevBuf<uint32_t> defq;        // pull: deferred rows
  DevBuf<uint64_t> defo;        // pull: their exclusive remaining-edge offsets
  DevBuf<uint32_t> vis, fb[2];  // visited / frontier bitmaps (cur = it & 1)
  DevBuf<uint32_t> changed;     // SSSP changed-bitmap
  DevBuf<Ctl> ctl;
  DevBuf<int32_t> ext_out;      // caller-order staging for host outputs
  std::unique_ptr<HostPinned<int32_t>> hdone;
  std::vector<cudaEvent_t> ev;  // 2 per recorded superstep
  bool attrs = false;
  ~TravCache() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

namespace {

TravCache& cache(Graph& g) {
  if (!g.trav) {
    g.trav = std::unique_ptr<TravCache, void (*)(TravCache*)>(new TravCache(),
                                                              [](TravCache* p) { delete p; });
    TravCache& c = *g.trav;
    cudaStream_t s = g.stream;
    const uint64_t n = g.n, words = (n + 31) / 32 + 1;
    c.n = n;
    for (int i = 0; i < 2; ++i) {
      c.q[i].alloc(n + 1, s);
      c.offs[i].alloc(n + 2, s);
      c.fb[i].alloc(words, s);
    }
    c.defq.alloc(n + 1, s);
    c.defo.alloc(n + 2, s);
    c.vis.alloc(words, s);
    c.ctl.alloc(1, s);
    c.ctl.zero(s);
    c.hdone = std::make_unique<HostPinned<int32_t>>(4);
    GM_CUDA(cudaStreamSynchronize(s));
  }
  return *g.trav;
}

__device__ __forceinline__ uint32_t find_source(const uint64_t* offs, uint32_t nq, uint64_t t) {
  uint32_t lo = 0, hi = nq;  // last i in [0, nq) with offs[i] <= t
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (offs[mid] <= t)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Warp-aggregated append of (v, its edge count) to a queue with packed
// (count, edges) reservation; writes q[pos] = v, offs[pos] = edge offset.
__device__ __forceinline__ void warp_enqueue(bool want, uint32_t v, uint32_t edges,
                                             unsigned long long* pack, uint32_t* q, uint64_t* offs) {
  const unsigned lane = lane_id();
  unsigned long long mine = want ? ((1ull << kCountShift) | edges) : 0ull;
  unsigned long long incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= unsigned(o)) incl += t;
  }
  const unsigned long long total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(pack, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  if (want) {
    const unsigned long long ex = base + incl - mine;
    const uint32_t pos = uint32_t(ex >> kCountShift);
    q[pos] = v;
    offs[pos] = ex & kEdgeMask;
  }
}

__device__ __forceinline__ bool fb_probe(const uint32_t* s_fb, uint32_t s_words,
                                         const uint32_t* __restrict__ fb, uint32_t u) {
  const uint32_t w = u >> 5;
  const uint32_t word = w < s_words ? s_fb[w] : __ldg(&fb[w]);
  return (word >> (u & 31u)) & 1u;
}

// ------------------------------------------------------------- control
__global__ void k_bfs_init(Ctl* ctl, uint32_t* vis, uint64_t words, uint64_t root_ext,
                           const uint32_t* perm, uint32_t* q1, uint64_t* offs1,
                           const uint32_t* deg, int32_t* level, uint64_t n, uint64_t m,
                           uint64_t nv, int32_t max_it) {
  const uint32_t root = perm ? perm[root_ext] : uint32_t(root_ext);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x)
    vis[i] = (i == (root >> 5)) ? (1u << (root & 31u)) : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q1[0] = root;
    offs1[0] = 0;
    offs1[1] = deg[root];
    level[root] = 0;
    ctl->nf = 1;
    ctl->mf = deg[root];
    ctl->it = 0;
    ctl->prev_pull = 0;
    ctl->cur_is_queue = 1;
    ctl->done = max_it <= 0;
    ctl->max_it = max_it;
    ctl->n_total = n;
    ctl->m_total = m;
    ctl->nv = nv;
  }
}

// Superstep prologue: direction choice and counter reset (one thread).
__global__ void k_decide(Ctl* ctl, uint64_t* offs_cur) {
  if (ctl->done) return;
  const int32_t it = ++ctl->it;
  const uint64_t nf = ctl->nf, mf = ctl->mf;
  int32_t pull;
  if (it == 1)
    pull = 0;
  else if (ctl->prev_pull)
    pull = nf * 24 >= ctl->n_total;
  else
    pull = double(mf) > 0.05 * double(ctl->m_total);
  ctl->dir = pull ? kPull : kPush;
  ctl->qpack = ctl->dpack = ctl->found_n = ctl->found_e = ctl->examined = 0;
  if (!pull && ctl->cur_is_queue) offs_cur[nf] = mf;
}

// Superstep epilogue (one thread): next frontier, stats record, termination.
__global__ void k_finish(Ctl* ctl, uint64_t* offs_next) {
  if (ctl->done) return;
  const int32_t it = ctl->it;
  uint64_t nn, mn;
  if (ctl->dir == kPush) {
    nn = ctl->qpack >> kCountShift;
    mn = ctl->qpack & kEdgeMask;
    offs_next[nn] = mn;
  } else {
    nn = ctl->found_n;
    mn = ctl->found_e;
  }
  if (it <= kMaxRecorded) {
    StepRec& r = ctl->rec[it - 1];
    r.active = int64_t(ctl->nf);
    r.updated = int64_t(nn);
    r.edges = int64_t(ctl->dir == kPush ? ctl->mf : ctl->examined);
    r.examined = int64_t(ctl->examined);
    r.dir = ctl->dir;
  }
  ctl->prev_pull = ctl->dir == kPull;
  ctl->cur_is_queue = ctl->dir == kPush;
  ctl->nf = nn;
  ctl->mf = mn;
  if (nn == 0 || it >= ctl->max_it) ctl->done = 1;
}

// ------------------------------------------------------------------- BFS
// bitmap -> queue (+ offsets) when a push follows a pull.
__global__ void __launch_bounds__(kThreads) k_bfs_b2q(const Ctl* ctl, const uint32_t* fb,
                                                      uint64_t words, const uint32_t* deg,
                                                      uint32_t* q, uint64_t* offs,
                                                      unsigned long long* pack) {
  if (ctl->done || ctl->dir != kPush || ctl->cur_is_queue) return;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint32_t word = fb[w];
    if (!word) continue;  // warp-uniform
    const uint32_t v = uint32_t(w * 32 + lane_id());
    const bool set = (word >> lane_id()) & 1u;
    warp_enqueue(set, v, set ? deg[v] : 0, pack, q, offs);
  }
}

// Edge-balanced push.  pack_cur holds the b2q counter (count of the current
// queue when it came from a bitmap); the frontier size is ctl->nf either way.
__global__ void __launch_bounds__(kThreads) k_bfs_push(Ctl* ctl, const uint32_t* __restrict__ q,
                                                       const uint64_t* __restrict__ offs,
                                                       const uint64_t* __restrict__ ptr,
                                                       const uint32_t* __restrict__ idx,
                                                       const uint32_t* __restrict__ deg,
                                                       int32_t* level, uint32_t* vis,
                                                       uint32_t* fb_next, uint32_t* qn,
                                                       uint64_t* offs_n) {
  if (ctl->done || ctl->dir != kPush) return;
  const uint32_t nq = uint32_t(ctl->nf);
  const uint64_t total = ctl->mf;
  const int32_t next_level = ctl->it;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t wb = warp * 32 * kEPT; wb < total; wb += nwarps * 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    uint32_t i = 0;
    uint64_t e = 0, rem = 0;
    if (t0 < total) {
      i = find_source(offs, nq, t0);
      e = ptr[q[i]] + (t0 - offs[i]);
      rem = (i + 1 < nq ? offs[i + 1] : total) - t0;
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      const uint64_t t = t0 + k;
      bool won = false;
      uint32_t v = 0;
      if (t < total) {
        while (rem == 0) {  // next queue entry with edges
          ++i;
          e = ptr[q[i]];
          rem = (i + 1 < nq ? offs[i + 1] : total) - offs[i];
        }
        v = idx[e];
        ++e;
        --rem;
        const uint32_t bit = 1u << (v & 31u);
        if (!(vis[v >> 5] & bit)) won = !(atomicOr(&vis[v >> 5], bit) & bit);
        if (won) {
          level[v] = next_level;
          atomicOr(&fb_next[v >> 5], bit);
        }
      }
      warp_enqueue(won, v, won ? deg[v] : 0, &ctl->qpack, qn, offs_n);
    }
  }
}

// Pull pass 1: thread per unvisited row, at most kPullProbes probes.
__global__ void __launch_bounds__(kThreads, 2) k_bfs_pull1(
    Ctl* ctl, const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ fb, uint32_t s_words, uint32_t* vis, uint32_t* nbm,
    int32_t* level, const uint32_t* __restrict__ outdeg, uint32_t* defq, uint64_t* defo) {
  if (ctl->done || ctl->dir != kPull) return;
  extern __shared__ uint32_t s_fb[];
  for (uint32_t i = threadIdx.x; i < s_words; i += blockDim.x) s_fb[i] = fb[i];
  __syncthreads();
  const uint64_t nv = ctl->nv;
  const int32_t next_level = ctl->it;
  const uint64_t words = (nv + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint32_t vw = vis[w];
    if (vw == 0xFFFFFFFFu) {  // warp-uniform: all 32 rows already visited
      if (lane == 0) nbm[w] = 0u;
      continue;
    }
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
    if (lane == 0) {
      nbm[w] = b;
      if (b) vis[w] = vw | b;
    }
    found_n += found;
    if (__any_sync(0xffffffffu, defer)) warp_enqueue(defer, uint32_t(v), rest, &ctl->dpack, defq, defo);
  }
  warp_add_u64(&ctl->found_n, found_n);
  warp_add_u64(&ctl->found_e, found_e);
  warp_add_u64(&ctl->examined, examined);
}

// Pull pass 2: edge-balanced over the deferred rows' remaining in-edges; a row
// is claimed once through its next-frontier bit.
__global__ void __launch_bounds__(kThreads, 2) k_bfs_pull2(
    Ctl* ctl, const uint32_t* __restrict__ defq, const uint64_t* __restrict__ defo,
    const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ fb, uint32_t s_words, uint32_t* vis, uint32_t* nbm,
    int32_t* level, const uint32_t* __restrict__ outdeg) {
  if (ctl->done || ctl->dir != kPull) return;
  const unsigned long long dp = ctl->dpack;
  const uint32_t ndef = uint32_t(dp >> kCountShift);
  const uint64_t total = dp & kEdgeMask;
  if (ndef == 0) return;
  extern __shared__ uint32_t s_fb[];
  for (uint32_t i = threadIdx.x; i < s_words; i += blockDim.x) s_fb[i] = fb[i];
  __syncthreads();
  const int32_t next_level = ctl->it;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long found_n = 0, found_e = 0, examined = 0;
  for (uint64_t wb = warp * 32 * kEPT; wb < total; wb += nwarps * 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    if (t0 >= total) continue;
    uint32_t i = find_source(defo, ndef, t0);
    uint32_t v = defq[i];
    uint64_t e = ptr[v] + kPullProbes + (t0 - defo[i]);
    uint64_t rem = (i + 1 < ndef ? defo[i + 1] : total) - t0;
    for (int k = 0; k < kEPT && t0 + k < total; ++k) {
      while (rem == 0) {
        ++i;
        v = defq[i];
        e = ptr[v] + kPullProbes;
        rem = (i + 1 < ndef ? defo[i + 1] : total) - defo[i];
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
  warp_add_u64(&ctl->found_n, found_n);
  warp_add_u64(&ctl->found_e, found_e);
  warp_add_u64(&ctl->examined, examined);
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
__global__ void k_sssp_init(Ctl* ctl, uint32_t* dist, uint64_t n, uint64_t root_ext,
                            const uint32_t* perm, uint32_t* q1, uint64_t* offs1, uint32_t* dq1,
                            const uint32_t* deg, uint64_t m, int32_t max_it) {
  const uint32_t root = perm ? perm[root_ext] : uint32_t(root_ext);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dist[i] = i == root ? 0u : 0xFFFFFFFFu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q1[0] = root;
    dq1[0] = 0;
    offs1[0] = 0;
    offs1[1] = deg[root];
    ctl->nf = 1;
    ctl->mf = deg[root];
    ctl->it = 0;
    ctl->prev_pull = 0;
    ctl->cur_is_queue = 1;
    ctl->done = max_it <= 0;
    ctl->max_it = max_it;
    ctl->n_total = n;
    ctl->m_total = m;
  }
}

// SSSP prologue: always push.
__global__ void k_sssp_decide(Ctl* ctl) {
  if (ctl->done) return;
  ++ctl->it;
  ctl->dir = kPush;
  ctl->qpack = ctl->examined = 0;
}

template <typename W>
__global__ void __launch_bounds__(kThreads) k_sssp_push(Ctl* ctl, const uint32_t* __restrict__ q,
                                                        const uint32_t* __restrict__ dq,
                                                        const uint64_t* __restrict__ offs,
                                                        const uint64_t* __restrict__ ptr,
                                                        const uint32_t* __restrict__ idx,
                                                        const W* __restrict__ wt,
                                                        const uint32_t* __restrict__ deg,
                                                        uint32_t* dist, uint32_t* changed,
                                                        uint32_t* qn, uint64_t* offs_n) {
  if (ctl->done) return;
  const uint32_t nq = uint32_t(ctl->nf);
  const uint64_t total = ctl->mf;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t wb = warp * 32 * kEPT; wb < total; wb += nwarps * 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    uint32_t i = 0;
    uint64_t e = 0, rem = 0, du = 0;
    if (t0 < total) {
      i = find_source(offs, nq, t0);
      du = dq[i];
      e = ptr[q[i]] + (t0 - offs[i]);
      rem = (i + 1 < nq ? offs[i + 1] : total) - t0;
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      const uint64_t t = t0 + k;
      bool won = false;
      uint32_t v = 0;
      if (t < total) {
        while (rem == 0) {
          ++i;
          du = dq[i];
          e = ptr[q[i]];
          rem = (i + 1 < nq ? offs[i + 1] : total) - offs[i];
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
      warp_enqueue(won, v, won ? deg[v] : 0, &ctl->qpack, qn, offs_n);
    }
  }
}

// Next frontier's message snapshot (after every relaxation of the superstep
// landed); resets the changed-bits for the next superstep.
__global__ void k_sssp_snapshot(const Ctl* ctl, const uint32_t* q, const uint32_t* dist,
                                uint32_t* dq, uint32_t* changed) {
  if (ctl->done) return;
  const uint32_t nq = uint32_t(ctl->qpack >> kCountShift);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x) {
    const uint32_t v = q[i];
    dq[i] = dist[v];
    changed[v >> 5] = 0u;
  }
}

template <typename T>
__global__ void k_gather_out(uint64_t n, const uint32_t* perm, const T* in, T* out) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    out[v] = in[perm ? perm[v] : v];
}

void ensure_events(TravCache& c, size_t need) {
  while (c.ev.size() < need) {
    cudaEvent_t e;
    GM_CUDA(cudaEventCreate(&e));
    c.ev.push_back(e);
  }
}

// Host driver shared by BFS and SSSP: enqueue supersteps in batches of
// kBatch, reading the device's done flag once per batch.
template <typename Enqueue>
int64_t run_batches(TravCache& c, cudaStream_t s, int64_t max_iters, bool collect, Enqueue&& step) {
  int32_t* done = c.hdone->get();
  int64_t enq = 0;
  while (enq < max_iters) {
    const int64_t nb = std::min<int64_t>(kBatch, max_iters - enq);
    for (int64_t b = 0; b < nb; ++b, ++enq) {
      const bool rec = collect && enq < kMaxRecorded;
      if (rec) ensure_events(c, size_t(2 * enq + 2));
      if (rec) GM_CUDA(cudaEventRecord(c.ev[2 * enq], s));
      step(enq + 1);
      if (rec) GM_CUDA(cudaEventRecord(c.ev[2 * enq + 1], s));
    }
    GM_CUDA(cudaMemcpyAsync(done, &c.ctl.get()->done, 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    if (*done) break;
  }
  return enq;
}

std::vector<gm_iteration_stats> read_records(TravCache& c, cudaStream_t s, int64_t enqueued,
                                             uint64_t n, uint64_t nv, bool collect) {
  std::vector<gm_iteration_stats> stats;
  if (!collect) return stats;
  int32_t it = 0;
  GM_CUDA(cudaMemcpyAsync(&it, &c.ctl.get()->it, 4, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  const int64_t nrec = std::min<int64_t>(it, kMaxRecorded);
  std::vector<StepRec> rec(size_t(nrec > 0 ? nrec : 1));
  if (nrec > 0)
    GM_CUDA(cudaMemcpyAsync(rec.data(), c.ctl.get()->rec, nrec * sizeof(StepRec),
                            cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < nrec; ++i) {
    const StepRec& r = rec[i];
    gm_iteration_stats st{};
    st.iteration = i + 1;
    st.active_before = r.active;
    st.messages_generated = r.active;
    st.vertices_updated = r.updated;
    float ms = 0;
    if (i < enqueued) GM_CUDA(cudaEventElapsedTime(&ms, c.ev[2 * i], c.ev[2 * i + 1]));
    st.spmv_seconds = ms * 1e-3;
    st.total_seconds = ms * 1e-3;
    st.edges_processed = r.edges;
    st.direction = r.dir == kPush ? 1 : 0;
    // pull: vis + ptr per candidate row, examined col ids, level + bitmap writes
    // push: queue + offsets + ptr per frontier vertex, col id per edge,
    //       level + queue + offsets per discovered vertex, next bitmap
    st.bytes_algorithmic = r.dir == kPush
                               ? int64_t(24 * r.active + 4 * r.edges + 16 * r.updated + n / 8)
                               : int64_t(16 * nv + 4 * r.examined + 4 * r.updated + 2 * n / 8);
    stats.push_back(st);
  }
  return stats;
}

}  // namespace

std::vector<gm_iteration_stats> bfs(Graph& g, uint64_t root, int64_t max_iters, int32_t* out,
                                    bool out_on_device, bool collect) {
  const uint64_t n = g.n;
  if (root >= n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(n));
  if (n >= (1ull << (64 - kCountShift)))
    fail(GM_EUSAGE, "bfs: graphs above 2^28 vertices are not supported by the packed queue");
  TravCache& c = cache(g);
  cudaStream_t s = g.stream;
  if (!c.level) c.level.alloc(n, s);
  if (!c.attrs) {
    GM_CUDA(cudaFuncSetAttribute(k_bfs_pull1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kSmemFbWords * 4)));
    GM_CUDA(cudaFuncSetAttribute(k_bfs_pull2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kSmemFbWords * 4)));
    c.attrs = true;
  }
  ensure_forward(g);
  const Csr& fw = g.fwd();
  const uint64_t words = (n + 31) / 32;
  // Pull rows: on a relabeled symmetric graph only the nonzero-degree prefix
  // can ever be reached.
  const uint64_t nv = (g.relabeled && g.symmetric) ? g.nonzero_outdeg : n;
  const uint32_t s_words = uint32_t(std::min<uint64_t>(kSmemFbWords, (nv + 31) / 32));
  const size_t smem = size_t(s_words) * 4;
  const uint32_t* perm = g.relabeled ? g.perm.get() : nullptr;
  const int32_t max_it = int32_t(std::min<int64_t>(max_iters, 0x7FFFFFFF));
  Ctl* ctl = c.ctl.get();
  k_bfs_init<<<grid_for(words + 1, 256), 256, 0, s>>>(ctl, c.vis.get(), words + 1, root, perm,
                                                      c.q[1].get(), c.offs[1].get(),
                                                      g.outdeg.get(), c.level.get(), n, g.m, nv,
                                                      max_it);
  GM_LAUNCH_CHECK();
  const int64_t enq = run_batches(c, s, max_iters, collect, [&](int64_t it) {
    const int cur = int(it & 1), nxt = cur ^ 1;
    GM_CUDA(cudaMemsetAsync(c.fb[nxt].get(), 0, (words + 1) * 4, s));
    k_decide<<<1, 1, 0, s>>>(ctl, c.offs[cur].get());
    GM_LAUNCH_CHECK();
    // push path (kernels exit at once when the device chose pull)
    k_bfs_b2q<<<kGrid, kThreads, 0, s>>>(ctl, c.fb[cur].get(), words, g.outdeg.get(), c.q[cur].get(),
                                          c.offs[cur].get(), &ctl->dpack);
    GM_LAUNCH_CHECK();
    k_bfs_push<<<kGrid, kThreads, 0, s>>>(ctl, c.q[cur].get(), c.offs[cur].get(), fw.ptr.get(),
                                           fw.idx.get(), g.outdeg.get(), c.level.get(), c.vis.get(),
                                           c.fb[nxt].get(), c.q[nxt].get(), c.offs[nxt].get());
    GM_LAUNCH_CHECK();
    // pull path
    k_bfs_pull1<<<kGrid, kThreads, smem, s>>>(ctl, g.in.ptr.get(), g.in.idx.get(), c.fb[cur].get(),
                                              s_words, c.vis.get(), c.fb[nxt].get(), c.level.get(),
                                              g.outdeg.get(), c.defq.get(), c.defo.get());
    GM_LAUNCH_CHECK();
    k_bfs_pull2<<<kGrid, kThreads, smem, s>>>(ctl, c.defq.get(), c.defo.get(), g.in.ptr.get(),
                                              g.in.idx.get(), c.fb[cur].get(), s_words, c.vis.get(),
                                              c.fb[nxt].get(), c.level.get(), g.outdeg.get());
    GM_LAUNCH_CHECK();
    k_finish<<<1, 1, 0, s>>>(ctl, c.offs[nxt].get());
    GM_LAUNCH_CHECK();
  });
  std::vector<gm_iteration_stats> stats = read_records(c, s, enq, n, nv, collect);
  if (out) {
    int32_t* dst = out;
    if (!out_on_device) {
      if (!c.ext_out) c.ext_out.alloc(n, s);
      dst = c.ext_out.get();
    }
    k_bfs_output<<<grid_for(n, 256), 256, 0, s>>>(n, perm, c.vis.get(), c.level.get(), dst);
    GM_LAUNCH_CHECK();
    if (!out_on_device) GM_CUDA(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
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
  if (n >= (1ull << (64 - kCountShift)))
    fail(GM_EUSAGE, "sssp: graphs above 2^28 vertices are not supported by the packed queue");
  TravCache& c = cache(g);
  cudaStream_t s = g.stream;
  if (!c.dist) {
    c.dist.alloc(n, s);
    c.dq[0].alloc(n + 1, s);
    c.dq[1].alloc(n + 1, s);
    c.changed.alloc((n + 31) / 32 + 1, s);
  }
  c.changed.zero(s);
  ensure_forward(g);
  const Csr& fw = g.fwd();
  const uint32_t* perm = g.relabeled ? g.perm.get() : nullptr;
  const int32_t max_it = int32_t(std::min<int64_t>(max_iters, 0x7FFFFFFF));
  Ctl* ctl = c.ctl.get();
  k_sssp_init<<<grid_for(n, 256), 256, 0, s>>>(ctl, c.dist.get(), n, root, perm, c.q[1].get(),
                                               c.offs[1].get(), c.dq[1].get(), g.outdeg.get(), g.m,
                                               max_it);
  GM_LAUNCH_CHECK();
  const bool u8 = g.value_type == GM_VAL_U8;
  const int64_t enq = run_batches(c, s, max_iters, collect, [&](int64_t it) {
    const int cur = int(it & 1), nxt = cur ^ 1;
    k_sssp_decide<<<1, 1, 0, s>>>(ctl);
    GM_LAUNCH_CHECK();
    if (u8)
      k_sssp_push<uint8_t><<<kGrid, kThreads, 0, s>>>(
          ctl, c.q[cur].get(), c.dq[cur].get(), c.offs[cur].get(), fw.ptr.get(), fw.idx.get(),
          fw.val.get(), g.outdeg.get(), c.dist.get(), c.changed.get(), c.q[nxt].get(),
          c.offs[nxt].get());
    else
      k_sssp_push<uint32_t><<<kGrid, kThreads, 0, s>>>(
          ctl, c.q[cur].get(), c.dq[cur].get(), c.offs[cur].get(), fw.ptr.get(), fw.idx.get(),
          reinterpret_cast<const uint32_t*>(fw.val.get()), g.outdeg.get(), c.dist.get(),
          c.changed.get(), c.q[nxt].get(), c.offs[nxt].get());
    GM_LAUNCH_CHECK();
    k_sssp_snapshot<<<kGrid, kThreads, 0, s>>>(ctl, c.q[nxt].get(), c.dist.get(), c.dq[nxt].get(),
                                               c.changed.get());
    GM_LAUNCH_CHECK();
    k_finish<<<1, 1, 0, s>>>(ctl, c.offs[nxt].get());
    GM_LAUNCH_CHECK();
  });
  std::vector<gm_iteration_stats> stats = read_records(c, s, enq, n, n, collect);
  for (auto& st : stats)  // SSSP reads a u8/u32 weight with every col id, and a snapshot per vertex
    st.bytes_algorithmic = int64_t(28 * st.active_before + 5 * st.edges_processed +
                                   20 * st.vertices_updated + n / 8);
  if (out) {
    uint32_t* dst = out;
    if (!out_on_device) {
      if (!c.ext_out) c.ext_out.alloc(n, s);
      dst = reinterpret_cast<uint32_t*>(c.ext_out.get());
    }
    k_gather_out<uint32_t><<<grid_for(n, 256), 256, 0, s>>>(n, perm, c.dist.get(), dst);
    GM_LAUNCH_CHECK();
    if (!out_on_device) GM_CUDA(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
  return stats;
}

}  // namespace gm
