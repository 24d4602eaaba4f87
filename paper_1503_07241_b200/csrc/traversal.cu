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
//        kHead in-neighbours per row (thread per row, one 16-byte head load);
//        rows still open
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
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "api_internal.cuh"

namespace gm {

namespace {

constexpr int kMaxRecorded = 4096;  // per-superstep records kept on device
constexpr int kBatch = 4;           // supersteps enqueued per host check
constexpr int kEPT = 4;             // edges per thread, edge-balanced passes
// Frontier-bitmap prefix staged per CTA: 96 KB at 2 CTAs per SM, 64 KB at 3.
// Frontier-bitmap prefix in shared memory per CTA (words): what it does not
// take stays L1 for the head and visited loads.  Measured (re-entry session,
// tools/gpu_r02y32.sh / y33.sh): the 2-CTA variant (scale 23) 24 K words
// 0.299 ms per BFS, 8 K 0.285, 4 K 0.281, 2 K 0.282, 1 K 0.332 (the hubs no
// longer fit); the 3-CTA variant (scale 28) 16 K 2.846 ms, 8 K 2.866, 4 K
// 2.899.  GM_BFS_PREFIX_WORDS overrides (measurement hook).
inline uint32_t smem_fb_words(int blocks_per_sm) {
  static const char* e = getenv("GM_BFS_PREFIX_WORDS");
  if (e) return uint32_t(std::max(32L, std::min(24L * 1024, strtol(e, nullptr, 10))));
  return blocks_per_sm >= 3 ? 16 * 1024 : 4 * 1024;
}
constexpr unsigned kGrid = 148 * 2;           // persistent grid for the SSSP kernels
constexpr unsigned kThreads = 1024;
constexpr int kCountShift = 36;  // packed counter: count << 36 | edges
constexpr unsigned long long kEdgeMask = (1ull << kCountShift) - 1;

enum Dir : int32_t { kPush = 1, kPull = 0 };
constexpr unsigned kHdrDone = 1, kHdrPrevPull = 2, kHdrCurIsQueue = 4, kHdrUImplicit = 8, kHdrUsel = 16;

struct StepRec {
  int64_t active, updated, edges, examined;
  int64_t deferred, deferred_edges;  // pull pass 2 work
  int32_t dir, pad;
};

// Device-resident superstep state.
struct Ctl {
  unsigned long long qpack;     // next queue (count << 36 | edges)
  unsigned long long dpack;     // deferred rows (count << 36 | remaining edges)
  unsigned long long bpack;     // bitmap -> queue conversion counter
  unsigned long long upack;     // next unvisited-row list length
  unsigned long long found_n, found_e, examined;
  unsigned long long nf, mf;    // current frontier: vertices, edges
  unsigned long long ucur;      // current unvisited-row list length
  unsigned int wcursor;         // implicit pull: next unclaimed visited-bitmap word
  int32_t it, dir, prev_pull, cur_is_queue, done, max_it, u_implicit, usel;
  int32_t queue_out;            // SSSP: pull supersteps also append to the queue
  uint64_t n_total, m_total, nv;
  // BFS superstep header, written by the epilogue thread and read once per CTA
  // (every warp reading the fields above hit one L2 line ~10K times per step):
  // nf, mf, ucur, it | flags << 32 (kHdr*).
  alignas(16) unsigned long long hdr[4];
  uint64_t t_start[kMaxRecorded];  // %globaltimer per superstep (cooperative kernel)
  uint64_t t_mid[kMaxRecorded];    // after the first phase (bitmap->queue / pull pass 1)
  uint64_t t_end[kMaxRecorded];
  StepRec rec[kMaxRecorded];
  uint64_t t_entry, t_exit;        // cooperative kernel entry / exit (GM_BFS_PHASES)
};

}  // namespace

struct TravCache {
  uint64_t n = 0;
  // BFS levels as stamps: BFS number i writes lbase_i + level, and a stamp
  // below lbase_i is "unreached", so no BFS clears the array (a 4-byte-per-
  // vertex memset or clearing pass, 0.16 ms at scale 28); the host advances
  // lbase by a bound on the BFS depth and zeroes the array only when the
  // 32-bit stamps would wrap.
  DevBuf<uint32_t> level;
  uint64_t lbase = 0;  // 0: the array needs zeroing before the next BFS
  // Compact output (symmetric degree relabel, isolated tail [nv, n)): bitmap
  // of callers with a nonzero degree, non-isolated callers before each block
  // of 1024 callers, and the internal id of every non-isolated caller in
  // caller order.
  DevBuf<uint32_t> nzb, nz_base, perm_c;
  DevBuf<uint32_t> dist;
  DevBuf<uint32_t> q[2];        // frontier queues (internal ids)
  DevBuf<uint64_t> offs[2];     // exclusive edge offsets, parallel to q (+1 total)
  DevBuf<uint32_t> dq[2];       // SSSP message snapshots parallel to q
  DevBuf<uint32_t> defq;        // pull: deferred rows
  DevBuf<uint32_t> ul[2];       // pull: unvisited-row lists
  DevBuf<uint32_t> hsoa;        // pull: in-neighbours 0..kSoa-1 of every row, slot-major
  DevBuf<uint4> head;           // pull: in-neighbours kSoa..kHead-1 per row (AoS)
  DevBuf<uint64_t> qe[2];       // start-edge pointers parallel to q
  DevBuf<uint64_t> defe;        // pull: deferred rows' next unprobed edge
  unsigned coop_grid = 0;
  int coop_blocks_per_sm = 0;  // k_bfs_coop variant, fixed at the first BFS
  DevBuf<uint64_t> defo;        // pull: their exclusive remaining-edge offsets
  DevBuf<uint32_t> vis, fb[2];  // visited / frontier bitmaps (cur = it & 1)
  DevBuf<uint32_t> changed;     // SSSP changed-bitmap
  DevBuf<uint32_t> msg;         // SSSP pull: superstep-start distance of frontier sources, else INF
  DevBuf<uint32_t> rowid;       // SSSP pull: row of every CSR(G^T) entry
  uint32_t pull_hub = 0;        // SSSP pull: msg[0, pull_hub) staged in shared memory
  unsigned pull_grid = 0;
  DevBuf<Ctl> ctl;
  DevBuf<int32_t> ext_out;      // caller-order staging for host outputs
  std::unique_ptr<HostPinned<int32_t>> hdone;
  bool attrs = false;
  // SSSP: one batch of kBatch supersteps captured as a CUDA graph (its kernels
  // read everything else from Ctl), keyed by the launch configuration
  cudaGraphExec_t sssp_exec = nullptr;
  int sssp_key = -1;
  int sssp_launches = 0;  // kernels per replay (for the launch counter)
  ~TravCache() {
    if (sssp_exec) cudaGraphExecDestroy(sssp_exec);
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
    c.defe.alloc(n + 1, s);
    c.qe[0].alloc(n + 1, s);
    c.qe[1].alloc(n + 1, s);
    c.ul[0].alloc(n + 1, s);
    c.ul[1].alloc(n + 1, s);
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
    if (offs) offs[pos] = ex & kEdgeMask;
  }
}

// Warp-private staging of queue appends in shared memory: appends are
// buffered and published CAP at a time with one packed atomicAdd on the queue
// counter (count << kCountShift | edges), instead of one atomicAdd per warp
// step, which serialises at the L2 when many warps append a few entries each.
// kOffs: also write each entry's exclusive edge offset; kQe: and a u64 payload.
constexpr uint32_t kPushCap = 64;  // SSSP push: staged appends per warp

template <uint32_t CAP, bool kOffs, bool kQe>
struct StagedQ {
  uint32_t* sv;  // [CAP] vertices
  uint32_t* sd;  // [CAP] edge counts (kOffs)
  uint64_t* se;  // [CAP] payloads (kQe)
  uint32_t cnt = 0;
  __device__ __forceinline__ void flush(unsigned long long* pack, uint32_t* q, uint64_t* offs,
                                        uint64_t* qe) {
    const unsigned lane = lane_id();
    if (cnt == 0) return;
    __syncwarp();
    unsigned long long tot_e = 0;
    if (kOffs)
      for (uint32_t b = 0; b < cnt; b += 32) {
        uint64_t d = b + lane < cnt ? sd[b + lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        tot_e += d;
      }
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(pack, (uint64_t(cnt) << kCountShift) | tot_e);
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint64_t bpos = base >> kCountShift;
    uint64_t carry = base & kEdgeMask;
    for (uint32_t b = 0; b < cnt; b += 32) {
      const bool in = b + lane < cnt;
      uint64_t d = (kOffs && in) ? sd[b + lane] : 0, incl = d;
      if (kOffs) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= unsigned(o)) incl += t;
        }
      }
      if (in) {
        q[bpos + b + lane] = sv[b + lane];
        if (kOffs) offs[bpos + b + lane] = carry + incl - d;
        if (kQe) qe[bpos + b + lane] = se[b + lane];
      }
      if (kOffs) carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    cnt = 0;
  }
  __device__ __forceinline__ void push(bool want, uint32_t v, uint32_t edges, uint64_t payload,
                                       unsigned long long* pack, uint32_t* q, uint64_t* offs,
                                       uint64_t* qe) {
    const unsigned lane = lane_id();
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    if (cnt + 32 > CAP) flush(pack, q, offs, qe);
    if (want) {
      const uint32_t pos = cnt + __popc(m & ((1u << lane) - 1u));
      sv[pos] = v;
      if (kOffs) sd[pos] = edges;
      if (kQe) se[pos] = payload;
    }
    cnt += __popc(m);
  }
};

// Warp-aggregated append of up to kMaxPer entries per lane: (vertex, edge
// count, start-edge pointer) -> q / offs / qe with one packed atomicAdd.
template <int kMaxPer>
__device__ __forceinline__ void warp_enqueue_multi(unsigned mask, const uint32_t* v,
                                                   const uint32_t* edges, const uint64_t* estart,
                                                   unsigned long long* pack, uint32_t* q,
                                                   uint64_t* offs, uint64_t* qe) {
  const unsigned lane = lane_id();
  unsigned long long mine = 0;
#pragma unroll
  for (int k = 0; k < kMaxPer; ++k)
    if ((mask >> k) & 1u) mine += (1ull << kCountShift) | edges[k];
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
  unsigned long long ex = base + incl - mine;
#pragma unroll
  for (int k = 0; k < kMaxPer; ++k) {
    if ((mask >> k) & 1u) {
      const uint32_t pos = uint32_t(ex >> kCountShift);
      q[pos] = v[k];
      offs[pos] = ex & kEdgeMask;
      qe[pos] = estart[k];
      ex += (1ull << kCountShift) | edges[k];
    }
  }
}

// ------------------------------------------------------------- control
// Also clears both frontier bitmaps and the control block's counters (three
// memsets per BFS before: stream operations that cost more than their bytes
// on small graphs).
__global__ void k_bfs_init(Ctl* ctl, uint32_t* vis, uint32_t* fb0, uint32_t* fb1, uint64_t words,
                           uint64_t root_ext, const uint32_t* perm, uint32_t* q1, uint64_t* offs1,
                           uint64_t* qe1, const uint64_t* out_ptr, const uint32_t* deg,
                           uint32_t* level, uint32_t lbase, uint64_t n, uint64_t m, uint64_t nv,
                           int32_t max_it) {
  const uint32_t root = perm ? perm[root_ext] : uint32_t(root_ext);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    vis[i] = (i == (root >> 5)) ? (1u << (root & 31u)) : 0u;
    fb0[i] = 0u;
    fb1[i] = 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    static_assert(offsetof(Ctl, t_start) % 8 == 0, "control block counters are 8-byte words");
    for (size_t b = 0; b < offsetof(Ctl, t_start); b += 8)
      *reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctl) + b) = 0ull;
    q1[0] = root;
    offs1[0] = 0;
    offs1[1] = deg[root];
    qe1[0] = out_ptr[root];
    level[root] = lbase;
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
    ctl->u_implicit = 1;  // first pull scans every row; later pulls the unvisited list
    ctl->usel = 0;
    ctl->ucur = 0;
    ctl->hdr[0] = 1;
    ctl->hdr[1] = deg[root];
    ctl->hdr[2] = 0;
    ctl->hdr[3] = uint64_t(kHdrCurIsQueue | kHdrUImplicit | (max_it <= 0 ? kHdrDone : 0u)) << 32;
  }
}

// Superstep epilogue (one thread): next frontier, stats record, termination.
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_finish(Ctl* ctl, uint64_t* offs_next) {
  if (ctl->done) return;
  const int32_t it = ctl->it;
  if (it <= kMaxRecorded) ctl->t_end[it - 1] = gtimer();
  uint64_t nn, mn;
  if (ctl->dir == kPush || ctl->queue_out) {
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
  ctl->cur_is_queue = ctl->dir == kPush || ctl->queue_out;
  ctl->nf = nn;
  ctl->mf = mn;
  if (nn == 0 || it >= ctl->max_it) ctl->done = 1;
}

// ------------------------------------------------------------------- BFS
// Caller-order output: out[x] = level of perm[x] (stamp - lbase, or -1 for a
// stamp below lbase: not reached by this BFS).  Generic form for graphs
// without the symmetric degree relabel (perm null: identity).
__global__ void k_bfs_output(uint64_t n, uint64_t root_ext, const uint32_t* perm,
                             const uint32_t* stamp, uint32_t lbase, int32_t* out) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t st = __ldg(&stamp[perm ? __ldg(&perm[v]) : uint32_t(v)]);
    out[v] = v == root_ext ? 0 : (st >= lbase ? int32_t(st - lbase) : -1);
  }
}

// Compact caller-order output under the symmetric degree relabel.  Isolated
// vertices form the internal tail [nv, n) and are unreachable (the root aside,
// handled by id), so their -1 needs no perm entry and no gather: a warp takes
// 1024 callers, reads their 32 words of the non-isolated bitmap, and only the
// set bits read a compacted perm entry (perm_c, non-isolated callers in caller
// order) and gather a stamp.  At scale 28 about half the vertices are
// isolated: the pass reads ~0.5 GB of perm_c instead of 1 GB of perm and
// writes only the output.  Within one degree class internal ids follow caller
// order, so the stamp gathers of nearby callers share sectors.
template <int kB>
__global__ void __launch_bounds__(256) k_bfs_output_nz(uint64_t n, uint64_t root_ext,
                                                       const uint32_t* __restrict__ nzb,
                                                       const uint32_t* __restrict__ nz_base,
                                                       const uint32_t* __restrict__ perm_c,
                                                       const uint32_t* __restrict__ stamp,
                                                       uint32_t lbase, int32_t* __restrict__ out) {
  const unsigned lane = lane_id();
  const uint64_t nwords = (n + 31) / 32, nblk = (n + 1023) / 1024;
  const uint64_t gw = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t b = gw; b < nblk; b += nw) {
    const uint64_t wi = b * 32 + lane;
    const uint32_t word = wi < nwords ? __ldcs(&nzb[wi]) : 0u;
    const uint32_t cnt = __popc(word);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= unsigned(o)) incl += t;
    }
    const uint32_t wbase = __ldg(&nz_base[b]) + incl - cnt;
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll 1
    for (int r0 = 0; r0 < 32; r0 += kB) {
      uint32_t st[kB];
      bool set[kB];
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const uint32_t wr = __shfl_sync(0xffffffffu, word, r0 + j);
        const uint32_t br = __shfl_sync(0xffffffffu, wbase, r0 + j);
        set[j] = (wr >> lane) & 1u;
        GM_DCHECK(!set[j] || br + __popc(wr & below) < n);
        st[j] = set[j] ? __ldcs(&perm_c[br + __popc(wr & below)]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        GM_DCHECK(!set[j] || st[j] < n);
        st[j] = set[j] ? __ldg(&stamp[st[j]]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const uint64_t x = b * 1024 + uint64_t(r0 + j) * 32 + lane;
        int32_t o = (set[j] && st[j] >= lbase) ? int32_t(st[j] - lbase) : -1;
        if (x == root_ext) o = 0;
        if (x < n) __stcs(&out[x], o);
      }
    }
  }
}

// Build the compact-output tables (once per graph): nzb bit x = (perm[x] < nv).
__global__ void k_nz_bits(uint64_t n, uint64_t nv, const uint32_t* perm, uint32_t* nzb,
                          uint32_t* blk_cnt) {
  const uint64_t nwords = (n + 31) / 32;
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~31ull; w0 < nwords * 32;
       w0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = w0 + lane_id();
    const unsigned bits = __ballot_sync(0xffffffffu, x < n && perm[x] < nv);
    if (lane_id() == 0) {
      nzb[x >> 5] = bits;
      atomicAdd(&blk_cnt[x >> 10], uint32_t(__popc(bits)));
    }
  }
}

__global__ void k_perm_compact(uint64_t n, const uint32_t* perm, const uint32_t* nzb,
                               const uint32_t* nz_base, uint32_t* perm_c) {
  const unsigned lane = lane_id();
  const uint64_t nwords = (n + 31) / 32, nblk = (n + 1023) / 1024;
  const uint64_t gw = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t b = gw; b < nblk; b += nw) {
    const uint64_t wi = b * 32 + lane;
    const uint32_t word = wi < nwords ? nzb[wi] : 0u;
    const uint32_t cnt = __popc(word);
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= unsigned(o)) incl += t;
    }
    uint32_t k = nz_base[b] + incl - cnt;
    for (int i = 0; i < 32; ++i)
      if ((word >> i) & 1u) perm_c[k++] = perm[wi * 32 + i];
  }
}

void build_compact_output(TravCache& c, const uint32_t* perm, uint64_t n, uint64_t nv, cudaStream_t s) {
  const uint64_t nwords = (n + 31) / 32, nblk = (n + 1023) / 1024;
  c.nzb.alloc(nwords + 1, s);
  c.nz_base.alloc(nblk + 1, s);
  c.perm_c.alloc(nv + 1, s);
  c.nz_base.zero(s);
  k_nz_bits<<<grid_for(nwords * 32, 256), 256, 0, s>>>(n, nv, perm, c.nzb.get(), c.nz_base.get());
  GM_LAUNCH_CHECK();
  size_t tmp = 0;
  GM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.nz_base.get(), c.nz_base.get(), int64_t(nblk), s));
  DevBuf<uint8_t> t(tmp + 1, s);
  GM_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, c.nz_base.get(), c.nz_base.get(), int64_t(nblk), s));
  k_perm_compact<<<grid_for(nblk * 32, 256), 256, 0, s>>>(n, perm, c.nzb.get(), c.nz_base.get(),
                                                         c.perm_c.get());
  GM_LAUNCH_CHECK();
}

// ------------------------------------------------ cooperative BFS (all supersteps)
// One persistent cooperative launch runs every superstep: phases are separated
// by grid-wide barriers, the direction is decided identically by every block
// from the device counters, and nothing returns to the host until the BFS is
// done.  Data another block wrote in an earlier phase is read with ld.global.cg
// (L2) so no SM sees a stale L1 line.
constexpr unsigned kCoopThreads = 512;

struct CoopArgs {
  Ctl* ctl;
  const uint64_t* in_ptr;
  const uint32_t* in_idx;   // CSR(G^T): pull
  const uint64_t* out_ptr;
  const uint32_t* out_idx;  // CSR(G): push
  const uint32_t* deg;      // out-degree
  const uint32_t* indeg;    // in-degree (pull row length)
  const uint32_t* hsoa;     // in-neighbour s of row v at hsoa[s * hstride + v], s < kSoa
  const uint4* head;        // in-neighbours kSoa..kHead-1 of each pull row (16 B chunks)
  uint32_t hstride;          // nv + 1 (< 2^28 + 1: 32-bit index math in the pull)
  uint32_t* level;          // stamps: lbase + level (TravCache::level)
  uint32_t lbase;
  uint32_t* vis;
  uint32_t* fb[2];
  uint32_t* q[2];
  uint64_t* offs[2];
  uint64_t* qe[2];          // start-edge pointer of each queued vertex
  uint32_t* ul[2];          // unvisited-row lists
  uint32_t* defq;
  uint64_t* defo;
  uint64_t* defe;           // deferred rows: first edge not probed in pass 1
  uint64_t n, nv, m, words_all;
  uint32_t s_words;
  int32_t use_ulist;        // later pulls walk the unvisited-row list (else every row)
  uint32_t pull_chunk;      // implicit pull, 3-CTA variant: visited words per claim (1..32)
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 32-way warp search: last i in [lo, hi) with offs[i] <= t, given offs[lo] <= t.
// Each round is one batch of 32 independent loads (log32 rounds).
__device__ __forceinline__ uint32_t warp_kary(const uint64_t* offs, uint32_t lo, uint32_t hi,
                                              uint64_t t) {
  const unsigned lane = lane_id();
  while (hi - lo > 1) {
    const uint32_t st = (hi - lo + 31) / 32;
    const uint64_t p = uint64_t(lo) + uint64_t(lane + 1) * st;
    const bool ok = p < hi && __ldcg(&offs[p]) <= t;
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    lo += uint32_t(__popc(b)) * st;
    hi = min(hi, lo + st);
  }
  return lo;
}

// Forward 32-way gallop from a known position (offs[lo] <= t): one round when
// the answer is within 32 entries, which is the common case between chunks.
__device__ __forceinline__ uint32_t warp_forward(const uint64_t* offs, uint32_t nq, uint32_t lo,
                                                 uint64_t t) {
  const unsigned lane = lane_id();
  uint64_t step = 1;
  for (;;) {
    const uint64_t p = uint64_t(lo) + uint64_t(lane + 1) * step;
    const bool ok = p < nq && __ldcg(&offs[p]) <= t;
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    if (b != 0xffffffffu) {
      const uint32_t base = lo + uint32_t(__popc(b) * step);
      return step == 1 ? base
                       : warp_kary(offs, base,
                                   uint32_t(uint64_t(nq) < base + step ? uint64_t(nq) : base + step),
                                   t);
    }
    lo += uint32_t(32 * step);
    step *= 32;
  }
}

// Per-lane gallop from the warp's chunk start (entries a few slots away).
__device__ __forceinline__ uint32_t lane_gallop(const uint64_t* offs, uint32_t nq, uint32_t lo,
                                                uint64_t t) {
  uint32_t hi = nq, step = 1;
  for (;;) {
    const uint32_t p = lo + step;
    if (p >= nq) break;
    if (__ldcg(&offs[p]) > t) {
      hi = p;
      break;
    }
    lo = p;
    step <<= 1;
  }
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldcg(&offs[mid]) <= t)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// First kHead in-neighbours of every pull row as two 16-byte words loaded in
// one round (0xFFFFFFFF pads short rows).  Built once per graph.
#ifndef GM_BFS_HEAD
#define GM_BFS_HEAD 16
#endif
constexpr int kHead = GM_BFS_HEAD;  // multiple of 4
constexpr int kHeadVec = kHead / 4;
// The first kSoa in-neighbours of every pull row live slot-major (hsoa[s][v]):
// a warp probing 32 consecutive rows' slot s reads one coalesced 128-byte line
// (4 B per open row) instead of a 64-byte head line each.  Under the degree
// relabel slot 0 is a row's highest-degree neighbour, which a large frontier
// holds most of the time, so most rows cost 4 B.  The rest of the head
// (slots kSoa..kHead-1) stays row-major for one-round 16-byte loads.
constexpr int kSoa = 4;
constexpr int kAosVec = kHeadVec - 1;  // 16-byte chunks after the slot-major part

__global__ void k_build_head(const uint64_t* ptr, const uint32_t* idx, uint64_t nv, uint64_t hstride,
                             uint32_t* hsoa, uint4* head) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < nv;
       v += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = ptr[v], e = ptr[v + 1];
#pragma unroll
    for (int k = 0; k < kSoa; ++k) hsoa[k * hstride + v] = b + k < e ? idx[b + k] : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < kAosVec; ++j) {
      uint32_t h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t t = b + kSoa + 4 * j + k;
        h[k] = t < e ? idx[t] : 0xFFFFFFFFu;
      }
      head[kAosVec * v + j] = make_uint4(h[0], h[1], h[2], h[3]);
    }
  }
}

__device__ __forceinline__ void coop_push(const CoopArgs& a, int cur, uint64_t nf, uint64_t total,
                                          int32_t next_level, uint64_t gwarp, uint64_t nwarps) {
  const uint64_t* offs = a.offs[cur];
  const uint64_t* qe = a.qe[cur];
  uint32_t* qn = a.q[cur ^ 1];
  uint64_t* on = a.offs[cur ^ 1];
  uint64_t* qen = a.qe[cur ^ 1];
  uint32_t* fbn = a.fb[cur ^ 1];
  const uint32_t nq = uint32_t(nf);
  const unsigned lane = lane_id();
  // Each warp owns a contiguous edge range: one warp search for its first
  // chunk, a forward gallop for the next ones.
  const uint64_t e_lo = total * gwarp / nwarps, e_hi = total * (gwarp + 1) / nwarps;
  uint32_t ib0 = 0;
  bool first = true;
  for (uint64_t wb = e_lo; wb < e_hi; wb += 32 * kEPT) {
    const uint64_t t0 = wb + uint64_t(lane) * kEPT;
    ib0 = first ? warp_kary(offs, 0, nq, wb) : warp_forward(offs, nq, ib0, wb);
    first = false;
    uint32_t i = lane_gallop(offs, nq, ib0, t0 < e_hi ? t0 : wb);
    // 1) resolve this lane's kEPT edge slots (offsets / start pointers only)
    uint64_t re[kEPT];
    int nk = 0;
    if (t0 < e_hi) {
      uint64_t ib = __ldcg(&offs[i]);
      uint64_t inx = i + 1 < nq ? __ldcg(&offs[i + 1]) : total;
      uint64_t es = __ldcg(&qe[i]);
#pragma unroll
      for (int k = 0; k < kEPT; ++k) {
        const uint64_t t = t0 + k;
        if (t < e_hi) {
          while (t >= inx) {
            ++i;
            ib = inx;
            inx = i + 1 < nq ? __ldcg(&offs[i + 1]) : total;
            es = __ldcg(&qe[i]);
          }
          re[k] = es + (t - ib);
          nk = k + 1;
        }
      }
    }
    // 2) all column loads in flight, then all visited probes
    uint32_t vk[kEPT], visw[kEPT];
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      GM_DCHECK(k >= nk || re[k] < a.m);
      vk[k] = k < nk ? __ldg(&a.out_idx[re[k]]) : 0u;
      GM_DCHECK(vk[k] < a.n);
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) visw[k] = k < nk ? __ldcg(&a.vis[vk[k] >> 5]) : 0xFFFFFFFFu;
    // 3) claim, then one warp-aggregated append for all winners
    uint32_t we[kEPT];
    uint64_t ws[kEPT];
    unsigned won = 0;
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      we[k] = 0;
      ws[k] = 0;
      if (k < nk) {
        const uint32_t v = vk[k], bit = 1u << (v & 31u);
        if (!(visw[k] & bit) && !(atomicOr(&a.vis[v >> 5], bit) & bit)) {
          a.level[v] = a.lbase + uint32_t(next_level);
          atomicOr(&fbn[v >> 5], bit);
          won |= 1u << k;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      if ((won >> k) & 1u) {
        const uint64_t ps = __ldg(&a.out_ptr[vk[k]]), pe = __ldg(&a.out_ptr[vk[k] + 1]);
        we[k] = uint32_t(pe - ps);
        ws[k] = ps;
      }
    }
    warp_enqueue_multi<kEPT>(won, vk, we, ws, &a.ctl->qpack, qn, on, qen);
  }
}

// Probe the first 4*hv in-neighbours of row v.  Round 1 loads the slot-major
// slots 0..3 (four coalesced 4-byte loads across the warp's rows) and their
// four frontier words together; round 2 (hv > 1, no hit yet, the row goes on)
// does the same for the row-major rest of the head.  All loads of a round are
// independent -- the row's probes are not a chain of dependent loads -- and
// `examined` still counts the probes a sequential scan would make (up to and
// including the first hit).  Returns found; sets defer/rest for rows with more
// in-edges.  hv is 1 when the frontier is large (the first probes then almost
// always hit).
__device__ __forceinline__ uint32_t probe_word(const uint32_t* s_fb, uint32_t s_words,
                                               const uint32_t* fbc, uint32_t u) {
  const uint32_t w = u >> 5;
  return w < s_words ? s_fb[w] : __ldcg(&fbc[w]);
}

__device__ __forceinline__ bool coop_probe_row(const CoopArgs& a, const uint32_t* s_fb,
                                               uint32_t s_words, const uint32_t* fbc, uint32_t v,
                                               int hv, bool& defer, uint32_t& rest,
                                               unsigned long long& examined) {
  defer = false;
  rest = 0;
  {
    // hv == 1 (large frontier): slot 0 alone first -- under the degree relabel
    // it is the row's largest neighbour and the frontier almost always holds it
    const int k0 = hv == 1 ? 1 : 0;
    if (k0) {
      const uint32_t u0 = __ldg(&a.hsoa[v]);
      if (u0 == 0xFFFFFFFFu) return false;
      GM_DCHECK(u0 < a.n && v < a.nv);
      ++examined;
      if ((probe_word(s_fb, s_words, fbc, u0) >> (u0 & 31u)) & 1u) return true;
    }
    uint32_t u[kSoa], hit = 0, valid = k0;
#pragma unroll
    for (int k = 0; k < kSoa; ++k) u[k] = k >= k0 ? __ldg(&a.hsoa[k * a.hstride + v]) : 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < kSoa; ++k) {
      if (u[k] != 0xFFFFFFFFu) {
        valid |= 1u << k;
        GM_DCHECK(u[k] < a.n && v < a.nv);
        hit |= ((probe_word(s_fb, s_words, fbc, u[k]) >> (u[k] & 31u)) & 1u) << k;
      }
    }
    // slots fill from 0: the first invalid slot ends the row
    if (hit) {
      examined += __ffs(hit) - k0;  // a slot probed above is counted there
      return true;
    }
    examined += __popc(valid) - k0;
    if (valid != (1u << kSoa) - 1) return false;
  }
  if (hv > 1) {
    // the row-major rest of the head in one round of loads, probed chunk by chunk
    uint4 hh[kAosVec];
#pragma unroll
    for (int j = 0; j < kAosVec; ++j)
      hh[j] = j < hv - 1 ? __ldg(&a.head[kAosVec * v + j])
                         : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
#pragma unroll
    for (int j = 0; j < kAosVec; ++j) {
      if (j >= hv - 1) break;
      const uint4 h = hh[j];
      const uint32_t u[4] = {h.x, h.y, h.z, h.w};
      uint32_t hit = 0, valid = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (u[k] != 0xFFFFFFFFu) {
          valid |= 1u << k;
          GM_DCHECK(u[k] < a.n);
          hit |= ((probe_word(s_fb, s_words, fbc, u[k]) >> (u[k] & 31u)) & 1u) << k;
        }
      }
      if (hit) {
        examined += __ffs(hit);
        return true;
      }
      examined += __popc(valid);
      if (valid != 0xFu) return false;
    }
  }
  const uint32_t d = __ldg(&a.indeg[v]);
  const uint32_t probed = 4u * uint32_t(hv);
  defer = d > probed;
  rest = defer ? d - probed : 0u;
  return false;
}

// kBlocksPerSm: 2 (64 registers, 32 warps per SM) or 3 (40 registers, 48
// warps): the large graphs' pulls are latency-bound and gain from the warps
// (scale 28: 994 -> 1036 GTEPS); small graphs lose more on the wider grid
// barriers than they gain (scale 23: 399 -> 388).  4 blocks (32 registers)
// spills too much (scale 28: 815).
template <int kBlocksPerSm>
__global__ void __launch_bounds__(kCoopThreads, kBlocksPerSm) k_bfs_coop(CoopArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint32_t s_fb[];
  const uint64_t gtid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t gthreads = uint64_t(gridDim.x) * blockDim.x;
  const uint32_t gwarp = uint32_t(gtid >> 5), nwarps = uint32_t(gthreads >> 5);
  const unsigned lane = lane_id();
  __shared__ unsigned long long s_hdr[4], s_bc[2];
  if (gtid == 0) a.ctl->t_entry = globaltimer();
  for (;;) {
    grid.sync();
    if (threadIdx.x < 2) {
      const uint4 h = __ldcg(reinterpret_cast<const uint4*>(a.ctl->hdr) + threadIdx.x);
      s_hdr[2 * threadIdx.x] = (uint64_t(h.y) << 32) | h.x;
      s_hdr[2 * threadIdx.x + 1] = (uint64_t(h.w) << 32) | h.z;
    }
    __syncthreads();
    const unsigned flags = unsigned(s_hdr[3] >> 32);
    if (flags & kHdrDone) break;
    const int32_t it = int32_t(uint32_t(s_hdr[3])) + 1;
    const int cur = it & 1;
    const uint64_t nf = s_hdr[0];
    uint64_t mf = s_hdr[1];  // after a pull: 0 until the queue conversion counts it
    const bool pull = it == 1 ? false
                              : ((flags & kHdrPrevPull) ? nf * 24 >= a.n : double(mf) > 0.05 * double(a.m));
    // A pull over a short unvisited list finds at most that many rows, so when
    // the list is below the pull threshold the next superstep is certainly a
    // push: the pull queues what it finds (with degrees) and the push skips
    // the bitmap -> queue conversion.
    const bool pull_queues = pull && !(flags & kHdrUImplicit) && s_hdr[2] * 24 < a.n;
    if (gtid == 0 && it <= kMaxRecorded) {
      a.ctl->t_start[it - 1] = globaltimer();
      a.ctl->t_mid[it - 1] = 0;
    }
    uint32_t* fbc = a.fb[cur];
    uint32_t* fbn = a.fb[cur ^ 1];
    if (!pull) {
      if (!(flags & kHdrCurIsQueue)) {  // frontier bitmap -> queue with edge offsets
        // Two passes over the warp's words: count (vertices, edges), reserve
        // the CTA's range with one atomicAdd, then write.  (Appending per warp
        // step put one atomicAdd per ~1 vertex on the single queue counter
        // when the frontier is sparse: 30 us for 26K vertices.)
        __shared__ unsigned long long s_wbase[kCoopThreads / 32];
        const uint64_t words = (a.n + 31) / 32;
        const unsigned wib = threadIdx.x >> 5;
        // blocks of 32 consecutive words dealt round-robin over the warps:
        // 128-byte loads, and every warp gets a statistically equal share
        unsigned long long mine = 0;  // (count << kCountShift) | edges of this lane's bits
        for (uint64_t k0 = gwarp * 32; k0 < words; k0 += nwarps * 32) {
          const uint64_t wl = k0 + lane;
          const uint32_t myword = wl < words ? __ldcg(&fbc[wl]) : 0u;
          unsigned nz = __ballot_sync(0xffffffffu, myword != 0u);
          while (nz) {
            const int j = __ffs(nz) - 1;
            nz &= nz - 1;
            const uint32_t word = __shfl_sync(0xffffffffu, myword, j);
            if ((word >> lane) & 1u) {
              const uint32_t v = uint32_t((k0 + j) * 32 + lane);
              mine += (1ull << kCountShift) | (__ldg(&a.out_ptr[v + 1]) - __ldg(&a.out_ptr[v]));
            }
          }
        }
        unsigned long long wsum = mine;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        if (lane == 0) s_wbase[wib] = wsum;
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long tot = 0;
          for (unsigned w = 0; w < kCoopThreads / 32; ++w) {
            const unsigned long long t = s_wbase[w];
            s_wbase[w] = tot;
            tot += t;
          }
          const unsigned long long base = tot ? atomicAdd(&a.ctl->bpack, tot) : 0ull;
          for (unsigned w = 0; w < kCoopThreads / 32; ++w) s_wbase[w] += base;
        }
        __syncthreads();
        unsigned long long pos = s_wbase[wib];  // running (position, edge offset) of the warp
        for (uint64_t k0 = gwarp * 32; k0 < words; k0 += nwarps * 32) {
          const uint64_t wl = k0 + lane;
          const uint32_t myword = wl < words ? __ldcg(&fbc[wl]) : 0u;
          unsigned nz = __ballot_sync(0xffffffffu, myword != 0u);
          while (nz) {
            const int j = __ffs(nz) - 1;
            nz &= nz - 1;
            const uint32_t word = __shfl_sync(0xffffffffu, myword, j);
            const bool set = (word >> lane) & 1u;
            const uint32_t v = uint32_t((k0 + j) * 32 + lane);
            uint64_t ps = 0, ed = 0;
            if (set) {
              ps = __ldg(&a.out_ptr[v]);
              ed = __ldg(&a.out_ptr[v + 1]) - ps;
            }
            const unsigned long long me = set ? ((1ull << kCountShift) | ed) : 0ull;
            unsigned long long incl = me;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= unsigned(o)) incl += t;
            }
            if (set) {
              const unsigned long long ex = pos + incl - me;
              const uint32_t qp = uint32_t(ex >> kCountShift);
              GM_DCHECK(qp < a.n && v < a.n);
              a.q[cur][qp] = v;
              a.offs[cur][qp] = ex & kEdgeMask;
              a.qe[cur][qp] = ps;
            }
            pos += __shfl_sync(0xffffffffu, incl, 31);
          }
        }
        grid.sync();
        if (gtid == 0 && it <= kMaxRecorded) a.ctl->t_mid[it - 1] = globaltimer();
        // the frontier's edges, counted by the conversion (a pull no longer
        // sums the degrees of what it finds: only a following push needs them)
        if (threadIdx.x == 0) s_bc[0] = __ldcg(&a.ctl->bpack);
        __syncthreads();
        mf = s_bc[0] & kEdgeMask;
      }
      coop_push(a, cur, nf, mf, it, gwarp, nwarps);
    } else {
      // A short unvisited list probes too few words to pay for staging the
      // hot prefix of the frontier bitmap (96 KB per CTA) in shared memory.
      const bool u_implicit = flags & kHdrUImplicit;
      const uint64_t ucur_n = s_hdr[2];
      const uint32_t sw = (!u_implicit && ucur_n * 64 < a.nv) ? 0u : a.s_words;
      for (uint32_t i = threadIdx.x; i < sw; i += blockDim.x) s_fb[i] = __ldcg(&fbc[i]);
      __syncthreads();
      unsigned long long found_n = 0, found_e = 0, examined = 0;
      const int us = (flags & kHdrUsel) ? 1 : 0;
      uint32_t* unext = a.ul[us ^ 1];
      // A large frontier leaves few rows unvisited: only then is the list of
      // the remaining rows worth building for the next pull.
      const bool build_list = a.use_ulist && nf * 16 >= a.n;
      const int hv = nf * 32 >= a.n ? 1 : kHeadVec;
      if (u_implicit) {
        const uint32_t words = uint32_t((a.nv + 31) / 32);
        // Large graphs (3-CTA variant): warps claim chunks of consecutive
        // visited words from a counter (the next claim is issued before the
        // current chunk is walked, so its latency hides): one coalesced
        // visited load per chunk, and warps that draw cheap words take more
        // of them -- static dealing left ~10% of the pull's stall samples at
        // the closing barrier (scale 28: 1036 -> 1212 GTEPS).  Small graphs
        // (2-CTA variant) deal words round-robin (warp g owns g, g + nwarps,
        // ...; lanes load the visited words of the warp's next 32 in one
        // round): too few chunks per warp there to balance dynamically
        // (scale 23: 400 vs 387 GTEPS at the best chunk size).  A run-time
        // choice between the two cost the large graphs 8% (1212 -> 1150).
        constexpr bool dyn = kBlocksPerSm >= 3;
        const uint32_t step = dyn ? 1u : nwarps, span = dyn ? a.pull_chunk : 32u;
        uint32_t next = 0;  // dyn: the warp's next claimed word; else its next block
        if (dyn) {
          if (lane == 0) next = atomicAdd(&a.ctl->wcursor, span);
          next = __shfl_sync(0xffffffffu, next, 0);
        }
        for (;;) {
         uint32_t c0;
         if (dyn) {
           if (next >= words) break;
           c0 = next;
           if (lane == 0) next = atomicAdd(&a.ctl->wcursor, span);
         } else {
           c0 = gwarp + next * nwarps;
           if (c0 >= words) break;
           next += 32;
         }
         const uint32_t wl = c0 + lane * step;
         const uint32_t myvis = (lane < span && wl < words) ? __ldcg(&a.vis[wl]) : 0xFFFFFFFFu;
         unsigned open_words = __ballot_sync(0xffffffffu, myvis != 0xFFFFFFFFu);
         while (open_words) {
          const int j = __ffs(open_words) - 1;
          open_words &= open_words - 1;
          const uint32_t w = c0 + j * step;
          // L2 prefetch of the next open word's head slots (no registers held:
          // the next iteration's slot loads then hit L2 instead of DRAM)
          if (open_words && lane < 2u * kSoa) {
            const unsigned k = lane >> 1;
            if (hv > 1 || k == 0) {
              const uint32_t w2 = c0 + (__ffs(open_words) - 1) * step;
              const uint32_t* p = a.hsoa + k * a.hstride + w2 * 32 + ((lane & 1u) ? 31 : 0);
              asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            }
          }
          const uint32_t vw = __shfl_sync(0xffffffffu, myvis, j);
          const uint32_t v = w * 32 + lane;
          bool found = false, defer = false;
          uint32_t rest = 0;
          const bool open = v < a.nv && !((vw >> lane) & 1u);
          if (open) {
            found = coop_probe_row(a, s_fb, sw, fbc, v, hv, defer, rest, examined);
            if (found) a.level[v] = a.lbase + uint32_t(it);
          }
          const unsigned b = __ballot_sync(0xffffffffu, found);
          if (lane == 0 && b) {
            fbn[w] = b;  // word exclusively owned in this pass
            a.vis[w] = vw | b;
          }
          found_n += found;
          if (__any_sync(0xffffffffu, defer)) {
            const uint32_t vv = uint32_t(v);
            const uint64_t es = defer ? __ldg(&a.in_ptr[v]) + 4u * hv : 0;
            warp_enqueue_multi<1>(defer ? 1u : 0u, &vv, &rest, &es, &a.ctl->dpack, a.defq, a.defo,
                                  a.defe);
          }
          const bool keep = open && !found;
          if (build_list && __any_sync(0xffffffffu, keep))
            warp_enqueue(keep, uint32_t(v), 0, &a.ctl->upack, unext, nullptr);
         }
         if (dyn) next = __shfl_sync(0xffffffffu, next, 0);
        }
      } else {
        const uint32_t cnt = uint32_t(ucur_n);
        const uint32_t* ucur = a.ul[us];
        for (uint32_t base = gwarp * 32; base < cnt; base += nwarps * 32) {
          const uint32_t i = base + lane;
          bool found = false, defer = false, open = false;
          uint32_t rest = 0, v = 0;
          if (i < cnt) {
            v = __ldcg(&ucur[i]);
            open = !((__ldcg(&a.vis[v >> 5]) >> (v & 31u)) & 1u);
            if (open) {
              found = coop_probe_row(a, s_fb, sw, fbc, v, hv, defer, rest, examined);
              if (found) {
                const uint32_t bit = 1u << (v & 31u);
                a.level[v] = a.lbase + uint32_t(it);
                atomicOr(&fbn[v >> 5], bit);
                atomicOr(&a.vis[v >> 5], bit);
              }
            }
          }
          found_n += found;
          if (pull_queues && __any_sync(0xffffffffu, found)) {
            uint64_t ps = 0;
            uint32_t dg = 0;
            if (found) {
              ps = __ldg(&a.out_ptr[v]);
              dg = uint32_t(__ldg(&a.out_ptr[v + 1]) - ps);
            }
            warp_enqueue_multi<1>(found ? 1u : 0u, &v, &dg, &ps, &a.ctl->qpack, a.q[cur ^ 1],
                                  a.offs[cur ^ 1], a.qe[cur ^ 1]);
          }
          if (__any_sync(0xffffffffu, defer)) {
            const uint64_t es = defer ? __ldg(&a.in_ptr[v]) + 4u * hv : 0;
            warp_enqueue_multi<1>(defer ? 1u : 0u, &v, &rest, &es, &a.ctl->dpack, a.defq, a.defo,
                                  a.defe);
          }
          const bool keep = open && !found;
          if (build_list && __any_sync(0xffffffffu, keep))
            warp_enqueue(keep, v, 0, &a.ctl->upack, unext, nullptr);
        }
      }
      grid.sync();
      if (gtid == 0 && it <= kMaxRecorded) a.ctl->t_mid[it - 1] = globaltimer();
      // pass 2: edge-balanced over the deferred rows' remaining in-edges:
      // resolve the slots, put every column load in flight, then probe.
      if (threadIdx.x == 0) s_bc[1] = __ldcg(&a.ctl->dpack);
      __syncthreads();
      const unsigned long long dp = s_bc[1];
      const uint32_t ndef = uint32_t(dp >> kCountShift);
      const uint64_t total = dp & kEdgeMask;
      const uint64_t e_lo = total * gwarp / nwarps, e_hi = total * (gwarp + 1) / nwarps;
      uint32_t ib0 = 0;
      bool first = true;
      for (uint64_t wb = e_lo; wb < e_hi; wb += 32 * kEPT) {
        const uint64_t t0 = wb + uint64_t(lane) * kEPT;
        ib0 = first ? warp_kary(a.defo, 0, ndef, wb) : warp_forward(a.defo, ndef, ib0, wb);
        first = false;
        uint32_t i = lane_gallop(a.defo, ndef, ib0, t0 < e_hi ? t0 : wb);
        uint32_t rv[kEPT];
        uint64_t re[kEPT];
        int nk = 0;
        if (t0 < e_hi) {
          uint64_t ib = __ldcg(&a.defo[i]);
          uint64_t inx = i + 1 < ndef ? __ldcg(&a.defo[i + 1]) : total;
          uint64_t es = __ldcg(&a.defe[i]);
          uint32_t v = __ldcg(&a.defq[i]);
#pragma unroll
          for (int k = 0; k < kEPT; ++k) {
            const uint64_t t = t0 + k;
            rv[k] = v;
            re[k] = 0;
            if (t < e_hi) {
              while (t >= inx) {
                ++i;
                ib = inx;
                inx = i + 1 < ndef ? __ldcg(&a.defo[i + 1]) : total;
                es = __ldcg(&a.defe[i]);
                v = __ldcg(&a.defq[i]);
              }
              rv[k] = v;
              re[k] = es + (t - ib);
              nk = k + 1;
            }
          }
        }
        uint32_t u[kEPT];
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          GM_DCHECK(k >= nk || (re[k] < a.m && rv[k] < a.nv));
          u[k] = k < nk ? __ldg(&a.in_idx[re[k]]) : 0xFFFFFFFFu;
          GM_DCHECK(k >= nk || u[k] < a.n);
        }
        // rows already found (by an earlier chunk) skip their probe; this load
        // is issued alongside the column loads, off the critical path
        uint32_t done_w[kEPT];
#pragma unroll
        for (int k = 0; k < kEPT; ++k) done_w[k] = k < nk ? __ldcg(&fbn[rv[k] >> 5]) : 0xFFFFFFFFu;
        unsigned won = 0;
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          const uint32_t bit = 1u << (rv[k] & 31u);
          if (k < nk && !(done_w[k] & bit)) {
            ++examined;
            const uint32_t w = u[k] >> 5;
            const uint32_t word = w < sw ? s_fb[w] : __ldcg(&fbc[w]);
            if ((word >> (u[k] & 31u)) & 1u) {
              const uint32_t v = rv[k];
              if (!(atomicOr(&fbn[v >> 5], bit) & bit)) {
                a.level[v] = a.lbase + uint32_t(it);
                atomicOr(&a.vis[v >> 5], bit);
                ++found_n;
                won |= 1u << k;
              }
            }
          }
        }
        if (pull_queues && __any_sync(0xffffffffu, won != 0u)) {
          uint64_t ps[kEPT];
          uint32_t dg[kEPT];
#pragma unroll
          for (int k = 0; k < kEPT; ++k) {
            ps[k] = 0;
            dg[k] = 0;
            if ((won >> k) & 1u) {
              ps[k] = __ldg(&a.out_ptr[rv[k]]);
              dg[k] = uint32_t(__ldg(&a.out_ptr[rv[k] + 1]) - ps[k]);
            }
          }
          warp_enqueue_multi<kEPT>(won, rv, dg, ps, &a.ctl->qpack, a.q[cur ^ 1], a.offs[cur ^ 1],
                                   a.qe[cur ^ 1]);
        }
      }
      warp_add_u64(&a.ctl->found_n, found_n);
      warp_add_u64(&a.ctl->found_e, found_e);
      warp_add_u64(&a.ctl->examined, examined);
    }
    grid.sync();
    // finish: the consumed frontier bitmap becomes the next step's output buffer
    for (uint64_t w = gtid; w < a.words_all; w += gthreads) fbc[w] = 0u;
    if (gtid == 0) {
      Ctl* c = a.ctl;
      uint64_t nn = 0, mn = 0;
      GM_DCHECK(!pull_queues || (c->qpack >> kCountShift) == c->found_n);
      if (!pull || pull_queues) {
        nn = c->qpack >> kCountShift;
        mn = c->qpack & kEdgeMask;
        a.offs[cur ^ 1][nn] = mn;
      }
      if (pull) {
        if (!pull_queues) {
          nn = c->found_n;
          mn = c->found_e;
        }
        c->ucur = c->upack >> kCountShift;
        const bool built = a.use_ulist && nf * 16 >= a.n;
        c->u_implicit = built ? 0 : 1;
        c->usel ^= 1;
      }
      if (it <= kMaxRecorded) {
        StepRec& r = c->rec[it - 1];
        r.active = int64_t(nf);
        r.updated = int64_t(nn);
        r.edges = int64_t(pull ? c->examined : mf);
        r.examined = int64_t(c->examined);
        r.deferred = int64_t(c->dpack >> kCountShift);
        r.deferred_edges = int64_t(c->dpack & kEdgeMask);
        r.dir = pull ? kPull : kPush;
        c->t_end[it - 1] = globaltimer();
      }
      c->prev_pull = pull;
      c->cur_is_queue = !pull || pull_queues;
      c->nf = nn;
      c->mf = mn;
      c->it = it;
      c->qpack = c->dpack = c->bpack = c->upack = 0;
      c->wcursor = 0;
      c->found_n = c->found_e = c->examined = 0;
      if (nn == 0 || it >= c->max_it) c->done = 1;
      c->hdr[0] = nn;
      c->hdr[1] = mn;
      c->hdr[2] = c->ucur;
      c->hdr[3] = uint64_t(uint32_t(it)) |
                  (uint64_t((c->done ? kHdrDone : 0u) | (pull ? kHdrPrevPull : 0u) |
                            (pull && !pull_queues ? 0u : kHdrCurIsQueue) |
                            (c->u_implicit ? kHdrUImplicit : 0u) |
                            (c->usel ? kHdrUsel : 0u))
                   << 32);
      __threadfence();
    }
  }
  if (gtid == 0) a.ctl->t_exit = globaltimer();
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
    ctl->queue_out = 1;
  }
}

// SSSP prologue: push (SpMSpV over CSR(G), atomicMin per improving edge)
// while the frontier's out-edges are few; pull (SpMV over CSR(G^T), a
// run-min per row, no atomics on hot destinations) once they exceed
// m / kSsspPullDiv (one pull pass costs about as much as a push over m/6
// edges at scale 23).  Both compute, for every v,
//   min(dist[v], min over frontier u of snapshot(u) + w(u, v))
// so distances and per-superstep stats are the same either way.
constexpr uint64_t kSsspPullDiv = 6;
__global__ void k_sssp_decide(Ctl* ctl, int allow_pull) {
  if (ctl->done) return;
  const int32_t it = ++ctl->it;
  if (it <= kMaxRecorded) ctl->t_start[it - 1] = gtimer();
  ctl->dir = (allow_pull && ctl->mf * kSsspPullDiv > ctl->m_total) ? kPull : kPush;
  ctl->qpack = ctl->examined = 0;
}

// pull: frontier snapshots into msg[] before the pass, back to INF after
__global__ void k_sssp_msg(const Ctl* ctl, const uint32_t* q, const uint32_t* dq, uint32_t* msg,
                           int clear) {
  if (ctl->done || ctl->dir != kPull) return;
  const uint32_t nq = uint32_t(ctl->nf);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x)
    msg[q[i]] = clear ? 0xFFFFFFFFu : dq[i];
}

constexpr uint32_t kSsspHub = 49152;  // frontier messages of the first ids in shared memory

// Gather msg[c]: ids below H from the shared copy, the rest from L2 (.cg),
// branch-free (both loads predicated, a select picks).
__device__ __forceinline__ uint32_t msg_gather(const uint32_t* __restrict__ s_msg, uint32_t H,
                                               const uint32_t* __restrict__ msg, uint32_t c,
                                               bool valid) {
  const uint32_t hv = s_msg[min(c, H - 1)];
  uint32_t gv = 0xFFFFFFFFu;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.cg.u32 %0, [%1];\n\t}"
      : "+r"(gv)
      : "l"(msg + c), "r"(uint32_t(valid && c >= H)));
  return !valid ? 0xFFFFFFFFu : c < H ? hv : gv;
}

// pull pass: a lane takes 8 consecutive CSR(G^T) entries per step (row id,
// source and weight as vector loads, 2 KB per warp step), gathers the 8
// messages (hub ids from the shared copy of msg[0, H)), and folds a running
// min per destination row along its entries; a row's min that beats dist[row]
// lowers it (atomicMin -- a row spans lanes) and sets the row's changed bit.
// The next frontier queue is built afterwards from the changed bitmap
// (k_sssp_pull_queue), so the pass itself has no queue appends and no
// shuffles.  Each warp keeps the next step's loads in flight while it gathers
// and folds the current one.
template <typename W>
__device__ __forceinline__ void pull_load(const uint32_t* __restrict__ rowid,
                                          const uint32_t* __restrict__ idx,
                                          const W* __restrict__ wt, uint64_t nnz, uint64_t j,
                                          uint32_t (&r)[8], uint32_t (&c)[8], uint32_t (&w)[8]) {
  if (j + 8 <= nnz) {
    const uint4 r0 = __ldcs(reinterpret_cast<const uint4*>(rowid + j));
    const uint4 r1 = __ldcs(reinterpret_cast<const uint4*>(rowid + j) + 1);
    const uint4 c0 = __ldcs(reinterpret_cast<const uint4*>(idx + j));
    const uint4 c1 = __ldcs(reinterpret_cast<const uint4*>(idx + j) + 1);
    r[0] = r0.x; r[1] = r0.y; r[2] = r0.z; r[3] = r0.w;
    r[4] = r1.x; r[5] = r1.y; r[6] = r1.z; r[7] = r1.w;
    c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w;
    c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
    if constexpr (sizeof(W) == 1) {
      const uint2 wv = __ldcs(reinterpret_cast<const uint2*>(wt + j));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        w[u] = (wv.x >> (8 * u)) & 0xFFu;
        w[4 + u] = (wv.y >> (8 * u)) & 0xFFu;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) w[u] = uint32_t(wt[j + u]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool in = j + u < nnz;
      r[u] = in ? rowid[j + u] : 0xFFFFFFFFu;
      c[u] = in ? idx[j + u] : 0u;
      w[u] = in ? uint32_t(wt[j + u]) : 0u;
    }
  }
}

template <typename W>
__global__ void __launch_bounds__(kThreads, 1) k_sssp_pull(Ctl* ctl, const uint32_t* __restrict__ rowid,
                                                           const uint32_t* __restrict__ idx,
                                                           const W* __restrict__ wt, uint64_t nnz,
                                                           const uint32_t* __restrict__ msg, uint32_t H,
                                                           uint32_t* dist, uint32_t* changed) {
  if (ctl->done || ctl->dir != kPull) return;
  extern __shared__ __align__(16) uint32_t s_msg[];
  for (uint32_t i = threadIdx.x; i < H / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(s_msg)[i] = __ldcg(reinterpret_cast<const uint4*>(msg) + i);
  __syncthreads();
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 8;
  uint64_t j = t * 8;
  uint32_t r[8], c[8], w[8];
  pull_load(rowid, idx, wt, nnz, j, r, c, w);
  for (; j < nnz; j += stride) {
    uint32_t m[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) m[u] = msg_gather(s_msg, H, msg, c[u], r[u] != 0xFFFFFFFFu);
    uint32_t rn[8], cn[8], wn[8];
    pull_load(rowid, idx, wt, nnz, j + stride, rn, cn, wn);
    uint32_t row = r[0], best = 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (r[u] != row) {
        if (best != 0xFFFFFFFFu && best < dist[row] && best < atomicMin(&dist[row], best))
          atomicOr(&changed[row >> 5], 1u << (row & 31u));
        row = r[u];
        best = 0xFFFFFFFFu;
      }
      if (m[u] != 0xFFFFFFFFu) {
        const uint64_t c64 = uint64_t(m[u]) + uint64_t(w[u]);
        best = min(best, c64 >= 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(c64));
      }
    }
    if (row != 0xFFFFFFFFu && best != 0xFFFFFFFFu && best < dist[row] &&
        best < atomicMin(&dist[row], best))
      atomicOr(&changed[row >> 5], 1u << (row & 31u));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      r[u] = rn[u];
      c[u] = cn[u];
      w[u] = wn[u];
    }
  }
  if (t == 0) ctl->examined = nnz;
}

// After a pull: the changed bitmap -> next frontier queue with edge offsets.
// Two passes over the warp's words (count, then write) with one atomicAdd per
// CTA on the queue counter.
__global__ void __launch_bounds__(kThreads) k_sssp_pull_queue(Ctl* ctl, const uint32_t* changed,
                                                              uint64_t words,
                                                              const uint32_t* __restrict__ deg,
                                                              uint32_t* qn, uint64_t* offs_n) {
  if (ctl->done || ctl->dir != kPull) return;
  __shared__ unsigned long long s_wbase[kThreads / 32];
  const uint64_t gwarp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id(), wib = threadIdx.x >> 5;
  unsigned long long mine = 0;
  for (uint64_t w = gwarp; w < words; w += nwarps * 32) {
    const uint64_t wl = w + uint64_t(lane) * nwarps;
    const uint32_t word = wl < words ? __ldcg(&changed[wl]) : 0u;
    for (uint32_t b = word; b; b &= b - 1)
      mine += (1ull << kCountShift) | __ldg(&deg[wl * 32 + __ffs(b) - 1]);
  }
  unsigned long long wsum = mine;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if (lane == 0) s_wbase[wib] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (unsigned w = 0; w < kThreads / 32; ++w) {
      const unsigned long long v = s_wbase[w];
      s_wbase[w] = tot;
      tot += v;
    }
    const unsigned long long base = tot ? atomicAdd(&ctl->qpack, tot) : 0ull;
    for (unsigned w = 0; w < kThreads / 32; ++w) s_wbase[w] += base;
  }
  __syncthreads();
  // lane order within the warp: exclusive scan of the lanes' sums
  unsigned long long incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= unsigned(o)) incl += v;
  }
  unsigned long long pos = s_wbase[wib] + incl - mine;
  for (uint64_t w = gwarp; w < words; w += nwarps * 32) {
    const uint64_t wl = w + uint64_t(lane) * nwarps;
    const uint32_t word = wl < words ? __ldcg(&changed[wl]) : 0u;
    for (uint32_t b = word; b; b &= b - 1) {
      const uint32_t v = uint32_t(wl * 32 + __ffs(b) - 1);
      const uint32_t qp = uint32_t(pos >> kCountShift);
      qn[qp] = v;
      offs_n[qp] = pos & kEdgeMask;
      pos += (1ull << kCountShift) | __ldg(&deg[v]);
    }
  }
}

__global__ void k_rowid(const uint64_t* ptr, uint64_t n, uint32_t* rowid) {
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t v = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; v < n;
       v += (uint64_t(gridDim.x) * blockDim.x) >> 5)
    for (uint64_t j = ptr[v] + lane; j < ptr[v + 1]; j += 32) rowid[j] = uint32_t(v);
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
  if (ctl->done || ctl->dir != kPush) return;
  const uint32_t nq = uint32_t(ctl->nf);
  const uint64_t total = ctl->mf;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  // appends staged per warp in shared memory, published kPushCap at a time
  // (one atomicAdd on the queue counter per flush instead of one per warp step)
  __shared__ uint32_t s_qv[kThreads / 32][kPushCap], s_qd[kThreads / 32][kPushCap];
  StagedQ<kPushCap, true, false> sq{s_qv[threadIdx.x >> 5], s_qd[threadIdx.x >> 5], nullptr};
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
      sq.push(won, v, won ? deg[v] : 0, 0, &ctl->qpack, qn, offs_n, nullptr);
    }
  }
  sq.flush(&ctl->qpack, qn, offs_n, nullptr);
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

// Host driver shared by BFS and SSSP: enqueue supersteps in batches of
// kBatch, reading the device's done flag once per batch.
// A full batch (kBatch supersteps, the first one odd, so the buffer parities
// repeat) is captured once as a CUDA graph and replayed: a light superstep is
// a handful of tiny kernels, and launching them one by one from the host left
// the GPU idle ~35 us per superstep.  Superstep times come from %globaltimer
// stamps the kernels write into Ctl.
template <typename Enqueue>
int64_t run_batches(TravCache& c, cudaStream_t s, int64_t max_iters, int key, Enqueue&& step) {
  int32_t* done = c.hdone->get();
  int64_t enq = 0;
  if (c.sssp_key != key && c.sssp_exec) {
    GM_CUDA(cudaGraphExecDestroy(c.sssp_exec));
    c.sssp_exec = nullptr;
  }
  while (enq < max_iters) {
    const int64_t nb = std::min<int64_t>(kBatch, max_iters - enq);
    if (nb == kBatch) {
      if (!c.sssp_exec) {
        cudaGraph_t graph;
        const uint64_t l0 = launches_so_far();
        GM_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (int64_t b = 0; b < kBatch; ++b) step(b + 1);
        GM_CUDA(cudaStreamEndCapture(s, &graph));
        c.sssp_launches = int(launches_so_far() - l0);
        GM_CUDA(cudaGraphInstantiate(&c.sssp_exec, graph, 0));
        GM_CUDA(cudaGraphDestroy(graph));
        c.sssp_key = key;
      }
      GM_CUDA(cudaGraphLaunch(c.sssp_exec, s));
      for (int k = 0; k < c.sssp_launches; ++k) ::gm::count_launch();
      enq += kBatch;
    } else {
      for (int64_t b = 0; b < nb; ++b, ++enq) step(enq + 1);
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
  std::vector<uint64_t> t0(rec.size()), t1(rec.size());
  if (nrec > 0) {
    GM_CUDA(cudaMemcpyAsync(t0.data(), c.ctl.get()->t_start, nrec * 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaMemcpyAsync(t1.data(), c.ctl.get()->t_end, nrec * 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
  }
  for (int64_t i = 0; i < nrec; ++i) {
    const StepRec& r = rec[i];
    gm_iteration_stats st{};
    st.iteration = i + 1;
    st.active_before = r.active;
    st.messages_generated = r.active;
    st.vertices_updated = r.updated;
    const double sec = i < enqueued && t1[i] > t0[i] ? double(t1[i] - t0[i]) * 1e-9 : 0.0;
    st.spmv_seconds = sec;
    st.total_seconds = sec;
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
                                    bool out_on_device, bool collect, bool async) {
  const uint64_t n = g.n;
  if (root >= n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(n));
  // a packed count holds a vertex count <= n - 1 (the source never re-enters)
  if (n > (1ull << (64 - kCountShift)))
    fail(GM_EUSAGE, "bfs: graphs above 2^28 vertices are not supported by the packed queue");
  TravCache& c = cache(g);
  cudaStream_t s = g.stream;
  const uint64_t words = (n + 31) / 32;
  // Pull rows: on a relabeled symmetric graph only the nonzero-degree prefix
  // can ever be reached.
  const uint64_t nv = (g.relabeled && g.symmetric && g.shards == 1) ? g.nonzero_outdeg : n;
  if (!c.coop_blocks_per_sm) {
    const char* e = getenv("GM_BFS_CTAS_PER_SM");  // test hook: force a variant
    const int forced = e ? atoi(e) : 0;
    c.coop_blocks_per_sm = (forced == 2 || forced == 3) ? forced : (n > (uint64_t(1) << 24) ? 3 : 2);
  }
  const int blocks_per_sm = c.coop_blocks_per_sm;
  void* const coop_fn = blocks_per_sm == 3 ? reinterpret_cast<void*>(k_bfs_coop<3>)
                                           : reinterpret_cast<void*>(k_bfs_coop<2>);
  const uint32_t s_words = uint32_t(std::min<uint64_t>(smem_fb_words(blocks_per_sm), (nv + 31) / 32));
  const size_t smem = size_t(smem_fb_words(blocks_per_sm)) * 4;
  if (!c.level) {
    c.level.alloc(n, s);
    c.hsoa.alloc(size_t(kSoa) * (nv + 1), s);
    c.head.alloc(size_t(kAosVec) * (nv + 1), s);
    if (nv) {
      k_build_head<<<grid_for(nv, 256), 256, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), nv, nv + 1,
                                                      c.hsoa.get(), c.head.get());
      GM_LAUNCH_CHECK();
    }
    GM_CUDA(cudaFuncSetAttribute(coop_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0, dev = 0, sms = 0;
    GM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop_fn, kCoopThreads, smem));
    GM_CUDA(cudaGetDevice(&dev));
    GM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1) fail(GM_ECUDA, "bfs: cooperative kernel does not fit on an SM");
    c.coop_grid = unsigned(std::min(per_sm, blocks_per_sm) * sms);
  }
  ensure_forward(g);
  const Csr& fw = g.fwd();
  const uint32_t* perm = g.relabeled ? g.perm.get() : nullptr;
  const int32_t max_it = int32_t(std::min<int64_t>(max_iters, 0x7FFFFFFF));
  Ctl* ctl = c.ctl.get();
  // level stamps of this BFS lie in [lbase, lbase + depth bound]
  const uint64_t depth_bound = std::min<uint64_t>(uint64_t(std::max(max_it, 0)), nv) + 1;
  if (c.lbase == 0 || c.lbase + depth_bound > 0xFFFFFFFFull) {
    GM_CUDA(cudaMemsetAsync(c.level.get(), 0, n * 4, s));
    // test hook (tests/test_gpu_parity.py): the first BFS of a graph starts
    // its stamps at GM_BFS_LBASE_START, so a test reaches the 32-bit wrap
    const char* hook = c.lbase == 0 ? getenv("GM_BFS_LBASE_START") : nullptr;
    const uint64_t start = hook ? strtoull(hook, nullptr, 0) : 1;
    c.lbase = (start >= 1 && start + depth_bound <= 0xFFFFFFFFull) ? start : 1;
  }
  const uint32_t lbase = uint32_t(c.lbase);
  c.lbase += depth_bound;
  k_bfs_init<<<grid_for(words + 1, 256), 256, 0, s>>>(ctl, c.vis.get(), c.fb[0].get(), c.fb[1].get(),
                                                      words + 1, root, perm, c.q[1].get(),
                                                      c.offs[1].get(), c.qe[1].get(), fw.ptr.get(),
                                                      g.outdeg.get(), c.level.get(), lbase, n, g.m,
                                                      nv, max_it);
  GM_LAUNCH_CHECK();
  CoopArgs a{};
  a.ctl = ctl;
  a.in_ptr = g.in.ptr.get();
  a.in_idx = g.in.idx.get();
  a.out_ptr = fw.ptr.get();
  a.out_idx = fw.idx.get();
  a.deg = g.outdeg.get();
  a.indeg = g.indeg.get();
  a.head = c.head.get();
  a.hsoa = c.hsoa.get();
  a.hstride = uint32_t(nv + 1);
  a.level = c.level.get();
  a.lbase = lbase;
  a.vis = c.vis.get();
  for (int i = 0; i < 2; ++i) {
    a.fb[i] = c.fb[i].get();
    a.q[i] = c.q[i].get();
    a.offs[i] = c.offs[i].get();
    a.qe[i] = c.qe[i].get();
    a.ul[i] = c.ul[i].get();
  }
  a.defq = c.defq.get();
  a.defo = c.defo.get();
  a.defe = c.defe.get();
  a.n = n;
  a.nv = nv;
  a.m = g.m;
  a.words_all = words + 1;
  a.s_words = s_words;
  {
    const char* e = getenv("GM_BFS_ULIST");
    a.use_ulist = e ? atoi(e) : 1;
  }
  {
    // 3-CTA variant's chunk claims (the 2-CTA variant deals words statically):
    // about 8+ claims per warp, 4..32 words (128..1024 rows) each
    const uint64_t vwords = (nv + 31) / 32, warps = uint64_t(c.coop_grid) * (kCoopThreads / 32);
    a.pull_chunk = uint32_t(std::max<uint64_t>(4, std::min<uint64_t>(32, vwords / (warps * 8))));
    const char* e = getenv("GM_BFS_PULL_CHUNK");  // test / tuning hook
    if (e && atoi(e) >= 1 && atoi(e) <= 32) a.pull_chunk = uint32_t(atoi(e));
  }
  void* args[] = {&a};
  g.ktimer.begin(s, "k_bfs_coop");
  GM_CUDA(cudaLaunchCooperativeKernel(coop_fn, dim3(c.coop_grid),
                                      dim3(kCoopThreads), args, smem, s));
  g.ktimer.end(s);
  ::gm::count_launch();
  std::vector<gm_iteration_stats> stats;
  if (collect) {
    int32_t it = 0;
    GM_CUDA(cudaMemcpyAsync(&it, &ctl->it, 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const int64_t nrec = std::min<int64_t>(it, kMaxRecorded);
    std::vector<StepRec> rec(size_t(nrec > 0 ? nrec : 1));
    std::vector<uint64_t> t0(rec.size()), t1(rec.size());
    if (nrec > 0) {
      GM_CUDA(cudaMemcpyAsync(rec.data(), ctl->rec, nrec * sizeof(StepRec), cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaMemcpyAsync(t0.data(), ctl->t_start, nrec * 8, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaMemcpyAsync(t1.data(), ctl->t_end, nrec * 8, cudaMemcpyDeviceToHost, s));
    }
    GM_CUDA(cudaStreamSynchronize(s));
    std::vector<uint64_t> tm(rec.size());
    if (nrec > 0 && getenv("GM_BFS_PHASES")) {
      GM_CUDA(cudaMemcpy(tm.data(), ctl->t_mid, nrec * 8, cudaMemcpyDeviceToHost));
      uint64_t te[2];
      GM_CUDA(cudaMemcpy(te, &ctl->t_entry, 16, cudaMemcpyDeviceToHost));
      fprintf(stderr, "bfs kernel entry->step1 %.1fus, last step end->exit %.1fus, entry->exit %.1fus\n",
              double(t0[0] - te[0]) * 1e-3, double(te[1] - t1[nrec - 1]) * 1e-3,
              double(te[1] - te[0]) * 1e-3);
      for (int64_t i = 1; i < nrec; ++i)
        fprintf(stderr, "bfs gap before step %lld: %.1fus\n", (long long)(i + 1), double(t0[i] - t1[i - 1]) * 1e-3);
      for (int64_t i = 0; i < nrec; ++i)
        fprintf(stderr, "bfs step %lld dir=%d phase1=%.1fus total=%.1fus examined=%lld deferred=%lld/%lld\n",
                (long long)(i + 1), rec[i].dir, tm[i] ? double(tm[i] - t0[i]) * 1e-3 : 0.0,
                double(t1[i] - t0[i]) * 1e-3, (long long)rec[i].examined, (long long)rec[i].deferred,
                (long long)rec[i].deferred_edges);
    }
    for (int64_t i = 0; i < nrec; ++i) {
      const StepRec& r = rec[i];
      gm_iteration_stats st{};
      st.iteration = i + 1;
      st.active_before = r.active;
      st.messages_generated = r.active;
      st.vertices_updated = r.updated;
      st.spmv_seconds = double(t1[i] - t0[i]) * 1e-9;
      st.total_seconds = st.spmv_seconds;
      st.edges_processed = r.edges;
      st.direction = r.dir == kPush ? 1 : 0;
      st.bytes_algorithmic = r.dir == kPush
                                 ? int64_t(24 * r.active + 4 * r.edges + 16 * r.updated + n / 8)
                                 : int64_t(16 * nv + 4 * r.examined + 4 * r.updated + 2 * n / 8);
      stats.push_back(st);
    }
  }
  if (out) {
    int32_t* dst = out;
    const bool host_async = !out_on_device && async;  // GM_OUT_HOST_ASYNC
    if (host_async) {
      dst = static_cast<int32_t*>(g.host_async.stage(s, n * 4));
    } else if (!out_on_device) {
      if (!c.ext_out) c.ext_out.alloc(n, s);
      dst = c.ext_out.get();
    }
    if (perm && nv < n) {
      if (!c.perm_c) build_compact_output(c, perm, n, nv, s);
      // rounds of 8 callers per lane between the gathers: 4 and 8 measure the
      // same at scale 28 (2.84 ms per BFS), 16 and 32 lose occupancy (3.15, 3.49)
      k_bfs_output_nz<8><<<grid_for((n + 1023) / 1024 * 32, 256), 256, 0, s>>>(
          n, root, c.nzb.get(), c.nz_base.get(), c.perm_c.get(), c.level.get(), lbase, dst);
    } else {
      k_bfs_output<<<grid_for(n, 256), 256, 0, s>>>(n, root, perm, c.level.get(), lbase, dst);
    }
    GM_LAUNCH_CHECK();
    if (host_async)
      g.host_async.issue(s, out, n * 4);
    else if (!out_on_device)
      GM_CUDA(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, s));
  }
  if (!async) GM_CUDA(cudaStreamSynchronize(s));
  return stats;
}

std::vector<gm_iteration_stats> sssp(Graph& g, uint64_t root, int64_t max_iters, uint32_t* out,
                                     bool out_on_device, bool collect, bool async) {
  const uint64_t n = g.n;
  if (root >= n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(n));
  if (g.value_type != GM_VAL_U8 && g.value_type != GM_VAL_U32)
    fail(GM_EUSAGE, std::string("sssp: needs u8 or u32 edge weights, graph stores ") +
                        value_name(g.value_type) + " (use GM_PROG_SSSP_REF for real weights)");
  // a packed count holds a vertex count <= n - 1 (the source never re-enters)
  if (n > (1ull << (64 - kCountShift)))
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
  // pull supersteps need CSR(G^T) with its weights and a row id per entry
  const char* pe = getenv("GM_SSSP_PULL");
  const bool allow_pull = !(pe && pe[0] == '0') && g.in.nnz > 0 && g.in.val.get() != nullptr &&
                          g.in.nnz < 0xFFFFFFFFull;
  if (allow_pull) {
    if (!c.rowid) {
      c.rowid.alloc(g.in.nnz, s);
      k_rowid<<<grid_for(n * 32, 256), 256, 0, s>>>(g.in.ptr.get(), n, c.rowid.get());
      GM_LAUNCH_CHECK();
      c.msg.alloc(n + 4, s);
      const char* he = getenv("GM_SSSP_HUB");  // measurement hook: hub window
      const uint64_t hub_cap = he ? std::min<uint64_t>(kSsspHub, strtoull(he, nullptr, 10)) : kSsspHub;
      c.pull_hub = uint32_t(std::max<uint64_t>(4, std::min<uint64_t>(hub_cap, n) & ~uint64_t(3)));
      int dev = 0, sms = 0;
      GM_CUDA(cudaGetDevice(&dev));
      GM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      c.pull_grid = unsigned(sms);
      GM_CUDA(cudaFuncSetAttribute(k_sssp_pull<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(c.pull_hub) * 4));
      GM_CUDA(cudaFuncSetAttribute(k_sssp_pull<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(c.pull_hub) * 4));
    }
    GM_CUDA(cudaMemsetAsync(c.msg.get(), 0xFF, (n + 4) * 4, s));
  }
  const int32_t max_it = int32_t(std::min<int64_t>(max_iters, 0x7FFFFFFF));
  Ctl* ctl = c.ctl.get();
  k_sssp_init<<<grid_for(n, 256), 256, 0, s>>>(ctl, c.dist.get(), n, root, perm, c.q[1].get(),
                                               c.offs[1].get(), c.dq[1].get(), g.outdeg.get(), g.m,
                                               max_it);
  GM_LAUNCH_CHECK();
  const bool u8 = g.value_type == GM_VAL_U8;
  const int key = (allow_pull ? 1 : 0) | (u8 ? 2 : 0);
  const int64_t enq = run_batches(c, s, max_iters, key, [&](int64_t it) {
    const int cur = int(it & 1), nxt = cur ^ 1;
    k_sssp_decide<<<1, 1, 0, s>>>(ctl, allow_pull ? 1 : 0);
    GM_LAUNCH_CHECK();
    if (allow_pull) {
      k_sssp_msg<<<kGrid, kThreads, 0, s>>>(ctl, c.q[cur].get(), c.dq[cur].get(), c.msg.get(), 0);
      GM_LAUNCH_CHECK();
      if (u8)
        k_sssp_pull<uint8_t><<<c.pull_grid, kThreads, size_t(c.pull_hub) * 4, s>>>(
            ctl, c.rowid.get(), g.in.idx.get(), g.in.val.get(), g.in.nnz, c.msg.get(), c.pull_hub,
            c.dist.get(), c.changed.get());
      else
        k_sssp_pull<uint32_t><<<c.pull_grid, kThreads, size_t(c.pull_hub) * 4, s>>>(
            ctl, c.rowid.get(), g.in.idx.get(), reinterpret_cast<const uint32_t*>(g.in.val.get()),
            g.in.nnz, c.msg.get(), c.pull_hub, c.dist.get(), c.changed.get());
      GM_LAUNCH_CHECK();
      k_sssp_pull_queue<<<kGrid, kThreads, 0, s>>>(ctl, c.changed.get(), (n + 31) / 32,
                                                   g.outdeg.get(), c.q[nxt].get(), c.offs[nxt].get());
      GM_LAUNCH_CHECK();
      k_sssp_msg<<<kGrid, kThreads, 0, s>>>(ctl, c.q[cur].get(), c.dq[cur].get(), c.msg.get(), 1);
      GM_LAUNCH_CHECK();
    }
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
  for (auto& st : stats) {
    if (st.direction == 1)  // push: a u8/u32 weight with every col id, a snapshot per vertex
      st.bytes_algorithmic = int64_t(28 * st.active_before + 5 * st.edges_processed +
                                     20 * st.vertices_updated + n / 8);
    else  // pull: row id + col id + u8 weight per entry, msg scatter/clear, dist per row
      st.bytes_algorithmic = int64_t(9 * g.in.nnz + 8 * st.active_before + 4 * n +
                                     20 * st.vertices_updated + n / 8);
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
  }
  if (!async) GM_CUDA(cudaStreamSynchronize(s));
  return stats;
}

}  // namespace gm
