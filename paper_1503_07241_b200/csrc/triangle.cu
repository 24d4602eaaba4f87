// triangle.cu -- exact triangle counting on a DAG-form graph.
//
// Reference: algo::triangle_count (include/semigraph/algorithms/triangle_count.hpp:
// 115-134) runs two supersteps: NeighborGatherProgram gives every vertex the
// ascending list of its in-neighbours (:29-63), ListIntersectProgram ships
// each list along the out-edges and the receiver counts the ids it shares with
// its own list (:68-111).  local_count[w] = sum over stored v -> w of
// |N_in(v) & N_in(w)|: each triangle a < b < c (caller ids) is counted once,
// at its largest vertex c.
//
// The id orientation the reference uses leaves hubs with in-lists of 10^5
// entries, which makes per-edge list intersection badly imbalanced on a GPU.
// The count is a property of the undirected graph, so the GPU lists every
// triangle once under the DEGREE orientation instead (Schank & Wagner's
// forward algorithm): an edge points from lower to higher (degree, id) rank,
// out-lists N+(u) then stay short (~sqrt(m)), and each triangle is found
// exactly once as u -> v, u -> x, v -> x.  The per-vertex counts of the
// reference orientation are recovered by crediting each listed triangle to
// its largest caller id, which is exactly the vertex the reference counts it
// at.  Integer sums, so totals and local counts are exact.
//
// Phase 1 (the reference's gather superstep) = building CSR+ of the degree
// orientation: one radix sort of the m oriented keys.  Phase 2 = k_tc_list: a
// warp per vertex u, lanes over v in N+(u), each lane walking N+(v) and
// binary-searching N+(u) for every x.
//
// The DAG precondition (every stored edge src < dst in caller ids; the
// reference throws InputError pointing at DAGIFY, :118-124) is checked on the
// device first; the reported edge is the smallest violating (src, dst).
#include <cub/cub.cuh>

#include "api_internal.cuh"

namespace gm {
namespace {

constexpr unsigned kTcThreads = 256;

__global__ void k_tc_check(const uint64_t* ptr, const uint32_t* idx, uint64_t n,
                           const uint32_t* iperm, unsigned long long* first) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t w = warp; w < n; w += nwarps) {
    const uint32_t cw = iperm ? iperm[w] : uint32_t(w);
    for (uint64_t k = ptr[w] + lane; k < ptr[w + 1]; k += 32) {
      const uint32_t v = idx[k];
      const uint32_t cv = iperm ? iperm[v] : v;
      if (cv >= cw) atomicMin(first, (unsigned long long)cv << 32 | cw);
    }
  }
}

// rank(x) = (undirected degree, internal id); an edge points up the ranking.
__device__ __forceinline__ bool rank_less(uint32_t a, uint32_t b, const uint32_t* deg) {
  const uint32_t da = deg[a], db = deg[b];
  return da != db ? da < db : a < b;
}

// Oriented key (lower rank << nb | higher rank) of every stored entry, and the
// out-degree of each vertex in the degree orientation.
__global__ void k_tc_orient(const uint64_t* ptr, const uint32_t* idx, uint64_t n, unsigned nb,
                            const uint32_t* deg, uint64_t* keys, uint32_t* plus_deg) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t w = warp; w < n; w += nwarps) {
    for (uint64_t k = ptr[w] + lane; k < ptr[w + 1]; k += 32) {
      const uint32_t v = idx[k];
      const uint32_t lo = rank_less(v, uint32_t(w), deg) ? v : uint32_t(w);
      const uint32_t hi = lo == v ? uint32_t(w) : v;
      keys[k] = (uint64_t(lo) << nb) | hi;
      atomicAdd(&plus_deg[lo], 1u);
    }
  }
}

__global__ void k_tc_deg(const uint32_t* indeg, const uint32_t* outdeg, uint64_t n, uint32_t* deg) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    deg[v] = indeg[v] + outdeg[v];
}

__global__ void k_tc_widen(const uint32_t* in, uint64_t n, uint64_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__global__ void k_tc_low(const uint64_t* keys, uint64_t m, uint64_t mask, uint32_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(keys[i] & mask);
}


// Triangle listing over CSR+ (rows = lower-rank endpoint u, N+(u) ascending):
// every triangle u < v < x (rank order) is found once, as x in N+(u) & N+(v)
// for v in N+(u).  The work is the wedge count W = sum over (u, v) of |N+(v)|
// (4.4e9 at scale 20), so the membership test must be cheap: N+(u) goes into
// a shared-memory hash set (open addressing, x + 1 stored, 0 = empty; at
// least twice as many slots as entries) and every lane probes the set for
// the x it loaded from N+(v) -- ~1-2 shared reads per wedge instead of a
// binary search with a dependent global load per step.  Two kernels by
// |N+(u)|: a warp per u with a warp-private 256-slot table (|N+(u)| <= 128),
// and a CTA per u with a table of up to kTcBigSlots slots; both claim their
// u's from a counter.  Longer lists (rare under the degree orientation: 666
// at scale 20) fall back to a binary search of N+(u) in global memory.
// kLocal credits each triangle to its largest caller id.
// Most probes miss (wedges that close no triangle), so a direct-mapped bit
// filter of N+(u) in front of the table answers them with one shared load
// and no probe loop (ncu of the table-only version: 120 instructions per 32
// wedges, stalled on the probe loop's dependent compares and branches).
constexpr unsigned kTcSmallMax = 128, kTcSmallSlots = 512, kTcSmallFilter = 128;  // words
constexpr unsigned kTcBigSlots = 16384;                                         // 64 KB
constexpr unsigned kTcBigFilter = 2048;                                          // 8 KB
constexpr unsigned kTcBigMax = kTcBigSlots / 4;

__device__ __forceinline__ uint32_t tc_hash(uint32_t x, uint32_t mask) {
  return (x * 0x9E3779B1u >> 7) & mask;
}
__device__ __forceinline__ uint32_t tc_fbit(uint32_t x) { return x * 0x85EBCA6Bu >> 11; }

__device__ __forceinline__ void tc_insert(uint32_t* tab, uint32_t mask, uint32_t* filt,
                                          uint32_t fmask, uint32_t x) {
  uint32_t h = tc_hash(x, mask);
  while (atomicCAS(&tab[h], 0u, x + 1u) != 0u) h = (h + 1) & mask;
  const uint32_t b = tc_fbit(x);
  atomicOr(&filt[(b >> 5) & fmask], 1u << (b & 31u));
}

__device__ __forceinline__ bool tc_member(const uint32_t* tab, uint32_t mask, const uint32_t* filt,
                                          uint32_t fmask, uint32_t x) {
  const uint32_t b = tc_fbit(x);
  if (!((filt[(b >> 5) & fmask] >> (b & 31u)) & 1u)) return false;
  uint32_t h = tc_hash(x, mask);
  for (;;) {
    const uint32_t t = tab[h];
    if (t == x + 1u) return true;
    if (t == 0u) return false;
    h = (h + 1) & mask;
  }
}

template <bool kLocal>
__device__ __forceinline__ void tc_credit(uint32_t u, uint32_t v, uint32_t x, const uint32_t* iperm,
                                          unsigned long long* local) {
  if constexpr (kLocal) {
    const uint32_t cu = iperm ? iperm[u] : u, cv = iperm ? iperm[v] : v, cx = iperm ? iperm[x] : x;
    atomicAdd(&local[max(cu, max(cv, cx))], 1ull);
  }
}

// Probe N+(v) = pi[vb, ve) against the hash set: lane takes entries lane,
// lane + step, ...; kTcRound entries' loads in flight per round (one load per
// probe round had left the probes waiting on global latency).
constexpr int kTcRound = 8;
template <bool kLocal>
__device__ __forceinline__ void tc_probe_list(const uint32_t* __restrict__ pi, uint64_t vb,
                                              uint64_t ve, unsigned lane, unsigned step,
                                              const uint32_t* tab, uint32_t mask,
                                              const uint32_t* filt, uint32_t fmask, uint32_t u,
                                              uint32_t v, const uint32_t* iperm,
                                              unsigned long long* local, unsigned long long& mine) {
  const uint32_t* __restrict__ lst = pi + vb;  // 32-bit indexing inside the list
  const uint32_t len = uint32_t(ve - vb);
  for (uint32_t k0 = lane; k0 < len; k0 += kTcRound * step) {
    uint32_t x[kTcRound];
#pragma unroll
    for (int q = 0; q < kTcRound; ++q) x[q] = k0 + q * step < len ? __ldg(&lst[k0 + q * step]) : ~0u;
#pragma unroll
    for (int q = 0; q < kTcRound; ++q) {
      if (x[q] != ~0u && tc_member(tab, mask, filt, fmask, x[q])) {
        ++mine;
        tc_credit<kLocal>(u, v, x[q], iperm, local);
      }
    }
  }
}

// A warp per u with 2 <= |N+(u)| <= kTcSmallMax.
template <bool kLocal>
__global__ void __launch_bounds__(kTcThreads) k_tc_small(const uint64_t* __restrict__ pp,
                                                         const uint32_t* __restrict__ pi, uint64_t n,
                                                         unsigned* claim, const uint32_t* iperm,
                                                         unsigned long long* local,
                                                         unsigned long long* total) {
  __shared__ uint32_t s_tab[kTcThreads / 32][kTcSmallSlots];
  __shared__ uint32_t s_filt[kTcThreads / 32][kTcSmallFilter];
  const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  uint32_t* tab = s_tab[w];
  uint32_t* filt = s_filt[w];
  constexpr uint32_t mask = kTcSmallSlots - 1, fmask = kTcSmallFilter - 1;
  for (unsigned i = lane; i < kTcSmallSlots; i += 32) tab[i] = 0u;
  for (unsigned i = lane; i < kTcSmallFilter; i += 32) filt[i] = 0u;
  __syncwarp();
  unsigned long long mine = 0;
  constexpr unsigned kStep = 32;  // u's per claim
  for (;;) {
    uint64_t u0 = 0;
    if (lane == 0) u0 = uint64_t(atomicAdd(claim, kStep)) ;
    u0 = __shfl_sync(0xffffffffu, u0, 0);
    if (u0 >= n) break;
    for (uint64_t u = u0; u < min(n, u0 + kStep); ++u) {
      const uint64_t ub = pp[u];
      const uint32_t nu = uint32_t(pp[u + 1] - ub);
      if (nu < 2 || nu > kTcSmallMax) continue;
      for (uint32_t j = lane; j < nu; j += 32) tc_insert(tab, mask, filt, fmask, __ldg(&pi[ub + j]));
      __syncwarp();
      for (uint32_t j = 0; j < nu; ++j) {
        const uint32_t v = __ldg(&pi[ub + j]);
        const uint64_t vb = pp[v], ve = pp[v + 1];
        tc_probe_list<kLocal>(pi, vb, ve, lane, 32, tab, mask, filt, fmask, uint32_t(u), v, iperm, local,
                              mine);
      }
      __syncwarp();
      for (uint32_t j = lane; j < nu; j += 32) {  // clear the slots and bits this u used
        const uint32_t x = __ldg(&pi[ub + j]);
        uint32_t h = tc_hash(x, mask);
        while (tab[h] != x + 1u) h = (h + 1) & mask;
        tab[h] = 0u;
        filt[(tc_fbit(x) >> 5) & fmask] = 0u;
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane == 0 && mine) atomicAdd(total, mine);
}

// First position in b[0, nb) with b >= x (b ascending).
__device__ __forceinline__ uint32_t lower_bound(const uint32_t* __restrict__ b, uint32_t nb,
                                                uint32_t x) {
  uint32_t l = 0, h = nb;
  while (l < h) {
    const uint32_t mid = (l + h) >> 1;
    if (__ldg(&b[mid]) < x)
      l = mid + 1;
    else
      h = mid;
  }
  return l;
}

// A CTA per u with |N+(u)| > kTcSmallMax: the table sized to >= 2 |N+(u)|
// slots (power of two); lists above kTcBigMax search N+(u) in global memory.
// The u's with long lists (|N+(u)| > kTcSmallMax), for k_tc_big to claim.
__global__ void k_tc_biglist(const uint64_t* pp, uint64_t n, uint32_t* list, unsigned* cnt) {
  for (uint64_t u0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~31ull; u0 < n;
       u0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = u0 + (threadIdx.x & 31u);
    const bool big = u < n && pp[u + 1] - pp[u] > kTcSmallMax;
    const unsigned b = __ballot_sync(0xffffffffu, big);
    if (!b) continue;
    unsigned base = 0;
    if ((threadIdx.x & 31u) == 0) base = atomicAdd(cnt, unsigned(__popc(b)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (big) list[base + __popc(b & ((1u << (threadIdx.x & 31u)) - 1u))] = uint32_t(u);
  }
}

template <bool kLocal>
__global__ void __launch_bounds__(kTcThreads) k_tc_big(const uint64_t* __restrict__ pp,
                                                       const uint32_t* __restrict__ pi,
                                                       const uint32_t* __restrict__ list,
                                                       const unsigned* nlist, unsigned* claim,
                                                       const uint32_t* iperm,
                                                       unsigned long long* local,
                                                       unsigned long long* total) {
  extern __shared__ uint32_t s_big[];  // kTcBigSlots table words, then kTcBigFilter filter words
  uint32_t* s_filt = s_big + kTcBigSlots;
  __shared__ uint64_t s_u;
  const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  constexpr unsigned kWarps = kTcThreads / 32;
  unsigned long long mine = 0;
  for (unsigned i = threadIdx.x; i < kTcBigSlots + kTcBigFilter; i += kTcThreads) s_big[i] = 0u;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned i = atomicAdd(claim, 1u);
      s_u = i < *nlist ? uint64_t(list[i]) : ~0ull;
    }
    __syncthreads();
    const uint64_t u = s_u;
    if (u == ~0ull) break;
    const uint64_t ub = pp[u];
    const uint32_t nu = uint32_t(pp[u + 1] - ub);
    const bool in_smem = nu <= kTcBigMax;
    uint32_t slots = 512, fwords = 128;
    while (slots < 4 * nu && slots < kTcBigSlots) slots <<= 1;
    while (fwords * 32 < 16 * nu && fwords < kTcBigFilter) fwords <<= 1;
    const uint32_t mask = slots - 1, fmask = fwords - 1;
    if (in_smem) {
      for (uint32_t j = threadIdx.x; j < nu; j += kTcThreads)
        tc_insert(s_big, mask, s_filt, fmask, __ldg(&pi[ub + j]));
    }
    __syncthreads();
    for (uint32_t j = w; j < nu; j += kWarps) {
      const uint32_t v = __ldg(&pi[ub + j]);
      const uint64_t vb = pp[v], ve = pp[v + 1];
      if (in_smem) {
        tc_probe_list<kLocal>(pi, vb, ve, lane, 32, s_big, mask, s_filt, fmask, uint32_t(u), v, iperm,
                              local, mine);
      } else {
        for (uint64_t k = vb + lane; k < ve; k += 32) {
          const uint32_t x = __ldg(&pi[k]);
          const uint32_t pos = lower_bound(pi + ub, nu, x);
          if (pos < nu && __ldg(&pi[ub + pos]) == x) {
            ++mine;
            tc_credit<kLocal>(uint32_t(u), v, x, iperm, local);
          }
        }
      }
    }
    __syncthreads();
    if (in_smem) {
      for (uint32_t i = threadIdx.x; i < slots; i += kTcThreads) s_big[i] = 0u;
      for (uint32_t i = threadIdx.x; i < fwords; i += kTcThreads) s_filt[i] = 0u;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane == 0 && mine) atomicAdd(total, mine);
}

}  // namespace

uint64_t triangle_count(Graph& g, uint64_t* local_host) {
  cudaStream_t s = g.stream;
  const uint64_t n = g.n, m = g.in.nnz;
  if (n == 0) return 0;
  const uint32_t* iperm = g.relabeled ? g.iperm.get() : nullptr;
  DevBuf<unsigned long long> ctr(2, s);
  GM_CUDA(cudaMemsetAsync(ctr.get(), 0xFF, 8, s));
  GM_CUDA(cudaMemsetAsync(ctr.get() + 1, 0, 8, s));
  const unsigned wgrid = grid_for(n * 32, kTcThreads);
  k_tc_check<<<wgrid, kTcThreads, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), n, iperm, ctr.get());
  GM_LAUNCH_CHECK();
  unsigned long long first = 0;
  GM_CUDA(cudaMemcpyAsync(&first, ctr.get(), 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (first != ~0ull)
    fail(GM_EINPUT, "triangle_count: edge " + std::to_string((first >> 32) + 1) + " -> " +
                        std::to_string((first & 0xFFFFFFFFull) + 1) +
                        " (1-based) violates src < dst; run DAGIFY preprocessing first");
  DevBuf<unsigned long long> local(local_host ? n : 0, s);
  if (local_host) local.zero(s);
  if (m) {
    // Phase 1: CSR+ of the degree orientation.
    const unsigned nb = g.nb;
    DevBuf<uint32_t> deg(n, s), plus(n, s);
    plus.zero(s);
    k_tc_deg<<<grid_for(n, 256), 256, 0, s>>>(g.indeg.get(), g.outdeg.get(), n, deg.get());
    GM_LAUNCH_CHECK();
    DevBuf<uint64_t> keys(m, s);
    k_tc_orient<<<wgrid, kTcThreads, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), n, nb, deg.get(),
                                              keys.get(), plus.get());
    GM_LAUNCH_CHECK();
    {
      DevBuf<uint64_t> k2(m, s);
      cub::DoubleBuffer<uint64_t> db(keys.get(), k2.get());
      size_t tmp = 0;
      GM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, int64_t(m), 0, int(2 * nb), s));
      DevBuf<uint8_t> t(tmp, s);
      GM_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, db, int64_t(m), 0, int(2 * nb), s));
      if (db.Current() != keys.get()) keys.swap(k2);
    }
    DevBuf<uint64_t> pp(n + 1, s);
    GM_CUDA(cudaMemsetAsync(pp.get(), 0, 8, s));
    k_tc_widen<<<grid_for(n, 256), 256, 0, s>>>(plus.get(), n, pp.get() + 1);
    GM_LAUNCH_CHECK();
    {
      size_t tmp = 0;
      GM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, pp.get() + 1, pp.get() + 1, int64_t(n), s));
      DevBuf<uint8_t> t(tmp, s);
      GM_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, pp.get() + 1, pp.get() + 1, int64_t(n), s));
    }
    DevBuf<uint32_t> pi(m, s);
    k_tc_low<<<grid_for(m, 256), 256, 0, s>>>(keys.get(), m, (uint64_t(1) << nb) - 1, pi.get());
    GM_LAUNCH_CHECK();
    keys.reset();
    // Phase 2: list every triangle once (short lists: a warp per u; long
    // lists: a CTA per u), u's claimed from counters.
    DevBuf<unsigned> claims(3, s);
    claims.zero(s);
    DevBuf<uint32_t> biglist(n + 1, s);
    k_tc_biglist<<<grid_for(n, 256), 256, 0, s>>>(pp.get(), n, biglist.get(), claims.get() + 2);
    GM_LAUNCH_CHECK();
    int dev = 0, sms = 0;
    GM_CUDA(cudaGetDevice(&dev));
    GM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t big_smem = (kTcBigSlots + kTcBigFilter) * 4;
    auto big = local_host ? k_tc_big<true> : k_tc_big<false>;
    GM_CUDA(cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, int(big_smem)));
    (local_host ? k_tc_small<true> : k_tc_small<false>)<<<unsigned(sms) * 8, kTcThreads, 0, s>>>(
        pp.get(), pi.get(), n, claims.get(), iperm, local.get(), ctr.get() + 1);
    GM_LAUNCH_CHECK();
    big<<<unsigned(sms) * 3, kTcThreads, big_smem, s>>>(pp.get(), pi.get(), biglist.get(),
                                                        claims.get() + 2, claims.get() + 1, iperm,
                                                        local.get(), ctr.get() + 1);
    GM_LAUNCH_CHECK();
  }
  unsigned long long total = 0;
  GM_CUDA(cudaMemcpyAsync(&total, ctr.get() + 1, 8, cudaMemcpyDeviceToHost, s));
  if (local_host) {
    // local[] is indexed by caller id already (credited through iperm)
    GM_CUDA(cudaMemcpyAsync(local_host, local.get(), n * 8, cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
  return total;
}

}  // namespace gm
