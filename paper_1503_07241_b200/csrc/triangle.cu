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

// Triangle listing over CSR+ (rows = lower-rank endpoint, ascending ids).
// kLocal credits each triangle to its largest caller id.
template <bool kLocal>
__global__ void __launch_bounds__(kTcThreads) k_tc_list(const uint64_t* __restrict__ pp,
                                                        const uint32_t* __restrict__ pi,
                                                        uint64_t n, const uint32_t* iperm,
                                                        unsigned long long* local,
                                                        unsigned long long* total) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long mine = 0;
  for (uint64_t u = warp; u < n; u += nwarps) {
    const uint64_t ub = pp[u];
    const uint32_t nu = uint32_t(pp[u + 1] - ub);
    if (nu < 2) continue;
    const uint32_t* U = pi + ub;
    for (uint32_t j = lane; j < nu; j += 32) {
      const uint32_t v = __ldg(&U[j]);
      const uint64_t vb = pp[v], ve = pp[v + 1];
      uint32_t lo = 0;  // x ascending: the search window only moves right
      for (uint64_t k = vb; k < ve && lo < nu; ++k) {
        const uint32_t x = __ldg(&pi[k]);
        const uint32_t pos = lo + lower_bound(U + lo, nu - lo, x);
        if (pos < nu && __ldg(&U[pos]) == x) {
          ++mine;
          if (kLocal) {
            const uint32_t cu = iperm ? iperm[u] : uint32_t(u);
            const uint32_t cv = iperm ? iperm[v] : v;
            const uint32_t cx = iperm ? iperm[x] : x;
            const uint32_t top = max(cu, max(cv, cx));
            atomicAdd(&local[top], 1ull);
          }
          lo = pos + 1;
        } else {
          lo = pos;
        }
      }
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
    // Phase 2: list every triangle once.
    if (local_host)
      k_tc_list<true><<<wgrid, kTcThreads, 0, s>>>(pp.get(), pi.get(), n, iperm, local.get(),
                                                   ctr.get() + 1);
    else
      k_tc_list<false><<<wgrid, kTcThreads, 0, s>>>(pp.get(), pi.get(), n, iperm, nullptr,
                                                    ctr.get() + 1);
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
