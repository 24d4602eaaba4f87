// triangle.cu -- exact triangle counting on a DAG-form graph.
//
// Reference: algo::triangle_count (include/semigraph/algorithms/triangle_count.hpp:
// 115-134) runs two supersteps: NeighborGatherProgram gives every vertex the
// ascending list of its in-neighbours (:29-63), ListIntersectProgram ships
// each list along the out-edges and the receiver counts the ids it shares with
// its own list (:68-111).  local_count[w] = sum over stored v -> w of
// |N_in(v) & N_in(w)|, and each triangle u < v < w is counted once, at w.
//
// On the GPU phase 1 is free: the rows of CSR(G^T) ARE the ascending
// in-neighbour lists (sorted by internal id; any total order intersects the
// same sets).  Phase 2 is one kernel: a warp per destination row w, lanes over
// the row's entries v; each lane intersects N_in(v) with N_in(w) by binary
// searching the shorter list's ids in the longer one.  Integer sums, so the
// per-vertex counts are exact and order independent.
//
// The DAG precondition (every stored edge src < dst in caller ids; the
// reference throws InputError pointing at DAGIFY, :118-124) is checked on the
// device first; the reported edge is the smallest violating (src, dst).
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

// Number of ids of the ascending list a[0, na) present in b[0, nb).
__device__ __forceinline__ uint64_t intersect_count(const uint32_t* __restrict__ a, uint64_t na,
                                                    const uint32_t* __restrict__ b, uint64_t nb) {
  if (na > nb) {
    const uint32_t* t = a;
    a = b;
    b = t;
    const uint64_t tn = na;
    na = nb;
    nb = tn;
  }
  uint64_t cnt = 0, lo = 0;
  for (uint64_t i = 0; i < na && lo < nb; ++i) {
    const uint32_t x = __ldg(&a[i]);
    uint64_t l = lo, h = nb;  // first position in b[lo, nb) with b >= x
    while (l < h) {
      const uint64_t mid = (l + h) >> 1;
      if (__ldg(&b[mid]) < x)
        l = mid + 1;
      else
        h = mid;
    }
    if (l < nb && __ldg(&b[l]) == x) {
      ++cnt;
      lo = l + 1;
    } else {
      lo = l;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(kTcThreads) k_tc_count(const uint64_t* __restrict__ ptr,
                                                         const uint32_t* __restrict__ idx,
                                                         uint64_t n, uint64_t* local,
                                                         unsigned long long* total) {
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long mine = 0;
  for (uint64_t w = warp; w < n; w += nwarps) {
    const uint64_t wb = ptr[w], we = ptr[w + 1];
    uint64_t c = 0;
    for (uint64_t k = wb + lane; k < we; k += 32) {
      const uint32_t v = idx[k];
      const uint64_t vb = ptr[v], ve = ptr[v + 1];
      c += intersect_count(idx + vb, ve - vb, idx + wb, we - wb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) local[w] = c;
    mine += c;
  }
  if (lane == 0 && mine) atomicAdd(total, mine);
}

}  // namespace

uint64_t triangle_count(Graph& g, uint64_t* local_host) {
  cudaStream_t s = g.stream;
  const uint64_t n = g.n;
  if (n == 0) return 0;
  const uint32_t* iperm = g.relabeled ? g.iperm.get() : nullptr;
  DevBuf<unsigned long long> ctr(2, s);
  GM_CUDA(cudaMemsetAsync(ctr.get(), 0xFF, 8, s));
  GM_CUDA(cudaMemsetAsync(ctr.get() + 1, 0, 8, s));
  const unsigned grid = grid_for(n * 32, kTcThreads);
  k_tc_check<<<grid, kTcThreads, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), n, iperm, ctr.get());
  GM_LAUNCH_CHECK();
  unsigned long long first = 0;
  GM_CUDA(cudaMemcpyAsync(&first, ctr.get(), 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (first != ~0ull)
    fail(GM_EINPUT, "triangle_count: edge " + std::to_string((first >> 32) + 1) + " -> " +
                        std::to_string((first & 0xFFFFFFFFull) + 1) +
                        " (1-based) violates src < dst; run DAGIFY preprocessing first");
  DevBuf<uint64_t> local(n, s);
  k_tc_count<<<grid, kTcThreads, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), n, local.get(),
                                         ctr.get() + 1);
  GM_LAUNCH_CHECK();
  unsigned long long total = 0;
  GM_CUDA(cudaMemcpyAsync(&total, ctr.get() + 1, 8, cudaMemcpyDeviceToHost, s));
  if (local_host) {
    DevBuf<uint64_t> ext(n, s);
    to_external(g, local.get(), ext.get(), 8);
    GM_CUDA(cudaMemcpyAsync(local_host, ext.get(), n * 8, cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
  return total;
}

}  // namespace gm
