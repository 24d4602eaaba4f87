// pagerank_hub.cu -- single-GPU normalised PageRank superstep with the hot
// sources in shared memory (the default path of gm_pagerank on one GPU).
//
// Same superstep as pagerank.cu (engine.hpp:176-189 for the BASELINE configs[0]
// program: all vertices active, a non-dangling u sends rank(u)/outdeg(u),
// receivers fold the sum, apply writes base + d*sum with base = (1-d)/N +
// d*D/N, un-messaged vertices take the empty sum), laid out for the B200's
// memory system instead of for a CSR walk:
//
// * Why: a random 4-byte gather that misses L1 costs one 32-byte L2 sector
//   request, and the chip serves ~270 G of those per second whatever the size
//   of x (tools/gather_bench.cu); shared memory serves ~1 T random loads per
//   second.  The 49,152 vertices with the most out-edges (the hubs) are the
//   sources of ~51% of all nonzeros of the scale-23 R-MAT graph, so one
//   persistent CTA per SM copies their messages into shared memory once per
//   superstep and only the tail goes to L2.  A larger hub window is slower:
//   the L1 left by the carveout holds the tail gathers' in-flight sectors
//   (tools/real_gather.py: 49,152 hubs 272 us, 57,984 hubs 488 us).
//
// * Positions: rows are stored in "position" order, not vertex order --
//   [long rows (in-degree > sell_max)][SELL-32 slices of the short rows,
//   bucketed by in-degree, descending][rows without in-edges] -- and every
//   per-row array (rank, message x, 1/outdeg, hub slot) is indexed by
//   position, so the apply + send epilogue is a coalesced store.  Column ids
//   are remapped once at build time: hub slot h in [0, H), else H + position
//   of the source.  The hubs' messages are also kept in a dense H-vector
//   (written by whoever applies a hub row), which is what the CTAs copy.
//
// * Work: chunks of ~4K nonzeros -- (a) pieces of long rows (in-degree >
//   kSellMax), 32 lanes across the row; a row split over several pieces is
//   folded in piece order by the last piece to finish (atomic ticket); (b)
//   groups of SELL-32 slices -- 32 rows of nearly equal in-degree stored
//   column-major, so each index load is one 128-byte line and a lane owns one
//   row, summing its entries in ascending source order (the reference's
//   per-row fold order, engine.hpp:59-66); (c) runs of rows without in-edges.
//   Chunk i belongs to CTA i mod G (every CTA gets the same mix) and the
//   CTA's warps claim its chunks through a shared counter, heaviest first.
//   Each warp keeps the indices of the next step and the gathers of this step
//   in flight while it sums the previous one (three-stage pipeline).  Each
//   chunk writes its dangling mass to its own slot and every CTA sums its
//   slots in chunk order, so results are bitwise reproducible run to run
//   whichever warp ran what.
//
// Algorithmic bytes/superstep are the same as the CTA kernel's:
// 4*nnz + 8*(N+1) + 16*N.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "api_internal.cuh"

namespace gm {

namespace {
constexpr int kHubWarps = 32;
constexpr int kHubThreads = kHubWarps * 32;
constexpr int kWIPT = 8;
constexpr uint32_t kStep = 32 * kWIPT;  // nonzeros (pieces) per step
constexpr uint32_t kHubCap = 49152;       // hub slots (shared memory 192 KB)
constexpr uint32_t kHubCapLarge = 24576;  // x beyond L2 (96 KB)
constexpr uint32_t kSellMax = 128;      // SELL rows: 0 < in-degree <= kSellMax
constexpr uint32_t kNoRow = 0xFFFFFFFFu;
constexpr uint32_t kNoHub = 0xFFFFFFFFu;   // hub_pos: not a hub
constexpr uint32_t kPadRow = 0xFFFFFFFEu;  // hub_pos: padding position of the last slice
constexpr uint32_t kPad = 0xFFFFFFFFu;     // column id of a padding entry
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr unsigned kInitBlocks = 296;
}  // namespace

struct PrHubCache {
  uint64_t n = 0, n_pos = 0, n_long = 0, n_slices = 0, n_lines = 0, n_in = 0;
  uint32_t H = 0, grid = 0, W = 0, n_multi = 0;
  DevBuf<uint32_t> pos_of;    // internal id -> position
  DevBuf<uint32_t> v_of_pos;  // position -> internal id (kNoRow for pads)
  DevBuf<uint32_t> hub_pos;   // position -> hub slot / kNoHub / kPadRow
  DevBuf<float> inv_pos;      // position -> 1/outdeg (0 for dangling and pads)
  // Tail messages live in xrow, indexed by "tail order": the position itself
  // while the message vector fits comfortably in L2, else the internal vertex
  // id (out-degree rank), which keeps the warm sources in few, L2-resident
  // lines once x (1 GB at scale 28) is far larger than L2.
  bool vertex_tail = false;
  DevBuf<uint32_t> xt_pos;    // position -> tail index (vertex_tail only)
  uint64_t n_xrow = 0;
  DevBuf<uint4> chunk;       // work chunks {kind, a, b, 0}; CTA b takes chunks b, b+G, ...
  uint32_t n_chunks = 0;
  DevBuf<uint32_t> long_idx;  // remapped columns of the long rows, row after row
  DevBuf<uint64_t> pc_beg;    // piece: first entry in long_idx
  DevBuf<uint32_t> pc_pos, pc_len, pc_slot;
  DevBuf<uint32_t> slot_first, slot_count;  // long rows split over several pieces
  DevBuf<float> piece_sum;
  DevBuf<unsigned> slot_ticket;
  DevBuf<uint32_t> sell_end;  // per slice: end line (exclusive)
  DevBuf<uint32_t> sell_idx;  // remapped columns, column-major slices (kPad pads)
  DevBuf<float> rank[2], xrow[2], xhub[2];
  DevBuf<float> dang;        // [max(grid + n_multi, kInitBlocks)]
  DevBuf<float> dang_chunk;  // per chunk
  DevBuf<float> scalars;
  DevBuf<unsigned> base_ticket;
  DevBuf<unsigned long long> ctr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~PrHubCache() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Branch-free gather: the shared load always runs (clamped index; a broadcast
// for tail lanes), the L2 load is predicated on the tail, a select picks.  (A
// ternary over the two loads compiles to a divergent branch per element.)
__device__ __forceinline__ float gather(const float* __restrict__ s_hub, uint32_t H,
                                        const float* __restrict__ xt, uint32_t c) {
  const float hv = s_hub[min(c, H - 1)];
  float gv = 0.0f;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.cg.f32 %0, [%1];\n\t}"
      : "+f"(gv)
      : "l"(xt + c), "r"(uint32_t(c >= H && c != kPad)));
  return c < H ? hv : gv;
}

enum : uint32_t { kChunkPiece = 0, kChunkSlices = 1, kChunkEmpty = 2 };

struct HubArgs {
  const uint4* chunk;  // {kind, a, b, 0}: piece a | slices [a, b) | positions [a, b)
  uint32_t n_chunks;
  uint32_t H;
  uint64_t n_long;        // position of the first SELL row
  const float* xhub_cur;  // [H]
  const float* xtail;     // xrow_cur - H: tail column c reads xtail[c]
  const uint32_t* long_idx;
  const uint64_t* pc_beg;
  const uint32_t* pc_pos;
  const uint32_t* pc_len;
  const uint32_t* pc_slot;
  const uint32_t* slot_first;
  const uint32_t* slot_count;
  float* piece_sum;
  unsigned* slot_ticket;
  const uint32_t* sell_end;
  const uint32_t* sell_idx;
  const float* inv_pos;
  const uint32_t* hub_pos;
  const uint32_t* xt_pos;  // position -> xrow index, or null (xrow is in position order)
  float* rank_next;
  float* xrow_next;
  float* xhub_next;
  float* scalars;  // [0] = this superstep's base (the last CTA writes the next one)
  float damping;
  float* dang_chunk;  // per chunk
  float* dang;        // [grid] per CTA, then [n_multi] split rows
  unsigned* base_ticket;  // CTAs done this superstep (the last computes the next base)
  uint32_t n_multi;
  uint64_t n;
};

struct Epi {
  float base, damping;
  uint32_t H;
  float* rank;
  float* xrow;
  float* xhub;
  // apply + send for the row at position p (iv, hs, xt prefetched)
  __device__ __forceinline__ void operator()(uint64_t p, float sum, float iv, uint32_t hs,
                                             uint64_t xt, float& dang) const {
    if (hs == kPadRow) return;
    const float r = base + damping * sum;
    const float x = r * iv;
    rank[p] = r;
    xrow[xt] = x;
    if (hs < H) xhub[hs] = x;
    if (iv == 0.0f) dang += r;
  }
};

// One piece of a long row: 32 lanes across it, lane-strided sums, fixed tree.
__device__ __forceinline__ float piece_sum_of(const uint32_t* __restrict__ col, uint32_t len,
                                              unsigned lane, const float* __restrict__ s_hub,
                                              uint32_t H, const float* __restrict__ xt) {
  float acc = 0.0f;
  uint32_t c[kWIPT];
  float v[kWIPT];
#pragma unroll
  for (int u = 0; u < kWIPT; ++u) {
    const uint32_t k = lane + 32u * u;
    c[u] = k < len ? __ldcs(&col[k]) : kPad;
  }
#pragma unroll
  for (int u = 0; u < kWIPT; ++u) v[u] = gather(s_hub, H, xt, c[u]);
#pragma unroll
  for (int u = 0; u < kWIPT; ++u) {
    const uint32_t k = kStep + lane + 32u * u;
    c[u] = k < len ? __ldcs(&col[k]) : kPad;
  }
  for (uint32_t k0 = 0; k0 < len; k0 += kStep) {
    float vn[kWIPT];
#pragma unroll
    for (int u = 0; u < kWIPT; ++u) vn[u] = gather(s_hub, H, xt, c[u]);
#pragma unroll
    for (int u = 0; u < kWIPT; ++u) {
      const uint32_t k = k0 + 2 * kStep + lane + 32u * u;
      c[u] = k < len ? __ldcs(&col[k]) : kPad;
    }
#pragma unroll
    for (int u = 0; u < kWIPT; ++u) acc += v[u];
#pragma unroll
    for (int u = 0; u < kWIPT; ++u) v[u] = vn[u];
  }
  return warp_sum(acc);
}

// Fixed-order sum of the dangling partials by a CTA of 1024 threads (k_hub_base,
// or the last CTA of k_pr_hub): thread t sums partials t, t + 1024, ..., then
// a warp tree and a tree over the 32 warps.
__device__ __forceinline__ void base_from_partials(const float* partial, uint32_t np, uint64_t n,
                                                   float damping, float* scalars) {
  __shared__ float red[32];
  float s = 0.0f;
  for (uint32_t i = threadIdx.x; i < np; i += 1024) s += __ldcg(&partial[i]);
  s = warp_sum(s);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = warp_sum(red[threadIdx.x]);
    if (threadIdx.x == 0) {
      const float nf = float(n), d = damping;
      scalars[0] = (1.0f - d) / nf + d * s / nf;
    }
  }
}

__global__ void __launch_bounds__(kHubThreads, 1) k_pr_hub(const HubArgs a) {
  extern __shared__ __align__(16) float s_hub[];
  __shared__ unsigned s_next;
  const unsigned tid = threadIdx.x, lane = tid & 31u;
  const uint32_t G = gridDim.x;
  if (tid == 0) s_next = 0;
  {  // hub messages -> shared memory (H is a multiple of 4)
    const float4* src = reinterpret_cast<const float4*>(a.xhub_cur);
    float4* dst = reinterpret_cast<float4*>(s_hub);
    for (uint32_t i = tid; i < a.H / 4; i += kHubThreads) dst[i] = __ldcg(&src[i]);
  }
  __syncthreads();
  const uint32_t H = a.H;
  const float* __restrict__ xt = a.xtail;
  const Epi epi{a.scalars[0], a.damping, H, a.rank_next, a.xrow_next, a.xhub_next};

  // The CTA's chunks are b, b + G, ...; its warps claim them in that order.
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(&s_next, 1u);
    const uint64_t ci = uint64_t(blockIdx.x) + uint64_t(__shfl_sync(0xffffffffu, k, 0)) * G;
    if (ci >= a.n_chunks) break;
    const uint4 ch = a.chunk[ci];
    float dang = 0.0f;
    if (ch.x == kChunkPiece) {
      const uint32_t p = ch.y;
      const uint32_t len = a.pc_len[p], pos = a.pc_pos[p], slot = a.pc_slot[p];
      const float iv = a.inv_pos[pos];
      const uint32_t hs = a.hub_pos[pos];
      const uint64_t xo = a.xt_pos ? a.xt_pos[pos] : pos;
      const float sum = piece_sum_of(a.long_idx + a.pc_beg[p], len, lane, s_hub, H, xt);
      if (slot == kNoSlot) {
        if (lane == 0) epi(pos, sum, iv, hs, xo, dang);
      } else {
        // a row split over several pieces: the last to finish folds them in order
        const uint32_t f = a.slot_first[slot], cnt = a.slot_count[slot];
        unsigned last = 0;
        if (lane == 0) {
          a.piece_sum[p] = sum;
          __threadfence();
          last = atomicAdd(&a.slot_ticket[slot], 1u) == cnt - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          float t = 0.0f;
          for (uint32_t i = lane; i < cnt; i += 32) t += __ldcg(&a.piece_sum[f + i]);
          t = warp_sum(t);
          if (lane == 0) {
            a.slot_ticket[slot] = 0;
            float dl = 0.0f;
            epi(pos, t, iv, hs, xo, dl);
            a.dang[G + slot] = dl;
          }
        }
      }
    } else if (ch.x == kChunkSlices) {
      // SELL-32 slices [sa, sb): one flat stream of 128-byte lines
      const uint32_t sa = ch.y, sb = ch.z;
      const uint32_t qa = sa ? a.sell_end[sa - 1] : 0, qb = a.sell_end[sb - 1];
      // slice ends, 32 at a time: lane j holds the end line of slice sbase + j
      uint32_t sbase = sa, ends = sa + lane < sb ? a.sell_end[sa + lane] : 0xFFFFFFFFu;
      uint32_t sl = sa;
      uint32_t e_cur = __shfl_sync(0xffffffffu, ends, 0);
      uint64_t p_cur = a.n_long + uint64_t(sl) * 32u + lane;
      float iv_cur = a.inv_pos[p_cur];
      uint32_t hs_cur = a.hub_pos[p_cur];
      uint64_t xt_cur = a.xt_pos ? a.xt_pos[p_cur] : p_cur;
      const uint32_t* __restrict__ col = a.sell_idx + lane;
      float acc = 0.0f;
      uint32_t c[kWIPT];
      float v[kWIPT];
#pragma unroll
      for (int u = 0; u < kWIPT; ++u) c[u] = qa + u < qb ? __ldcs(&col[uint64_t(qa + u) * 32u]) : kPad;
#pragma unroll
      for (int u = 0; u < kWIPT; ++u) v[u] = gather(s_hub, H, xt, c[u]);
#pragma unroll
      for (int u = 0; u < kWIPT; ++u) {
        const uint32_t q = qa + kWIPT + u;
        c[u] = q < qb ? __ldcs(&col[uint64_t(q) * 32u]) : kPad;
      }
      for (uint32_t q0 = qa; q0 < qb; q0 += kWIPT) {
        float vn[kWIPT];
#pragma unroll
        for (int u = 0; u < kWIPT; ++u) vn[u] = gather(s_hub, H, xt, c[u]);
#pragma unroll
        for (int u = 0; u < kWIPT; ++u) {
          const uint32_t q = q0 + 2 * kWIPT + u;
          c[u] = q < qb ? __ldcs(&col[uint64_t(q) * 32u]) : kPad;
        }
#pragma unroll
        for (int u = 0; u < kWIPT; ++u) {
          acc += v[u];
          if (q0 + u + 1 == e_cur) {  // slice sl ends with this line (warp-uniform)
            epi(p_cur, acc, iv_cur, hs_cur, xt_cur, dang);
            acc = 0.0f;
            ++sl;
            if (sl - sbase == 32) {
              sbase = sl;
              ends = sl + lane < sb ? a.sell_end[sl + lane] : 0xFFFFFFFFu;
            }
            e_cur = __shfl_sync(0xffffffffu, ends, sl - sbase);
            p_cur += 32;
            if (sl < sb) {
              iv_cur = a.inv_pos[p_cur];
              hs_cur = a.hub_pos[p_cur];
              xt_cur = a.xt_pos ? a.xt_pos[p_cur] : p_cur;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kWIPT; ++u) v[u] = vn[u];
      }
    } else {
      // rows without in-edges, positions [a, b): the empty sum
      for (uint64_t p0 = ch.y; p0 < ch.z; p0 += 4 * 32) {
        float iv[4];
        uint32_t hs[4];
        uint64_t xo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t p = p0 + lane + 32u * u;
          iv[u] = p < ch.z ? a.inv_pos[p] : 0.0f;
          hs[u] = p < ch.z ? a.hub_pos[p] : kPadRow;
          xo[u] = (a.xt_pos && p < ch.z) ? a.xt_pos[p] : p;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) epi(p0 + lane + 32u * u, 0.0f, iv[u], hs[u], xo[u], dang);
      }
    }
    dang = warp_sum(dang);
    if (lane == 0) a.dang_chunk[ci] = dang;
  }
  // this CTA's dangling mass: its chunks' partials in chunk order
  __syncthreads();
  if (tid < 32) {
    float t = 0.0f;
    for (uint64_t ci = blockIdx.x + uint64_t(lane) * G; ci < a.n_chunks; ci += 32ull * G)
      t += __ldcg(&a.dang_chunk[ci]);
    t = warp_sum(t);
    if (lane == 0) a.dang[blockIdx.x] = t;
  }
  // The last CTA to finish turns the partials into the next superstep's base
  // (the work of k_hub_base, same fixed-order sum, so the same bits): one
  // launch per superstep fewer (every CTA captured this superstep's base
  // when it started, so overwriting it now is safe).
  __shared__ bool s_last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(a.base_ticket, 1u) == G - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    base_from_partials(a.dang, G + a.n_multi, a.n, a.damping, a.scalars);
    if (tid == 0) *a.base_ticket = 0;
  }
}

// base = (1-d)/N + d*D/N from fixed-order partials (one CTA of 1024 threads).
__global__ void __launch_bounds__(1024) k_hub_base(const float* partial, uint32_t np, uint64_t n,
                                                   double damping, float* scalars) {
  base_from_partials(partial, np, n, float(damping), scalars);
}

// Initial state: rank 1/N at every vertex position (0 at pads), x = rank/outdeg,
// hub messages; per-block dangling partials of the initial ranks.
__global__ void k_hub_init(uint64_t n_pos, uint64_t n, const float* __restrict__ inv_pos,
                           const uint32_t* __restrict__ hub_pos,
                           const uint32_t* __restrict__ xt_pos, uint32_t H, float* rank,
                           float* rank_other, float* xrow, float* xhub, float* partial) {
  __shared__ float red[32];
  const float r0 = 1.0f / float(n);
  float d = 0.0f;
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n_pos;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t hs = hub_pos[p];
    const bool pad = hs == kPadRow;
    const float r = pad ? 0.0f : r0, iv = inv_pos[p], x = r * iv;
    rank[p] = r;
    rank_other[p] = 0.0f;
    if (!pad) xrow[xt_pos ? xt_pos[p] : p] = x;
    if (hs < H) xhub[hs] = x;
    if (!pad && iv == 0.0f) d += r;
  }
  d = warp_sum(d);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = d;
  __syncthreads();
  if (threadIdx.x < 32) {
    d = warp_sum(threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f);
    if (threadIdx.x == 0) partial[blockIdx.x] = d;
  }
}

// vertices_updated of a stats superstep (rule S7): positions with in-edges
// whose rank changed bitwise (pads hold 0 in both buffers).
__global__ void k_hub_count(uint64_t n_in, const float* old_rank, const float* new_rank,
                            unsigned long long* ctr) {
  unsigned long long c = 0;
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n_in;
       p += uint64_t(gridDim.x) * blockDim.x)
    c += __float_as_uint(old_rank[p]) != __float_as_uint(new_rank[p]);
  warp_add_u64(ctr, c);
}

__global__ void k_hub_out(uint64_t n, const uint32_t* __restrict__ pos_of,
                          const float* __restrict__ rank_pos, float* __restrict__ out) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    out[v] = rank_pos[pos_of[v]];
}

// ---- build ----

__global__ void k_hub_meta(uint64_t n_pos, const uint32_t* __restrict__ v_of_pos,
                           const uint32_t* __restrict__ outdeg, float* __restrict__ inv_pos) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n_pos;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = v_of_pos[p];
    const uint32_t od = v == kNoRow ? 0u : outdeg[v];
    inv_pos[p] = od ? 1.0f / float(od) : 0.0f;  // as k_pr_init (pagerank.cu)
  }
}

// column id: hub slot, else H + tail index (position, or the vertex itself
// when tail_of is null)
__device__ __forceinline__ uint32_t remap(uint32_t src, const uint32_t* __restrict__ slot_of,
                                          const uint32_t* __restrict__ tail_of, uint32_t H) {
  const uint32_t h = slot_of[src];
  return h != kNoHub ? h : H + (tail_of ? tail_of[src] : src);
}

// long rows: a warp per row copies its remapped sources
__global__ void k_hub_fill_long(uint64_t n_long, const uint32_t* __restrict__ v_of_pos,
                                const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
                                const uint64_t* __restrict__ long_ptr,
                                const uint32_t* __restrict__ slot_of,
                                const uint32_t* __restrict__ pos_of, uint32_t H,
                                uint32_t* __restrict__ out) {
  const uint64_t lane = threadIdx.x & 31u;
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / 32; i < n_long;
       i += uint64_t(gridDim.x) * blockDim.x / 32) {
    const uint32_t row = v_of_pos[i];
    const uint64_t j = ptr[row], d = ptr[row + 1] - j, o = long_ptr[i];
    for (uint64_t k = lane; k < d; k += 32) out[o + k] = remap(idx[j + k], slot_of, pos_of, H);
  }
}

// SELL rows: a thread per row writes its remapped sources down its lane of the
// slice's lines (pads were set to kPad)
__global__ void k_hub_fill_sell(uint64_t n_sell, uint64_t n_long, const uint32_t* __restrict__ v_of_pos,
                                const uint32_t* __restrict__ sell_end,
                                const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
                                const uint32_t* __restrict__ slot_of,
                                const uint32_t* __restrict__ pos_of, uint32_t H,
                                uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n_sell;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t row = v_of_pos[n_long + e];
    if (row == kNoRow) continue;
    const uint64_t sl = e / 32, line0 = sl ? sell_end[sl - 1] : 0;
    const uint64_t j = ptr[row], d = ptr[row + 1] - j;
    uint32_t* o = out + line0 * 32u + (e % 32);
    for (uint64_t k = 0; k < d; ++k) o[k * 32u] = remap(idx[j + k], slot_of, pos_of, H);
  }
}

template <typename T>
void upload(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.alloc(h.size() + 1, s);
  if (!h.empty())
    GM_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

PrHubCache& hub_cache(Graph& g) {
  if (g.prhub) return *g.prhub;
  g.prhub = std::unique_ptr<PrHubCache, void (*)(PrHubCache*)>(new PrHubCache(),
                                                              [](PrHubCache* p) { delete p; });
  PrHubCache& c = *g.prhub;
  cudaStream_t s = g.stream;
  const uint64_t n = g.n, nnz = g.in.nnz;
  c.n = n;
  int dev = 0, sms = 0;
  GM_CUDA(cudaGetDevice(&dev));
  GM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  c.grid = uint32_t(sms);
  c.W = c.grid * kHubWarps;
  std::vector<uint64_t> ptr(n + 1);
  std::vector<uint32_t> outdeg(n);
  GM_CUDA(cudaMemcpyAsync(ptr.data(), g.in.ptr.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaMemcpyAsync(outdeg.data(), g.outdeg.get(), n * 4, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (n >= kPadRow) fail(GM_EENGINE, "pagerank: graph too large for the hub kernel");

  // hubs: the vertices with the most out-edges (ties: lower id first)
  std::vector<uint32_t> slot_of(n, kNoHub);
  uint64_t nz = 0;
  for (uint64_t v = 0; v < n; ++v) nz += outdeg[v] != 0;
  // Hub window: 49,152 slots (192 KB) while x is L2-sized; 24,576 (96 KB)
  // beyond that, where the tail gathers miss L2 and the L1 that the smaller
  // copy leaves holds their sectors (scale 28, ms per superstep by window:
  // 49,152 28.3; 32,768 22.0; 24,576 21.7; 16,384 21.8; 8,192 22.5; the
  // CTA-tile kernel 24.0).  GM_PR_HUBCAP overrides (measurement hook).
  const char* hc = getenv("GM_PR_HUBCAP");
  const uint64_t cap = hc ? std::min<uint64_t>(kHubCap, std::max<uint64_t>(4, strtoull(hc, nullptr, 10)))
                          : (n * 4 <= (64ull << 20) ? kHubCap : kHubCapLarge);
  const uint64_t nh = std::min<uint64_t>(cap, nz);
  {
    std::vector<uint32_t> order;
    order.reserve(nz);
    for (uint64_t v = 0; v < n; ++v)
      if (outdeg[v]) order.push_back(uint32_t(v));
    auto more = [&](uint32_t x, uint32_t y) {
      return outdeg[x] != outdeg[y] ? outdeg[x] > outdeg[y] : x < y;
    };
    if (nh < order.size()) std::nth_element(order.begin(), order.begin() + nh, order.end(), more);
    std::sort(order.begin(), order.begin() + nh, more);
    for (uint64_t h = 0; h < nh; ++h) slot_of[order[h]] = uint32_t(h);
  }
  c.H = uint32_t(std::max<uint64_t>(4, (nh + 3) & ~uint64_t(3)));

  // positions: [long rows][SELL slices][rows without in-edges]
  const uint32_t sell_max = kSellMax;
  std::vector<uint32_t> longs, zeros;
  std::vector<uint64_t> bucket(sell_max + 1, 0);
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t d = ptr[r + 1] - ptr[r];
    if (d == 0)
      zeros.push_back(uint32_t(r));
    else if (d > sell_max)
      longs.push_back(uint32_t(r));
    else
      ++bucket[d];
  }
  std::vector<uint64_t> start(sell_max + 1, 0);
  uint64_t nshort = 0;
  for (uint32_t d = sell_max; d >= 1; --d) {
    start[d] = nshort;
    nshort += bucket[d];
  }
  const uint64_t nslices = (nshort + 31) / 32;
  c.n_long = longs.size();
  c.n_slices = nslices;
  c.n_in = c.n_long + nslices * 32;
  c.n_pos = c.n_in + zeros.size();
  std::vector<uint32_t> v_of_pos(c.n_pos, kNoRow), pos_of(n), sdeg(nslices * 32, 0);
  for (uint64_t i = 0; i < longs.size(); ++i) v_of_pos[i] = longs[i];
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t d = ptr[r + 1] - ptr[r];
    if (d >= 1 && d <= sell_max) {
      const uint64_t e = start[d]++;
      v_of_pos[c.n_long + e] = uint32_t(r);
      sdeg[e] = uint32_t(d);
    }
  }
  for (uint64_t i = 0; i < zeros.size(); ++i) v_of_pos[c.n_in + i] = zeros[i];
  for (uint64_t p = 0; p < c.n_pos; ++p)
    if (v_of_pos[p] != kNoRow) pos_of[v_of_pos[p]] = uint32_t(p);
  {
    const char* e = getenv("GM_PR_TAIL");
    c.vertex_tail = e ? std::string(e) == "vertex" : n * 4 > (48ull << 20);
  }
  c.n_xrow = c.vertex_tail ? n : c.n_pos;
  if (c.vertex_tail) upload(c.xt_pos, v_of_pos, s);  // pads hold kNoRow, never written
  std::vector<uint32_t> hub_pos(c.n_pos);
  for (uint64_t p = 0; p < c.n_pos; ++p)
    hub_pos[p] = v_of_pos[p] == kNoRow ? kPadRow : slot_of[v_of_pos[p]];
  std::vector<uint32_t> send(nslices);
  uint64_t lines = 0;
  for (uint64_t sl = 0; sl < nslices; ++sl) {
    lines += sdeg[sl * 32];
    send[sl] = uint32_t(lines);
  }
  c.n_lines = lines;
  std::vector<uint64_t> long_ptr(c.n_long + 1, 0);
  for (uint64_t i = 0; i < c.n_long; ++i)
    long_ptr[i + 1] = long_ptr[i] + (ptr[longs[i] + 1] - ptr[longs[i]]);
  if (lines >= 0xFFFFFFF0ull || c.H + c.n_pos >= kPad || c.H + n >= kPad || nslices >= 0xFFFFFFF0ull)
    fail(GM_EENGINE, "pagerank: graph too large for the hub kernel");

  // Work chunks, heaviest first: pieces of <= kPieceMax nonzeros of the long
  // rows (a longer row is split, its pieces folded in order by the last to
  // finish), groups of slices of ~kGroupLines lines, runs of kEmptyRun rows
  // without in-edges.  Chunk i goes to CTA i mod G, so every CTA gets the same
  // mix, and the CTA's 32 warps claim its chunks dynamically.
  constexpr uint64_t kPieceMax = 2048, kGroupLines = 32, kEmptyRun = 512;
  std::vector<uint4> chunks;
  std::vector<uint32_t> pc_pos, pc_len, pc_slot, slot_first, slot_count;
  std::vector<uint64_t> pc_beg;
  for (uint64_t i = 0; i < c.n_long; ++i) {
    const uint64_t beg = long_ptr[i], end = long_ptr[i + 1];
    const uint64_t cnt = (end - beg + kPieceMax - 1) / kPieceMax;
    const uint32_t slot = cnt > 1 ? uint32_t(slot_first.size()) : kNoSlot;
    if (cnt > 1) {
      slot_first.push_back(uint32_t(pc_len.size()));
      slot_count.push_back(uint32_t(cnt));
    }
    for (uint64_t k = 0; k < cnt; ++k) {
      const uint64_t b0 = beg + k * kPieceMax;
      chunks.push_back(make_uint4(kChunkPiece, uint32_t(pc_len.size()), 0, 0));
      pc_pos.push_back(uint32_t(i));
      pc_beg.push_back(b0);
      pc_len.push_back(uint32_t(std::min(kPieceMax, end - b0)));
      pc_slot.push_back(slot);
    }
  }
  // heaviest pieces first (stable: a split row's pieces stay in order)
  std::stable_sort(chunks.begin(), chunks.end(), [&](const uint4& x, const uint4& y) {
    return pc_len[x.y] > pc_len[y.y];
  });
  for (uint64_t sl = 0; sl < nslices;) {
    uint64_t e = sl, l = 0;
    while (e < nslices && (e == sl || l + sdeg[e * 32] <= kGroupLines)) l += sdeg[32 * e++];
    chunks.push_back(make_uint4(kChunkSlices, uint32_t(sl), uint32_t(e), 0));
    sl = e;
  }
  for (uint64_t z = 0; z < zeros.size(); z += kEmptyRun)
    chunks.push_back(make_uint4(kChunkEmpty, uint32_t(c.n_in + z),
                                uint32_t(c.n_in + std::min<uint64_t>(zeros.size(), z + kEmptyRun)), 0));
  if (chunks.size() >= 0xFFFFFFF0ull) fail(GM_EENGINE, "pagerank: too many work chunks");
  c.n_chunks = uint32_t(chunks.size());
  c.n_multi = uint32_t(slot_first.size());

  // device arrays
  upload(c.pos_of, pos_of, s);
  upload(c.v_of_pos, v_of_pos, s);
  upload(c.hub_pos, hub_pos, s);
  upload(c.chunk, chunks, s);
  c.dang_chunk.alloc(chunks.size() + 1, s);
  upload(c.pc_beg, pc_beg, s);
  upload(c.pc_pos, pc_pos, s);
  upload(c.pc_len, pc_len, s);
  upload(c.pc_slot, pc_slot, s);
  upload(c.slot_first, slot_first, s);
  upload(c.slot_count, slot_count, s);
  upload(c.sell_end, send, s);
  c.piece_sum.alloc(pc_len.size() + 1, s);
  c.slot_ticket.alloc(c.n_multi + 1, s);
  c.slot_ticket.zero(s);
  c.inv_pos.alloc(c.n_pos + 1, s);
  k_hub_meta<<<grid_for(c.n_pos, 256), 256, 0, s>>>(c.n_pos, c.v_of_pos.get(), g.outdeg.get(),
                                                    c.inv_pos.get());
  GM_LAUNCH_CHECK();
  {
    DevBuf<uint32_t> slot_d;
    upload(slot_d, slot_of, s);
    DevBuf<uint64_t> long_ptr_d;
    upload(long_ptr_d, long_ptr, s);
    c.long_idx.alloc(long_ptr[c.n_long] + 1, s);
    if (c.n_long) {
      k_hub_fill_long<<<grid_for(c.n_long * 32, 256), 256, 0, s>>>(
          c.n_long, c.v_of_pos.get(), g.in.ptr.get(), g.in.idx.get(), long_ptr_d.get(),
          slot_d.get(), c.vertex_tail ? nullptr : c.pos_of.get(), c.H, c.long_idx.get());
      GM_LAUNCH_CHECK();
    }
    c.sell_idx.alloc(lines * 32 + 1, s);
    GM_CUDA(cudaMemsetAsync(c.sell_idx.get(), 0xFF, (lines * 32 + 1) * 4, s));
    if (nslices) {
      k_hub_fill_sell<<<grid_for(nslices * 32, 256), 256, 0, s>>>(
          nslices * 32, c.n_long, c.v_of_pos.get(), c.sell_end.get(), g.in.ptr.get(),
          g.in.idx.get(), slot_d.get(), c.vertex_tail ? nullptr : c.pos_of.get(), c.H,
          c.sell_idx.get());
      GM_LAUNCH_CHECK();
    }
    GM_CUDA(cudaStreamSynchronize(s));
  }
  for (int b = 0; b < 2; ++b) {
    c.rank[b].alloc(c.n_pos + 1, s);
    c.xrow[b].alloc(c.n_xrow + 1, s);
    c.xhub[b].alloc(c.H, s);
    c.xhub[b].zero(s);
  }
  c.dang.alloc(std::max<uint64_t>(kInitBlocks, uint64_t(c.grid) + c.n_multi) + 1, s);
  c.scalars.alloc(4, s);
  c.base_ticket.alloc(1, s);
  c.base_ticket.zero(s);
  c.ctr.alloc(4, s);
  GM_CUDA(cudaEventCreate(&c.e0));
  GM_CUDA(cudaEventCreate(&c.e1));
  GM_CUDA(cudaFuncSetAttribute(k_pr_hub, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(c.H) * 4));
  GM_CUDA(cudaStreamSynchronize(s));
  return c;
}

}  // namespace

// The hub path serves every whole-graph superstep on one GPU; beyond an
// L2-sized message vector it runs with the smaller hub window (kHubCapLarge),
// which beats the CTA-tile kernel of pagerank.cu at scale 28 (21.7 vs 24.0 ms
// per superstep; with the full 192 KB window it had lost, 26.6-28.3 ms).
// GM_PR_HUB=0/1 forces either path; the CTA-tile kernel keeps serving the
// row-sharded supersteps.
bool pagerank_hub_enabled(const Graph& g) {
  if (g.n == 0 || g.in.nnz == 0) return false;
  const char* e = getenv("GM_PR_HUB");
  if (e && e[0] == '0') return false;
  return true;
}

std::vector<gm_iteration_stats> pagerank_hub(Graph& g, double damping, int64_t iters, float* out,
                                             bool out_on_device, bool collect, bool async) {
  std::vector<gm_iteration_stats> stats;
  PrHubCache& c = hub_cache(g);
  cudaStream_t s = g.stream;
  const uint64_t n = g.n;
  const float d = float(damping);
  int cur = 0;
  k_hub_init<<<kInitBlocks, 256, 0, s>>>(c.n_pos, n, c.inv_pos.get(), c.hub_pos.get(),
                                         c.vertex_tail ? c.xt_pos.get() : nullptr, c.H,
                                         c.rank[0].get(), c.rank[1].get(), c.xrow[0].get(),
                                         c.xhub[0].get(), c.dang.get());
  GM_LAUNCH_CHECK();
  k_hub_base<<<1, 1024, 0, s>>>(c.dang.get(), kInitBlocks, n, damping, c.scalars.get());
  GM_LAUNCH_CHECK();
  for (int64_t it = 1; it <= iters; ++it) {
    if (collect) GM_CUDA(cudaEventRecord(c.e0, s));
    HubArgs a;
    a.chunk = c.chunk.get();
    a.n_chunks = c.n_chunks;
    a.H = c.H;
    a.n_long = c.n_long;
    a.xhub_cur = c.xhub[cur].get();
    a.xtail = c.xrow[cur].get() - c.H;
    a.long_idx = c.long_idx.get();
    a.pc_beg = c.pc_beg.get();
    a.pc_pos = c.pc_pos.get();
    a.pc_len = c.pc_len.get();
    a.pc_slot = c.pc_slot.get();
    a.slot_first = c.slot_first.get();
    a.slot_count = c.slot_count.get();
    a.piece_sum = c.piece_sum.get();
    a.slot_ticket = c.slot_ticket.get();
    a.sell_end = c.sell_end.get();
    a.sell_idx = c.sell_idx.get();
    a.inv_pos = c.inv_pos.get();
    a.hub_pos = c.hub_pos.get();
    a.xt_pos = c.vertex_tail ? c.xt_pos.get() : nullptr;
    a.rank_next = c.rank[cur ^ 1].get();
    a.xrow_next = c.xrow[cur ^ 1].get();
    a.xhub_next = c.xhub[cur ^ 1].get();
    a.scalars = c.scalars.get();
    a.damping = d;
    a.dang_chunk = c.dang_chunk.get();
    a.dang = c.dang.get();
    a.base_ticket = c.base_ticket.get();
    a.n_multi = c.n_multi;
    a.n = n;
    g.ktimer.begin(s, "k_pr_hub");
    k_pr_hub<<<c.grid, kHubThreads, size_t(c.H) * 4, s>>>(a);
    g.ktimer.end(s);
    GM_LAUNCH_CHECK();
    cur ^= 1;
    if (!collect) continue;
    GM_CUDA(cudaEventRecord(c.e1, s));
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
    k_hub_count<<<grid_for(c.n_in, 256), 256, 0, s>>>(c.n_in, c.rank[cur ^ 1].get(),
                                                     c.rank[cur].get(), c.ctr.get());
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
    DevBuf<float> internal(n, s);
    k_hub_out<<<grid_for(n, 256), 256, 0, s>>>(n, c.pos_of.get(), c.rank[cur].get(), internal.get());
    GM_LAUNCH_CHECK();
    if (out_on_device) {
      to_external(g, internal.get(), out, 4);
    } else {
      DevBuf<float> ext(n, s);
      to_external(g, internal.get(), ext.get(), 4);
      GM_CUDA(cudaMemcpyAsync(out, ext.get(), n * 4, cudaMemcpyDeviceToHost, s));
    }
  }
  if (!async) GM_CUDA(cudaStreamSynchronize(s));
  return stats;
}

}  // namespace gm
