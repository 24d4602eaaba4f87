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
#include <cub/device/device_radix_sort.cuh>

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
constexpr uint32_t kHubCap = 49152;     // hub slots (shared memory 192 KB)
constexpr uint32_t kSellMax = 128;      // SELL rows: 0 < in-degree <= kSellMax
constexpr uint32_t kNoRow = 0xFFFFFFFFu;
constexpr uint32_t kNoHub = 0xFFFFFFFFu;   // hub_pos: not a hub
constexpr uint32_t kPadRow = 0xFFFFFFFEu;  // hub_pos: padding position of the last slice
constexpr uint32_t kPad = 0xFFFFFFFFu;     // column id of a padding entry
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr unsigned kInitBlocks = 296;
// Propagation-blocked tail (GM_PR_PB): see the block comment above k_pb_scatter.
constexpr uint32_t kPbThreads = 512;   // pass 2 (k_pb_bucket)
constexpr uint32_t kPbScThreads = 1024;  // pass 1 (k_pb_scatter)
constexpr uint32_t kPbGroup = 8;  // pass-1 entries per thread step (one 16-byte index load)
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
  DevBuf<unsigned long long> ctr;
  uint64_t n_count = 0;  // positions counted by vertices_updated (rows with in-edges)
  // Propagation-blocked tail (pb): the tail entries of rows with in-degree <=
  // pb_big leave the hub kernel; per round, pass 1 (k_pb_scatter) writes their
  // messages into bins in (chunk, bucket) order and pass 2 (k_pb_bucket) folds
  // every bucket's bins into ytail in shared memory.
  bool pb = false;
  uint32_t pb_cw = 0, pb_C = 0, pb_cap = 0, pb_big = 0;
  uint64_t pb_tail = 0;
  std::vector<uint32_t> pb_round_items, pb_round_buckets;  // per round + 1: first item / bucket
  std::vector<uint64_t> pb_round_base;                      // per round: first padded bin index
  DevBuf<uint16_t> pb_src;   // padded bin order: source offset in the chunk window
  DevBuf<uint16_t> pb_perm;  // padded bin order: slot in the bucket's destination order
  DevBuf<float> pb_bins;     // one round of bins
  DevBuf<uint4> pb_items;    // pass-1 items {chunk, begin, end, 0} (padded indices)
  DevBuf<uint2> pb_bucket;   // {first position, end position}
  DevBuf<uint2> pb_runs;     // [bucket][chunk] {padded start, length}
  DevBuf<uint32_t> pb_tptr;  // [n_pos + 1] tail entries before each position (destination order)
  DevBuf<float> ytail;       // [n_pos] tail sum per position
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
  const float* scalars;
  float damping;
  float* dang_chunk;  // per chunk
  float* dang;        // [grid] per CTA, then [n_multi] split rows
  const float* ytail;  // [n_pos] or null
};

struct Epi {
  float base, damping;
  uint32_t H;
  float* rank;
  float* xrow;
  float* xhub;
  const float* ytail;  // propagation-blocked tail sums, or null
  // apply + send for the row at position p (iv, hs, xt prefetched)
  __device__ __forceinline__ void operator()(uint64_t p, float sum, float iv, uint32_t hs,
                                             uint64_t xt, float& dang) const {
    if (hs == kPadRow) return;
    if (ytail) sum += __ldcg(&ytail[p]);
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
  const Epi epi{a.scalars[0], a.damping, H, a.rank_next, a.xrow_next, a.xhub_next, a.ytail};

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
}

// base = (1-d)/N + d*D/N from fixed-order partials (one CTA).
__global__ void __launch_bounds__(1024) k_hub_base(const float* partial, uint32_t np, uint64_t n,
                                                   double damping, float* scalars) {
  __shared__ float red[32];
  float s = 0.0f;
  for (uint32_t i = threadIdx.x; i < np; i += 1024) s += partial[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = warp_sum(red[threadIdx.x]);
    if (threadIdx.x == 0) {
      const float nf = float(n), d = float(damping);
      scalars[0] = (1.0f - d) / nf + d * s / nf;
    }
  }
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

// Entries the hub kernel keeps: all of a row with in-degree > big, else the
// hub sources only when the tail is propagation-blocked (big = 0: keep all).
__device__ __forceinline__ bool hub_keeps(uint32_t src, uint64_t deg, uint32_t big,
                                          const uint32_t* __restrict__ slot_of) {
  return big == 0 || deg > big || slot_of[src] != kNoHub;
}

// long rows: a warp per row copies its kept, remapped sources
__global__ void k_hub_fill_long(uint64_t n_long, const uint32_t* __restrict__ v_of_pos,
                                const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
                                const uint64_t* __restrict__ long_ptr,
                                const uint32_t* __restrict__ slot_of,
                                const uint32_t* __restrict__ pos_of, uint32_t H, uint32_t big,
                                uint32_t* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / 32; i < n_long;
       i += uint64_t(gridDim.x) * blockDim.x / 32) {
    const uint32_t row = v_of_pos[i];
    const uint64_t j = ptr[row], d = ptr[row + 1] - j;
    uint64_t o = long_ptr[i];
    for (uint64_t k0 = 0; k0 < d; k0 += 32) {
      const uint64_t k = k0 + lane;
      const uint32_t src = k < d ? idx[j + k] : 0u;
      const bool keep = k < d && hub_keeps(src, d, big, slot_of);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) out[o + __popc(m & ((1u << lane) - 1u))] = remap(src, slot_of, pos_of, H);
      o += __popc(m);
    }
  }
}

// SELL rows: a thread per row writes its kept, remapped sources down its lane
// of the slice's lines (pads were set to kPad)
__global__ void k_hub_fill_sell(uint64_t n_sell, uint64_t n_long, const uint32_t* __restrict__ v_of_pos,
                                const uint32_t* __restrict__ sell_end,
                                const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
                                const uint32_t* __restrict__ slot_of,
                                const uint32_t* __restrict__ pos_of, uint32_t H, uint32_t big,
                                uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n_sell;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t row = v_of_pos[n_long + e];
    if (row == kNoRow) continue;
    const uint64_t sl = e / 32, line0 = sl ? sell_end[sl - 1] : 0;
    const uint64_t j = ptr[row], d = ptr[row + 1] - j;
    uint32_t* o = out + line0 * 32u + (e % 32);
    uint64_t w = 0;
    for (uint64_t k = 0; k < d; ++k) {
      const uint32_t src = idx[j + k];
      if (hub_keeps(src, d, big, slot_of)) o[(w++) * 32u] = remap(src, slot_of, pos_of, H);
    }
  }
}

// ---- propagation-blocked tail ----
//
// Why: the hub kernel's tail gathers (one random 4-byte x[src] per entry) run
// at the L1TEX's ~1 distinct line per SM cycle (~270 G/s, tools/gather_bench.cu;
// the TMA unit is slower still, tools/tma_gather_bench.cu).  Propagation
// blocking (Beamer et al., IPDPS'17) turns them into streams: the tail entries
// are stored once, at build, in *bin order* -- (round, source chunk, destination
// bucket, destination, source) -- and every superstep
//   pass 1 (k_pb_scatter): a CTA per piece of a (round, chunk) segment stages
//     the chunk's window of x (CW positions) in shared memory and writes
//     bins[i] = window[src16[i]]: a 2-byte read and a 4-byte write per entry,
//     both sequential;
//   pass 2 (k_pb_bucket): a CTA per destination bucket (a position range with
//     <= cap tail entries) reads its runs of bins, one per chunk, scatters them
//     into shared memory in destination order (perm16, 2 bytes per entry) and
//     folds each row in ascending source position: ytail[p], deterministic.
// The hub kernel keeps the hub entries (shared memory) and the whole of every
// row with in-degree > big, and adds ytail[p] in its epilogue.  Rounds split
// the buckets so one round's bins stay L2-resident between the two passes.

__global__ void k_pb_deg(uint64_t n, const uint64_t* __restrict__ ptr,
                         const uint32_t* __restrict__ idx, const uint32_t* __restrict__ slot_of,
                         uint32_t big, uint32_t* __restrict__ kd, uint32_t* __restrict__ td) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = ptr[r], d = ptr[r + 1] - j;
    uint32_t h = 0;
    if (d > big) {
      h = uint32_t(d);
    } else {
      for (uint64_t k = 0; k < d; ++k) h += slot_of[idx[j + k]] != kNoHub;
    }
    kd[r] = h;
    td[r] = uint32_t(d - h);
  }
}

// tail entries of row r, as (position of r) << pbits | position of the source
__global__ void k_pb_key2(uint64_t n, const uint64_t* __restrict__ ptr,
                          const uint32_t* __restrict__ idx, const uint32_t* __restrict__ slot_of,
                          const uint32_t* __restrict__ pos_of, const uint64_t* __restrict__ toff,
                          uint32_t big, unsigned pbits, uint64_t* __restrict__ key2) {
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t r = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / 32; r < n;
       r += uint64_t(gridDim.x) * blockDim.x / 32) {
    const uint64_t j = ptr[r], d = ptr[r + 1] - j;
    if (d == 0 || d > big) continue;
    const uint64_t pr = uint64_t(pos_of[r]) << pbits;
    uint64_t o = toff[r];
    for (uint64_t k0 = 0; k0 < d; k0 += 32) {
      const uint64_t k = k0 + lane;
      const uint32_t src = k < d ? idx[j + k] : 0u;
      const bool tail = k < d && slot_of[src] == kNoHub;
      const unsigned m = __ballot_sync(0xffffffffu, tail);
      if (tail) key2[o + __popc(m & ((1u << lane) - 1u))] = pr | pos_of[src];
      o += __popc(m);
    }
  }
}

struct PbKey {
  unsigned pbits, cbits;
  uint32_t cw;
  __device__ __forceinline__ uint64_t make(uint32_t round, uint32_t pr, uint32_t pu) const {
    const uint32_t c = pu / cw;
    return (uint64_t(round) << (cbits + pbits + 16)) | (uint64_t(c) << (pbits + 16)) |
           (uint64_t(pr) << 16) | (pu - c * cw);
  }
  __device__ __forceinline__ uint32_t round(uint64_t k) const { return uint32_t(k >> (cbits + pbits + 16)); }
  __device__ __forceinline__ uint32_t chunk(uint64_t k) const {
    return uint32_t(k >> (pbits + 16)) & ((1u << cbits) - 1u);
  }
  __device__ __forceinline__ uint32_t pr(uint64_t k) const {
    return uint32_t(k >> 16) & uint32_t((1ull << pbits) - 1u);
  }
};

__global__ void k_pb_key1(uint64_t m, const uint64_t* __restrict__ key2, unsigned pbits,
                          const uint32_t* __restrict__ bucket_of_pos,
                          const uint32_t* __restrict__ round_of_bucket, PbKey pk,
                          uint64_t* __restrict__ key1, uint32_t* __restrict__ val) {
  const uint64_t mask = (1ull << pbits) - 1u;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = key2[i];
    const uint32_t pr = uint32_t(k >> pbits), pu = uint32_t(k & mask);
    key1[i] = pk.make(round_of_bucket[bucket_of_pos[pr]], pr, pu);
    val[i] = uint32_t(i);
  }
}

__global__ void k_pb_count(uint64_t m, const uint64_t* __restrict__ key1, PbKey pk, uint32_t C,
                           const uint32_t* __restrict__ bucket_of_pos, uint32_t* __restrict__ cnt) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = key1[e];
    atomicAdd(&cnt[uint64_t(bucket_of_pos[pk.pr(k)]) * C + pk.chunk(k)], 1u);
  }
}

__global__ void k_pb_place(uint64_t m, const uint64_t* __restrict__ key1,
                           const uint32_t* __restrict__ val, PbKey pk, uint32_t C,
                           const int64_t* __restrict__ delta,
                           const uint32_t* __restrict__ bucket_of_pos,
                           const uint2* __restrict__ bucket, const uint32_t* __restrict__ tptr,
                           uint16_t* __restrict__ src16, uint16_t* __restrict__ perm16) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = key1[e];
    const uint64_t pe = uint64_t(int64_t(e) + delta[uint64_t(pk.round(k)) * C + pk.chunk(k)]);
    src16[pe] = uint16_t(k & 0xFFFFu);
    perm16[pe] = uint16_t(val[e] - tptr[bucket[bucket_of_pos[pk.pr(k)]].x]);
  }
}

// Pass 1: bins[i - base] = x[chunk window + src16[i]] over one item.
__global__ void __launch_bounds__(kPbScThreads, 1) k_pb_scatter(const uint4* __restrict__ items,
                                                           const float* __restrict__ xrow,
                                                           uint64_t n_xrow, uint32_t cw,
                                                           const uint16_t* __restrict__ src16,
                                                           float* __restrict__ bins,
                                                           uint64_t base) {
  extern __shared__ __align__(16) float win[];
  const uint4 it = items[blockIdx.x];
  const uint64_t w0 = uint64_t(it.x) * cw;
  const uint32_t wl = uint32_t(n_xrow - w0 < cw ? n_xrow - w0 : cw);
  {
    const float4* s4 = reinterpret_cast<const float4*>(xrow + w0);
    float4* d4 = reinterpret_cast<float4*>(win);
    for (uint32_t i = threadIdx.x; i < wl / 4; i += blockDim.x) d4[i] = __ldcg(&s4[i]);
    for (uint32_t i = (wl & ~3u) + threadIdx.x; i < wl; i += blockDim.x) win[i] = __ldcg(&xrow[w0 + i]);
  }
  __syncthreads();
  const uint4* s8 = reinterpret_cast<const uint4*>(src16);
  float4* b4 = reinterpret_cast<float4*>(bins - base);
  const uint32_t g1 = it.z / kPbGroup;
  auto put = [&](uint32_t g, uint4 q) {
    float4 lo, hi;
    lo.x = win[q.x & 0xFFFFu];
    lo.y = win[q.x >> 16];
    lo.z = win[q.y & 0xFFFFu];
    lo.w = win[q.y >> 16];
    hi.x = win[q.z & 0xFFFFu];
    hi.y = win[q.z >> 16];
    hi.z = win[q.w & 0xFFFFu];
    hi.w = win[q.w >> 16];
    b4[2 * uint64_t(g)] = lo;
    b4[2 * uint64_t(g) + 1] = hi;
  };
  uint32_t g = it.y / kPbGroup + threadIdx.x;
  for (; g + 3 * blockDim.x < g1; g += 4 * blockDim.x) {  // four index loads in flight
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = __ldcs(&s8[g + u * blockDim.x]);
#pragma unroll
    for (int u = 0; u < 4; ++u) put(g + u * blockDim.x, q[u]);
  }
  for (; g < g1; g += blockDim.x) put(g, __ldcs(&s8[g]));
}

// Pass 2: a CTA per bucket.  Runs (one per chunk) -> shared memory in
// destination order -> per-row folds in ascending source position -> ytail.
__global__ void __launch_bounds__(kPbThreads) k_pb_bucket(const uint2* __restrict__ bucket,
                                                          const uint2* __restrict__ runs, uint32_t C,
                                                          const uint16_t* __restrict__ perm16,
                                                          const float* __restrict__ bins,
                                                          uint64_t base,
                                                          const uint32_t* __restrict__ tptr,
                                                          float* __restrict__ ytail) {
  extern __shared__ __align__(16) float srt[];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t b = blockIdx.x;
  const uint2 pr = bucket[b];
  const uint2* rb = runs + uint64_t(b) * C;
  // the warp's runs are c = warp + j*nw; lane j holds run j's descriptor (32 at a time)
  for (uint32_t c0 = warp; c0 < C; c0 += 32 * nw) {
    const uint32_t cl = c0 + lane * nw;
    const uint2 mine = cl < C ? rb[cl] : make_uint2(0u, 0u);
    const uint32_t nr = min(32u, (C - c0 + nw - 1) / nw);
    for (uint32_t j = 0; j < nr; j += 2) {  // two runs' loads in flight
      const uint32_t xa = __shfl_sync(0xffffffffu, mine.x, j), la = __shfl_sync(0xffffffffu, mine.y, j);
      const uint32_t xb = __shfl_sync(0xffffffffu, mine.x, j + 1 < 32 ? j + 1 : 0);
      const uint32_t lb = j + 1 < nr ? __shfl_sync(0xffffffffu, mine.y, j + 1) : 0u;
      const uint32_t lm = max(la, lb);
      for (uint32_t k0 = 0; k0 < lm; k0 += 64) {
        uint32_t pi[4];
        float v[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t k = k0 + lane + 32u * (u & 1);
          const uint32_t x = u < 2 ? xa : xb, l = u < 2 ? la : lb;
          ok[u] = k < l;
          const uint64_t i = uint64_t(x) + k;
          pi[u] = ok[u] ? __ldcs(&perm16[i]) : 0u;
          v[u] = ok[u] ? __ldcg(&bins[i - base]) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ok[u]) srt[pi[u]] = v[u];
      }
    }
  }
  __syncthreads();
  const uint32_t t0 = tptr[pr.x];
  for (uint32_t p0 = pr.x + warp * 32u; p0 < pr.y; p0 += nw * 32u) {
    const uint32_t p = p0 + lane;
    uint32_t lo = 0, hi = 0;
    if (p < pr.y) {
      lo = tptr[p] - t0;
      hi = tptr[p + 1] - t0;
    }
    float sum = 0.0f;
    unsigned longs = __ballot_sync(0xffffffffu, hi - lo > 32u);
    if (hi - lo <= 32u)
      for (uint32_t k = lo; k < hi; ++k) sum += srt[k];
    while (longs) {  // long rows: the warp folds lane-strided partials with a fixed tree
      const int l = __ffs(longs) - 1;
      longs &= longs - 1;
      const uint32_t a = __shfl_sync(0xffffffffu, lo, l), z = __shfl_sync(0xffffffffu, hi, l);
      float t = 0.0f;
      for (uint32_t k = a + lane; k < z; k += 32) t += srt[k];
      t = warp_sum(t);
      if (int(lane) == l) sum = t;
    }
    if (p < pr.y) ytail[p] = sum;
  }
}

template <typename T>
void upload(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.alloc(h.size() + 1, s);
  if (!h.empty())
    GM_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* e = getenv(name);
  return e && *e ? uint32_t(strtoul(e, nullptr, 10)) : dflt;
}

template <typename K, typename V>
void pb_sort(DevBuf<K>& keys, DevBuf<V>* vals, uint64_t m, int end_bit, cudaStream_t s) {
  if (m <= 1) return;
  DevBuf<K> k2(m, s);
  cub::DoubleBuffer<K> dk(keys.get(), k2.get());
  size_t tmp = 0;
  if (vals) {
    DevBuf<V> v2(m, s);
    cub::DoubleBuffer<V> dv(vals->get(), v2.get());
    GM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int64_t(m), 0, end_bit, s));
    DevBuf<uint8_t> t(tmp, s);
    GM_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, dk, dv, int64_t(m), 0, end_bit, s));
    if (dv.Current() != vals->get()) vals->swap(v2);
  } else {
    GM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, dk, int64_t(m), 0, end_bit, s));
    DevBuf<uint8_t> t(tmp, s);
    GM_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, dk, int64_t(m), 0, end_bit, s));
  }
  if (dk.Current() != keys.get()) keys.swap(k2);
  GM_CUDA(cudaStreamSynchronize(s));
}

// Build the propagation-blocked layout of the tail entries (see k_pb_scatter).
void pb_build(PrHubCache& c, Graph& g, const std::vector<uint32_t>& td,
              const std::vector<uint32_t>& v_of_pos, const uint32_t* slot_d) {
  cudaStream_t s = g.stream;
  const uint64_t n = g.n, np = c.n_pos;
  // tail entries per position; destination-order offsets
  std::vector<uint32_t> tptr(np + 1);
  uint64_t E = 0;
  for (uint64_t p = 0; p < np; ++p) {
    tptr[p] = uint32_t(E);
    E += v_of_pos[p] == kNoRow ? 0 : td[v_of_pos[p]];
    if (E >= 0xFFFFFFF0ull) fail(GM_EENGINE, "pagerank: too many tail entries for the pb layout");
  }
  tptr[np] = uint32_t(E);
  c.pb_tail = E;
  c.ytail.alloc(np + 1, s);
  c.ytail.zero(s);
  upload(c.pb_tptr, tptr, s);
  c.pb_round_items.assign(1, 0);
  c.pb_round_buckets.assign(1, 0);
  c.pb_round_base.clear();
  if (E == 0) return;
  // buckets: position ranges holding <= cap tail entries and <= 8 rows per
  // thread, over the positions with in-edges (ytail stays 0 beyond n_count)
  std::vector<uint2> buckets;
  std::vector<uint32_t> bucket_of_pos(np);
  {
    const uint64_t np_in = c.n_count, max_rows = 8 * kPbThreads;
    uint64_t p0 = 0, cnt = 0;
    for (uint64_t p = np_in; p < np; ++p) bucket_of_pos[p] = 0;
    for (uint64_t p = 0; p < np_in; ++p) {
      const uint64_t t = tptr[p + 1] - tptr[p];
      if ((cnt + t > c.pb_cap || p - p0 >= max_rows) && p > p0) {
        buckets.push_back(make_uint2(uint32_t(p0), uint32_t(p)));
        p0 = p;
        cnt = 0;
      }
      bucket_of_pos[p] = uint32_t(buckets.size());
      cnt += t;
    }
    buckets.push_back(make_uint2(uint32_t(p0), uint32_t(np_in)));
  }
  const uint64_t nb = buckets.size();
  // rounds: bucket ranges of ~E/R entries (their bins stay in L2 between the passes)
  const uint32_t R = std::max(1u, env_u32("GM_PB_ROUNDS", 1));
  std::vector<uint32_t> round_of_bucket(nb);
  {
    const uint64_t cap = (E + R - 1) / R;
    uint64_t acc = 0;
    uint32_t r = 0;
    for (uint64_t b = 0; b < nb; ++b) {
      const uint64_t t = tptr[buckets[b].y] - tptr[buckets[b].x];
      if (acc + t > cap && acc > 0) {
        ++r;
        acc = 0;
        c.pb_round_buckets.push_back(uint32_t(b));
      }
      round_of_bucket[b] = r;
      acc += t;
    }
    c.pb_round_buckets.push_back(uint32_t(nb));
  }
  const uint32_t nR = uint32_t(c.pb_round_buckets.size() - 1);
  const uint32_t C = uint32_t((c.n_xrow + c.pb_cw - 1) / c.pb_cw);
  c.pb_C = C;
  PbKey pk{bits_for(np + 1), bits_for(C), c.pb_cw};
  const unsigned rbits = bits_for(nR);
  if (rbits + pk.cbits + pk.pbits + 16 > 64 || 2 * pk.pbits > 64)
    fail(GM_EENGINE, "pagerank: graph too large for the pb layout");
  DevBuf<uint32_t> bop_d, rob_d;
  DevBuf<uint2> bucket_d;
  upload(bop_d, bucket_of_pos, s);
  upload(rob_d, round_of_bucket, s);
  upload(bucket_d, buckets, s);
  // destination order: (position of the row, position of the source)
  DevBuf<uint64_t> key(E, s);
  {
    std::vector<uint64_t> toff(n + 1, 0);
    for (uint64_t r = 0; r < n; ++r) toff[r + 1] = toff[r] + td[r];
    DevBuf<uint64_t> toff_d;
    upload(toff_d, toff, s);
    k_pb_key2<<<grid_for(n * 32, 256), 256, 0, s>>>(n, g.in.ptr.get(), g.in.idx.get(), slot_d,
                                                   c.pos_of.get(), toff_d.get(), c.pb_big, pk.pbits,
                                                   key.get());
    GM_LAUNCH_CHECK();
    pb_sort<uint64_t, uint32_t>(key, nullptr, E, 2 * pk.pbits, s);
  }
  // bin order: (round, chunk, destination, source); val = destination-order index
  DevBuf<uint64_t> key1(E, s);
  DevBuf<uint32_t> val(E, s);
  k_pb_key1<<<grid_for(E, 256), 256, 0, s>>>(E, key.get(), pk.pbits, bop_d.get(), rob_d.get(), pk,
                                            key1.get(), val.get());
  GM_LAUNCH_CHECK();
  key.reset();
  pb_sort(key1, &val, E, int(rbits + pk.cbits + pk.pbits + 16), s);
  // run lengths per (bucket, chunk)
  std::vector<uint32_t> cnt(nb * C);
  {
    DevBuf<uint32_t> cnt_d(nb * C + 1, s);
    cnt_d.zero(s);
    k_pb_count<<<grid_for(E, 256), 256, 0, s>>>(E, key1.get(), pk, C, bop_d.get(), cnt_d.get());
    GM_LAUNCH_CHECK();
    GM_CUDA(cudaMemcpyAsync(cnt.data(), cnt_d.get(), nb * C * 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
  }
  // padded layout: every (round, chunk) segment starts on a multiple of kPbGroup;
  // pass-1 items are pieces of <= item entries of one segment
  const uint64_t item = std::max<uint64_t>(kPbGroup, env_u32("GM_PB_ITEM", 65536) & ~(kPbGroup - 1));
  std::vector<uint2> runs(nb * C);
  std::vector<int64_t> delta(uint64_t(nR) * C);
  std::vector<uint4> items;
  uint64_t pe = 0, e = 0, max_round = 0;
  for (uint32_t r = 0; r < nR; ++r) {
    c.pb_round_base.push_back(pe);
    const uint32_t b0 = c.pb_round_buckets[r], b1 = c.pb_round_buckets[r + 1];
    for (uint32_t ch = 0; ch < C; ++ch) {
      delta[uint64_t(r) * C + ch] = int64_t(pe) - int64_t(e);
      const uint64_t seg = pe;
      for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t k = cnt[uint64_t(b) * C + ch];
        runs[uint64_t(b) * C + ch] = make_uint2(uint32_t(pe), k);
        pe += k;
        e += k;
      }
      pe = (pe + kPbGroup - 1) & ~uint64_t(kPbGroup - 1);
      for (uint64_t i = seg; i < pe; i += item)
        items.push_back(make_uint4(ch, uint32_t(i), uint32_t(std::min(pe, i + item)), 0));
    }
    c.pb_round_items.push_back(uint32_t(items.size()));
    max_round = std::max(max_round, pe - c.pb_round_base.back());
  }
  if (pe >= 0xFFFFFFF0ull) fail(GM_EENGINE, "pagerank: too many tail entries for the pb layout");
  upload(c.pb_items, items, s);
  upload(c.pb_runs, runs, s);
  c.pb_bucket.swap(bucket_d);
  c.pb_bins.alloc(max_round + kPbGroup, s);
  c.pb_src.alloc(pe + kPbGroup, s);
  c.pb_perm.alloc(pe + kPbGroup, s);
  c.pb_src.zero(s);
  c.pb_perm.zero(s);
  {
    DevBuf<int64_t> delta_d;
    upload(delta_d, delta, s);
    k_pb_place<<<grid_for(E, 256), 256, 0, s>>>(E, key1.get(), val.get(), pk, C, delta_d.get(),
                                               bop_d.get(), c.pb_bucket.get(), c.pb_tptr.get(),
                                               c.pb_src.get(), c.pb_perm.get());
    GM_LAUNCH_CHECK();
    GM_CUDA(cudaStreamSynchronize(s));
  }
  GM_CUDA(cudaFuncSetAttribute(k_pb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(c.pb_cw) * 4));
  GM_CUDA(cudaFuncSetAttribute(k_pb_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(c.pb_cap) * 4));
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
  const uint64_t nh = std::min<uint64_t>(kHubCap, nz);
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
  DevBuf<uint32_t> slot_d;
  upload(slot_d, slot_of, s);

  // Propagation-blocked tail: on by default while x is L2-sized (the hub path's
  // own range); GM_PR_PB=0/1 forces it.
  {
    const char* e = getenv("GM_PR_TAIL");
    c.vertex_tail = e ? std::string(e) == "vertex" : n * 4 > (48ull << 20);
    const char* pbe = getenv("GM_PR_PB");
    c.pb = !c.vertex_tail && nh < nz && (pbe ? pbe[0] == '1' : false);
    c.pb_cw = env_u32("GM_PB_CW", 32768);
    c.pb_cap = env_u32("GM_PB_CAP", 16384);
    c.pb_big = std::min(c.pb_cap, env_u32("GM_PB_BIG", 16384));
    if (c.pb_cw > 65536 || c.pb_cw % 8 || c.pb_cap > 65536 || c.pb_big == 0)
      fail(GM_EUSAGE, "pagerank: GM_PB_CW must be a multiple of 8 <= 65536, GM_PB_CAP <= 65536");
  }
  // kd: entries the hub kernel keeps per row; td: tail entries left to pb
  std::vector<uint32_t> kd(n), td;
  if (c.pb) {
    DevBuf<uint32_t> kd_d(n + 1, s), td_d(n + 1, s);
    k_pb_deg<<<grid_for(n, 256), 256, 0, s>>>(n, g.in.ptr.get(), g.in.idx.get(), slot_d.get(),
                                             c.pb_big, kd_d.get(), td_d.get());
    GM_LAUNCH_CHECK();
    td.resize(n);
    GM_CUDA(cudaMemcpyAsync(kd.data(), kd_d.get(), n * 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaMemcpyAsync(td.data(), td_d.get(), n * 4, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
  } else {
    for (uint64_t r = 0; r < n; ++r) kd[r] = uint32_t(ptr[r + 1] - ptr[r]);
  }

  // positions: [long rows][SELL slices][rows without (kept) in-edges]
  const uint32_t sell_max = kSellMax;
  std::vector<uint32_t> longs, zeros;
  std::vector<uint64_t> bucket(sell_max + 1, 0);
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t d = kd[r];
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
    const uint64_t d = kd[r];
    if (d >= 1 && d <= sell_max) {
      const uint64_t e = start[d]++;
      v_of_pos[c.n_long + e] = uint32_t(r);
      sdeg[e] = uint32_t(d);
    }
  }
  // pb: rows whose in-edges are all tail entries come first among the zeros
  if (c.pb) std::stable_partition(zeros.begin(), zeros.end(), [&](uint32_t r) { return td[r] != 0; });
  c.n_count = c.n_in;
  for (uint64_t i = 0; i < zeros.size(); ++i) {
    v_of_pos[c.n_in + i] = zeros[i];
    if (c.pb && td[zeros[i]]) c.n_count = c.n_in + i + 1;
  }
  for (uint64_t p = 0; p < c.n_pos; ++p)
    if (v_of_pos[p] != kNoRow) pos_of[v_of_pos[p]] = uint32_t(p);
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
    long_ptr[i + 1] = long_ptr[i] + kd[longs[i]];
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
  const uint32_t big = c.pb ? c.pb_big : 0u;
  {
    DevBuf<uint64_t> long_ptr_d;
    upload(long_ptr_d, long_ptr, s);
    c.long_idx.alloc(long_ptr[c.n_long] + 1, s);
    if (c.n_long) {
      k_hub_fill_long<<<grid_for(c.n_long * 32, 256), 256, 0, s>>>(
          c.n_long, c.v_of_pos.get(), g.in.ptr.get(), g.in.idx.get(), long_ptr_d.get(),
          slot_d.get(), c.vertex_tail ? nullptr : c.pos_of.get(), c.H, big, c.long_idx.get());
      GM_LAUNCH_CHECK();
    }
    c.sell_idx.alloc(lines * 32 + 1, s);
    GM_CUDA(cudaMemsetAsync(c.sell_idx.get(), 0xFF, (lines * 32 + 1) * 4, s));
    if (nslices) {
      k_hub_fill_sell<<<grid_for(nslices * 32, 256), 256, 0, s>>>(
          nslices * 32, c.n_long, c.v_of_pos.get(), c.sell_end.get(), g.in.ptr.get(),
          g.in.idx.get(), slot_d.get(), c.vertex_tail ? nullptr : c.pos_of.get(), c.H, big,
          c.sell_idx.get());
      GM_LAUNCH_CHECK();
    }
    GM_CUDA(cudaStreamSynchronize(s));
  }
  if (c.pb) pb_build(c, g, td, v_of_pos, slot_d.get());
  for (int b = 0; b < 2; ++b) {
    c.rank[b].alloc(c.n_pos + 1, s);
    c.xrow[b].alloc(c.n_xrow + 1, s);
    c.xhub[b].alloc(c.H, s);
    c.xhub[b].zero(s);
  }
  c.dang.alloc(std::max<uint64_t>(kInitBlocks, uint64_t(c.grid) + c.n_multi) + 1, s);
  c.scalars.alloc(4, s);
  c.ctr.alloc(4, s);
  GM_CUDA(cudaEventCreate(&c.e0));
  GM_CUDA(cudaEventCreate(&c.e1));
  GM_CUDA(cudaFuncSetAttribute(k_pr_hub, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(c.H) * 4));
  GM_CUDA(cudaStreamSynchronize(s));
  return c;
}

}  // namespace

// The hub path serves whole-graph supersteps on one GPU while the message
// vector is L2-sized (<= 64 MB, scale <= 24 R-MAT); beyond that the gathers
// are DRAM-sector bound and the CTA-tile kernel of pagerank.cu, whose
// out-degree-ordered x keeps the warm sources L2-resident, is faster (scale
// 28: 24 ms vs 26.6 ms per superstep).  GM_PR_HUB=0/1 forces either path.
bool pagerank_hub_enabled(const Graph& g) {
  if (g.n == 0 || g.in.nnz == 0) return false;
  const char* e = getenv("GM_PR_HUB");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return g.n * 4 <= (64ull << 20);
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
    a.ytail = c.pb ? c.ytail.get() : nullptr;
    if (c.pb) {
      for (size_t r = 0; r + 1 < c.pb_round_items.size(); ++r) {
        const uint32_t i0 = c.pb_round_items[r], i1 = c.pb_round_items[r + 1];
        const uint32_t b0 = c.pb_round_buckets[r], b1 = c.pb_round_buckets[r + 1];
        const uint64_t base = c.pb_round_base[r];
        if (i1 > i0) {
          k_pb_scatter<<<i1 - i0, kPbScThreads, size_t(c.pb_cw) * 4, s>>>(
              c.pb_items.get() + i0, c.xrow[cur].get(), c.n_xrow, c.pb_cw, c.pb_src.get(),
              c.pb_bins.get(), base);
          GM_LAUNCH_CHECK();
        }
        if (b1 > b0) {
          k_pb_bucket<<<b1 - b0, kPbThreads, size_t(c.pb_cap) * 4, s>>>(
              c.pb_bucket.get() + b0, c.pb_runs.get() + uint64_t(b0) * c.pb_C, c.pb_C,
              c.pb_perm.get(), c.pb_bins.get(), base, c.pb_tptr.get(), c.ytail.get());
          GM_LAUNCH_CHECK();
        }
      }
    }
    k_pr_hub<<<c.grid, kHubThreads, size_t(c.H) * 4, s>>>(a);
    GM_LAUNCH_CHECK();
    k_hub_base<<<1, 1024, 0, s>>>(c.dang.get(), c.grid + c.n_multi, n, damping, c.scalars.get());
    GM_LAUNCH_CHECK();
    cur ^= 1;
    if (!collect) continue;
    GM_CUDA(cudaEventRecord(c.e1, s));
    GM_CUDA(cudaMemsetAsync(c.ctr.get(), 0, 8, s));
    k_hub_count<<<grid_for(c.n_count, 256), 256, 0, s>>>(c.n_count, c.rank[cur ^ 1].get(),
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
