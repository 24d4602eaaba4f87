// engine.cuh -- device-side VertexProgram engine (generic path, exact semantics).
//
// Mirrors semigraph::Engine (include/semigraph/engine.hpp:67-264) for ANY
// program: user functors are __device__ members of a program struct compiled
// into the kernels below as template parameters.  The device program contract
// restates the VertexProgram concept (include/semigraph/core.hpp:239-253):
//
//   using vertex_t, message_t, reduced_t, edge_t;   // edge_t = gm::NoEdge to ignore values
//   static constexpr gm_value_type kEdgeType;        // storage the program reads
//   __host__ __device__ Direction direction() const;
//   __device__ bool send_message(const vertex_t&, uint64_t v, message_t* out) const;  // false = nullopt
//   __device__ reduced_t process_message(const message_t&, const edge_t&, const vertex_t& dst) const;
//   __device__ reduced_t reduce(const reduced_t&, const reduced_t&) const;
//   __device__ reduced_t reduce_identity() const;
//   __device__ vertex_t apply(const reduced_t&, const vertex_t&) const;
//   __device__ bool equal(const vertex_t&, const vertex_t&) const;                      // operator==
//
// Programs that can fail set `static constexpr bool kCanFail = true` and take a
// trailing `int& err` in send/process/apply (the device analogue of a throwing
// callback); the engine attaches the vertex / (column, row) context exactly like
// engine.hpp:90-94, 158-162, 251-257.
//
// Semantics (SURVEY.md 8b rules S1-S9): bulk-synchronous reads, y valid iff one
// contribution landed, first fold reduce(identity, r), per-row fold order =
// ascending internal source id (caller order on graphs built without
// GM_RELABEL), BOTH merges out-route first, apply clears all flags and
// re-activates changed vertices only, zero budget is a no-op.
//
// Layout: properties / messages / reduced values are AoS device arrays in
// internal order; validity and activity are 32-bit-word bitmaps built with
// __ballot_sync (one word per warp, no atomics on the flags).  The pull SpMV is
// one thread per destination row so the fold order is the reference's; the
// specialised kernels (pagerank.cu, traversal.cu, cf.cu) trade that order for
// throughput where the program's reduce is exact or tolerance-checked.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "graph.cuh"

namespace gm {

enum class Direction : int { OUT = 0, IN = 1, BOTH = 2 };

struct NoEdge {};

template <typename P, typename = void>
struct can_fail : std::false_type {};
template <typename P>
struct can_fail<P, std::void_t<decltype(P::kCanFail)>> : std::bool_constant<P::kCanFail> {};

// Programs whose reduce is exactly associative and commutative with a true
// identity (min of doubles, integer sums) may fold a row in any order and
// get the sequential result bit for bit; they declare kExactReorder.
template <typename P, typename = void>
struct exact_reorder : std::false_type {};
template <typename P>
struct exact_reorder<P, std::void_t<decltype(P::kExactReorder)>>
    : std::bool_constant<P::kExactReorder> {};

// __shfl_xor_sync of any trivially copyable value, 32 bits at a time
template <typename T>
__device__ __forceinline__ T shfl_xor_any(const T& v, int o) {
  static_assert(sizeof(T) % 4 == 0, "shuffled values must be whole 32-bit words");
  uint32_t w[sizeof(T) / 4];
  memcpy(w, &v, sizeof(T));
#pragma unroll
  for (int i = 0; i < int(sizeof(T) / 4); ++i) w[i] = __shfl_xor_sync(0xffffffffu, w[i], o);
  T out;
  memcpy(&out, w, sizeof(T));
  return out;
}

enum Phase : int { kPhaseNone = 0, kPhaseSend = 1, kPhaseSpmv = 2, kPhaseApply = 3 };

struct DevError {
  int code;
  int phase;
  uint64_t vertex, col, row;
};

__device__ __forceinline__ void record_error(DevError* e, int code, int phase, uint64_t v,
                                             uint64_t col, uint64_t row) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->phase = phase;
    e->vertex = v;
    e->col = col;
    e->row = row;
  }
}

template <typename E>
__device__ __forceinline__ E load_edge(const uint8_t* val, uint64_t e) {
  if constexpr (std::is_same_v<E, NoEdge>) {
    return E{};
  } else {
    return reinterpret_cast<const E*>(val)[e];
  }
}

__device__ __forceinline__ uint64_t ext_id(const uint32_t* iperm, uint64_t v) {
  return iperm ? uint64_t(iperm[v]) : v;
}

// Adds lane 0's counts of every warp to ctr[0] (a) and ctr[1] (b, if nonzero
// anywhere) with one atomic per CTA: an atomic per warp step on one counter
// serialised at its L2 slice (k_send 0.36 ms at scale 23, 262 K words x 2).
// Every thread of the CTA must call it.
__device__ __forceinline__ void block_add_u64(unsigned long long* ctr, unsigned long long a,
                                              unsigned long long b) {
  __shared__ unsigned long long s_ab[2];
  if (threadIdx.x == 0) s_ab[0] = s_ab[1] = 0;
  __syncthreads();
  if ((threadIdx.x & 31u) == 0) {
    if (a) atomicAdd(&s_ab[0], a);
    if (b) atomicAdd(&s_ab[1], b);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_ab[0]) atomicAdd(&ctr[0], s_ab[0]);
    if (s_ab[1]) atomicAdd(&ctr[1], s_ab[1]);
  }
}

// ---------------------------------------------------------------- kernels
// Phase 1, engine.hpp:76-98: x[v] = send(prop[v]) for active v.
template <typename P>
__global__ void k_send(P p, uint64_t n, const typename P::vertex_t* props, const uint32_t* active,
                       const uint32_t* iperm, typename P::message_t* x, uint32_t* xbits,
                       unsigned long long* ctr, DevError* err) {
  // A warp takes 32 consecutive activity words (one coalesced load), then
  // only the nonzero ones, lane = vertex: a small frontier costs a pass over
  // the N/8-byte bitmap, not a warp step per word (the light supersteps of
  // the reference BfsProgram spent ~40 us here).
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long na = 0, no = 0;  // lane 0's running counts
  for (uint64_t w0 = warp * 32; w0 < words; w0 += nwarps * 32) {
    const uint64_t wl = w0 + lane;
    uint32_t aw = wl < words ? active[wl] : 0u;
    if (wl == words - 1 && (n & 31u)) aw &= (1u << (n & 31u)) - 1u;
    unsigned todo = __ballot_sync(0xffffffffu, aw != 0u);
    uint32_t mine = 0;  // this lane's word of xbits
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t word = __shfl_sync(0xffffffffu, aw, j);
      const uint64_t v = (w0 + uint64_t(j)) * 32 + lane;
      const bool act = (word >> lane) & 1u;
      bool ok = false;
      if (act) {
        typename P::message_t m;
        if constexpr (can_fail<P>::value) {
          int ec = 0;
          ok = p.send_message(props[v], ext_id(iperm, v), &m, ec);
          if (ec) {
            record_error(err, ec, kPhaseSend, ext_id(iperm, v), 0, 0);
            ok = false;
          }
        } else {
          ok = p.send_message(props[v], ext_id(iperm, v), &m);
        }
        if (ok) x[v] = m;
      }
      const unsigned ob = __ballot_sync(0xffffffffu, ok);
      if (lane == unsigned(j)) mine = ob;
      if (lane == 0) {
        na += __popc(word);
        no += __popc(ob);
      }
    }
    if (wl < words) xbits[wl] = mine;
  }
  block_add_u64(ctr, na, no);
}

// Frontier-proportional superstep (SpMSpV push), engine.hpp:224-260 with the
// columns that are not in x skipped (:234-236): only the valid messages'
// out-edges are visited.  Exactly order-free programs (kExactReorder, no
// failing callbacks, reduced_t of 4 or 8 bytes) fold each contribution into
// y[k] with a compare-and-swap loop: y holds reduce_identity() wherever it is
// not valid (set once, restored by apply), so the first contribution is
// reduce(identity, r) as S4 requires and any interleaving gives the
// sequential fold's bits.
template <typename P>
struct can_push
    : std::bool_constant<exact_reorder<P>::value && !can_fail<P>::value &&
                         (sizeof(typename P::reduced_t) == 4 || sizeof(typename P::reduced_t) == 8)> {};

template <typename R, typename P>
__device__ __forceinline__ void atomic_reduce(const P& p, R* addr, const R& r) {
  using W = std::conditional_t<sizeof(R) == 8, unsigned long long, unsigned int>;
  W* a = reinterpret_cast<W*>(addr);
  W old = *reinterpret_cast<volatile W*>(a);
  for (;;) {
    R ov;
    memcpy(&ov, &old, sizeof(R));
    const R nv = p.reduce(ov, r);
    W nb;
    memcpy(&nb, &nv, sizeof(R));
    if (nb == old) return;  // no change (e.g. min already smaller)
    const W prev = atomicCAS(a, old, nb);
    if (prev == old) return;
    old = prev;
  }
}

// The valid messages as a queue with their out-degrees (for the push), built
// from xbits after k_send.
__global__ void k_msg_queue(uint64_t n, const uint32_t* xbits, const uint64_t* out_ptr,
                            uint32_t* q, unsigned long long* ctr);

// qoff[i] = out-edges of the queue's sources before i (exclusive, qoff[nq] = total):
// the degrees, then an in-place exclusive scan (CUB) over nq + 1 entries
__global__ void k_queue_degrees(const uint32_t* q, const unsigned long long* qn,
                                const uint64_t* out_ptr, uint64_t* deg);
void exclusive_scan_u64(uint64_t* data, uint64_t n, cudaStream_t s);

// Edge-balanced: thread t handles the t-th frontier edge (its source found by
// a binary search over the queue offsets), so a hub source's edges spread
// over the whole grid instead of serialising one warp.
template <typename P>
__global__ void __launch_bounds__(256) k_push(P p, const uint32_t* q, const unsigned long long* qn,
                                              const uint64_t* qoff, const uint64_t* ptr,
                                              const uint32_t* idx, const uint8_t* val,
                                              const typename P::message_t* x,
                                              const typename P::vertex_t* props,
                                              typename P::reduced_t* y, uint32_t* ybits) {
  const uint64_t nq = qn[0], total = qn[1];
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = nq;  // last i with qoff[i] <= t
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (qoff[mid] <= t)
        lo = mid;
      else
        hi = mid;
    }
    const uint32_t j = q[lo];
    const uint64_t e = ptr[j] + (t - qoff[lo]);
    const uint32_t k = idx[e];
    const typename P::reduced_t r =
        p.process_message(x[j], load_edge<typename P::edge_t>(val, e), props[k]);
    atomic_reduce(p, &y[k], r);
    const uint32_t bit = 1u << (k & 31u);
    if (!(ybits[k >> 5] & bit)) atomicOr(&ybits[k >> 5], bit);
  }
}

template <typename P>
__global__ void k_fill_identity(P p, uint64_t n, typename P::reduced_t* y) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    y[v] = p.reduce_identity();
}

// Rows longer than this go to k_pull_long (a warp per row).
constexpr uint64_t kLongRow = 32;

// Phase 2, engine.hpp:224-260: one thread per destination row, entries in
// ascending source order, first contribution folded as reduce(identity, r).
// Rows with more than kLongRow entries are left to k_pull_long (launched
// after this kernel: it ORs its rows' bits into the words written here).
template <typename P>
__global__ void k_pull(P p, uint64_t n, const uint64_t* ptr, const uint32_t* idx,
                       const uint8_t* val, const typename P::message_t* x, const uint32_t* xbits,
                       const typename P::vertex_t* props, const uint32_t* iperm,
                       typename P::reduced_t* y, uint32_t* ybits, DevError* err) {
  using R = typename P::reduced_t;
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint64_t k = w * 32 + lane_id();
    bool any = false;
    if (k < n && ptr[k + 1] - ptr[k] <= kLongRow) {
      R acc = p.reduce_identity();
      const uint64_t e1 = ptr[k + 1];
      for (uint64_t e = ptr[k]; e < e1; ++e) {
        const uint32_t j = idx[e];
        if (!bit_test(xbits, j)) continue;
        R r;
        if constexpr (can_fail<P>::value) {
          int ec = 0;
          r = p.process_message(x[j], load_edge<typename P::edge_t>(val, e), props[k], ec);
          if (ec) {
            record_error(err, ec, kPhaseSpmv, 0, ext_id(iperm, j), ext_id(iperm, k));
            break;
          }
        } else {
          r = p.process_message(x[j], load_edge<typename P::edge_t>(val, e), props[k]);
        }
        acc = any ? p.reduce(acc, r) : p.reduce(p.reduce_identity(), r);
        any = true;
      }
      if (any) y[k] = acc;
    }
    const unsigned b = __ballot_sync(0xffffffffu, any);
    if (lane_id() == 0 && b) atomicOr(&ybits[w], b);  // k_pull_long may run concurrently
  }
}

// Order-free programs (kExactReorder, no failing callbacks): a group of
// kGroup lanes per short row, lanes striding over the row's entries (the
// group's index loads are one 32-byte sector) and a shuffle tree combining
// the partial folds -- bit-identical to the sequential fold by the program's
// declaration.  Replaces k_pull's thread per row (32 scattered rows per load
// instruction) for those programs.
constexpr unsigned kGroup = 8;

template <typename P>
__global__ void __launch_bounds__(256) k_pull_group(P p, uint64_t n, const uint64_t* ptr,
                                                    const uint32_t* idx, const uint8_t* val,
                                                    const typename P::message_t* x,
                                                    const uint32_t* xbits,
                                                    const typename P::vertex_t* props,
                                                    typename P::reduced_t* y, uint32_t* ybits) {
  using R = typename P::reduced_t;
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id(), sub = lane % kGroup, grp = lane / kGroup;
  for (uint64_t w = warp; w < words; w += nwarps) {
    unsigned word = 0;
#pragma unroll 1
    for (unsigned r0 = 0; r0 < 32; r0 += 32 / kGroup) {
      const uint64_t k = w * 32 + r0 + grp;
      bool any = false;
      R acc = p.reduce_identity();
      if (k < n) {
        const uint64_t e0 = ptr[k], e1 = ptr[k + 1];
        if (e1 - e0 <= kLongRow) {
          for (uint64_t e = e0 + sub; e < e1; e += kGroup) {
            const uint32_t j = idx[e];
            if (!bit_test(xbits, j)) continue;
            const R r = p.process_message(x[j], load_edge<typename P::edge_t>(val, e), props[k]);
            acc = any ? p.reduce(acc, r) : p.reduce(p.reduce_identity(), r);
            any = true;
          }
        }
      }
#pragma unroll
      for (unsigned o = kGroup / 2; o > 0; o >>= 1) {
        const R other = shfl_xor_any(acc, int(o));
        const bool oany = __shfl_xor_sync(0xffffffffu, any, int(o));
        if (oany) {
          acc = any ? p.reduce(acc, other) : other;
          any = true;
        }
      }
      if (sub == 0 && any) y[k] = acc;
      const unsigned b = __ballot_sync(0xffffffffu, sub == 0 && any);
      // lane grp*kGroup holds row r0 + grp's flag
#pragma unroll
      for (unsigned g2 = 0; g2 < 32 / kGroup; ++g2)
        if ((b >> (g2 * kGroup)) & 1u) word |= 1u << (r0 + g2);
    }
    if (lane == 0 && word) atomicOr(&ybits[w], word);  // k_pull_long may run concurrently
  }
}

// Order-free programs split long rows into pieces of <= kPiece entries, a
// warp per piece, each piece's fold combined into y[k] with atomic_reduce (y
// is the identity wherever invalid): a hub row no longer serialises one warp.
constexpr uint64_t kPiece = 2048;

__global__ void k_piece_counts(const uint32_t* rows, uint64_t nrows, const uint64_t* ptr,
                               uint64_t* cnt);
__global__ void k_piece_fill(const uint32_t* rows, uint64_t nrows, const uint64_t* ptr,
                             const uint64_t* off, uint32_t* prow, uint64_t* pbeg);

template <typename P>
__global__ void __launch_bounds__(256) k_pull_pieces(P p, const uint32_t* prow, const uint64_t* pbeg,
                                                     uint64_t npieces, const uint64_t* ptr,
                                                     const uint32_t* idx, const uint8_t* val,
                                                     const typename P::message_t* x,
                                                     const uint32_t* xbits,
                                                     const typename P::vertex_t* props,
                                                     typename P::reduced_t* y, uint32_t* ybits) {
  using R = typename P::reduced_t;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t i = warp; i < npieces; i += nwarps) {
    const uint32_t k = prow[i];
    const uint64_t b = pbeg[i], e1 = min(ptr[k + 1], b + kPiece);
    const typename P::vertex_t vk = props[k];
    R acc = p.reduce_identity();
    bool any = false;
    for (uint64_t e = b + lane; e < e1; e += 32) {
      const uint32_t j = idx[e];
      if (!bit_test(xbits, j)) continue;
      const R r = p.process_message(x[j], load_edge<typename P::edge_t>(val, e), vk);
      acc = any ? p.reduce(acc, r) : p.reduce(p.reduce_identity(), r);
      any = true;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const R other = shfl_xor_any(acc, o);
      const bool oany = __shfl_xor_sync(0xffffffffu, any, o);
      if (oany) {
        acc = any ? p.reduce(acc, other) : other;
        any = true;
      }
    }
    if (lane == 0 && any) {
      atomic_reduce(p, &y[k], acc);
      atomicOr(&ybits[k >> 5], 1u << (k & 31u));
    }
  }
}

// Long rows (> kLongRow entries): a warp per row.  The 32 lanes evaluate 32
// consecutive entries at once (bit test, message load, process_message) and
// stage the results in shared memory; lane 0 then folds them strictly in entry
// order -- the reference's per-row order, so any reduce, associative or not,
// gives the thread-per-row result bit for bit -- while the next 32 entries'
// loads are the warp's only other work.  The first failing entry of a row (in
// entry order) is the one reported.
constexpr unsigned kLongThreads = 256;

template <typename P>
__global__ void __launch_bounds__(kLongThreads) k_pull_long(
    P p, const uint32_t* rows, uint64_t nrows, const uint64_t* ptr, const uint32_t* idx,
    const uint8_t* val, const typename P::message_t* x, const uint32_t* xbits,
    const typename P::vertex_t* props, const uint32_t* iperm, typename P::reduced_t* y,
    uint32_t* ybits, DevError* err) {
  using R = typename P::reduced_t;
  using M = typename P::message_t;
  using E = typename P::edge_t;
  __shared__ __align__(16) unsigned char s_raw[kLongThreads * sizeof(R)];
  R* s_r = reinterpret_cast<R*>(s_raw) + (threadIdx.x & ~31u);
  const unsigned lane = lane_id();
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  // Three-stage pipeline per warp: the column ids of chunk c+2 and the
  // messages, validity words and edge values of chunk c+1 are in flight while
  // chunk c is processed and folded (messages are loaded unconditionally --
  // every id is in range -- so no load waits on the bit test).
  struct Staged {
    bool in = false;
    uint32_t j = 0, word = 0;
    M m{};
    E ed{};
  };
  for (uint64_t i = warp; i < nrows; i += nwarps) {
    const uint32_t k = rows[i];
    const uint64_t e0 = ptr[k], e1 = ptr[k + 1];
    const typename P::vertex_t vk = props[k];
    auto load_idx = [&](uint64_t b) { return b + lane < e1 ? idx[b + lane] : 0u; };
    auto load_msg = [&](uint64_t b, uint32_t j, Staged& st) {
      st.in = b + lane < e1;
      st.j = j;
      if (st.in) {
        st.word = xbits[j >> 5];
        st.m = x[j];
        st.ed = load_edge<E>(val, b + lane);
      }
    };
    R acc = p.reduce_identity();
    bool any = false;
    Staged cur, nxt;
    load_msg(e0, load_idx(e0), cur);
    uint32_t jn = load_idx(e0 + 32);
    for (uint64_t base = e0; base < e1; base += 32) {
      if (base + 32 < e1) load_msg(base + 32, jn, nxt);
      jn = load_idx(base + 64);
      const bool valid = cur.in && ((cur.word >> (cur.j & 31u)) & 1u);
      int ec = 0;
      R r{};
      if (valid) {
        if constexpr (can_fail<P>::value)
          r = p.process_message(cur.m, cur.ed, vk, ec);
        else
          r = p.process_message(cur.m, cur.ed, vk);
      }
      if constexpr (can_fail<P>::value) {
        const unsigned fm = __ballot_sync(0xffffffffu, ec != 0);
        if (fm) {  // the row's first failing entry; the superstep aborts
          if (int(lane) == __ffs(fm) - 1)
            record_error(err, ec, kPhaseSpmv, 0, ext_id(iperm, cur.j), ext_id(iperm, k));
          any = false;
          break;
        }
      }
      if constexpr (exact_reorder<P>::value && !can_fail<P>::value) {
        // order-free programs: every lane folds its own entries, the warp
        // combines the 32 partials at the end of the row
        if (valid) {
          acc = any ? p.reduce(acc, r) : p.reduce(p.reduce_identity(), r);
          any = true;
        }
        cur = nxt;
        continue;
      }
      // valid contributions packed in entry order; lane 0 folds a count in
      // branch-free groups of 8 (a predicate and branch per entry cost ~3x
      // the reduce itself)
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      if (valid) s_r[__popc(vm & ((1u << lane) - 1u))] = r;
      __syncwarp();
      if (lane == 0 && vm) {
        const int cnt = __popc(vm);
        int t = 0;
        if (!any) {
          acc = p.reduce(p.reduce_identity(), s_r[0]);
          any = true;
          t = 1;
        }
        for (; t + 8 <= cnt; t += 8) {
          R v8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v8[u] = s_r[t + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = p.reduce(acc, v8[u]);
        }
        for (; t < cnt; ++t) acc = p.reduce(acc, s_r[t]);
      }
      __syncwarp();
      cur = nxt;
    }
    if constexpr (exact_reorder<P>::value && !can_fail<P>::value) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const R other = shfl_xor_any(acc, o);
        const bool oany = __shfl_xor_sync(0xffffffffu, any, o);
        if (oany) {
          acc = any ? p.reduce(acc, other) : other;
          any = true;
        }
      }
    }
    if (lane == 0 && any) {
      y[k] = acc;
      atomicOr(&ybits[k >> 5], 1u << (k & 31u));
    }
  }
}

// Hub rows of order-sensitive programs (more than kHubRow entries, no failing
// callbacks): one CTA per row.  The row's fold has to stay one sequential
// chain -- reduce(...reduce(reduce(identity, r0), r1)..., r_last) in entry
// order is the reference's result bit for bit -- but everything before it
// need not: 15 producer warps gather the messages and evaluate
// process_message for 32-entry chunks into a shared-memory ring, and one
// consumer thread folds the ring in entry order, so the chain runs at the
// reduce's latency instead of behind one warp's load round trips.  (k_pull_long
// has the warp's lane 0 fold while the same warp loads the next chunks: the
// hub row -- 10^5 entries and more at scale 23 -- was the superstep's
// critical path, 6.3 ms of a 7 ms superstep.)
constexpr uint64_t kHubRow = 4096;
constexpr unsigned kHubThreads = 512;
constexpr unsigned kHubSlot = 64;  // entries per ring slot (two per producer lane)
// ring slots: 32 (16 KB of 8-byte values), fewer for wide reduced values
template <typename R>
constexpr unsigned hub_ring() {
  return kHubSlot * sizeof(R) * 32u <= 40960u ? 32u
         : 40960u / (kHubSlot * unsigned(sizeof(R))) >= 4u ? 40960u / (kHubSlot * unsigned(sizeof(R)))
                                                            : 4u;
}

// Shared-memory flag handshake of k_pull_hub: acquire / release at CTA scope
// (a full __threadfence_block is a MEMBAR.SC per slot on the consumer's
// critical path).
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v)
               : "r"(unsigned(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}

// Rows are claimed from `claim` (zeroed before the launch), longest first: the
// CTA holding the longest row takes no other, so the superstep's critical path
// is that row's fold alone (grid-stride dealing had added ~6 more rows to it).
template <typename P>
__global__ void __launch_bounds__(kHubThreads) k_pull_hub(
    P p, const uint32_t* rows, uint64_t nrows, unsigned* claim, const uint64_t* ptr,
    const uint32_t* idx, const uint8_t* val, const typename P::message_t* x, const uint32_t* xbits,
    uint64_t nx, const typename P::vertex_t* props, typename P::reduced_t* y, uint32_t* ybits) {
  using R = typename P::reduced_t;
  using E = typename P::edge_t;
  using M = typename P::message_t;
  constexpr unsigned kHubRing = hub_ring<R>();
  __shared__ __align__(16) unsigned char s_raw[kHubRing * kHubSlot * sizeof(R)];
  R* ring = reinterpret_cast<R*>(s_raw);
  __shared__ unsigned s_cnt[kHubRing];
  __shared__ int s_ready[kHubRing];  // slot number + 1 once the slot holds it
  __shared__ int s_consumed;         // slots the consumer has folded (published every 2)
  __shared__ unsigned s_row;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  constexpr unsigned kProducers = kHubThreads / 32 - 1;
  for (;;) {
    for (unsigned t = threadIdx.x; t < kHubRing; t += blockDim.x) s_ready[t] = 0;
    if (threadIdx.x == 0) {
      s_consumed = 0;
      s_row = atomicAdd(claim, 1u);
    }
    __syncthreads();
    const uint64_t i = s_row;
    if (i >= nrows) break;
    const uint32_t k = rows[i];
    const uint64_t e0 = ptr[k], e1 = ptr[k + 1];
    const int nsl = int((e1 - e0 + kHubSlot - 1) / kHubSlot);
    if (warp > 0) {
      const typename P::vertex_t vk = props[k];
      int c = int(warp) - 1;
      auto col = [&](int cc, int h) -> uint32_t {
        const uint64_t e = e0 + uint64_t(cc) * kHubSlot + 32u * h + lane;
        return cc < nsl && e < e1 ? idx[e] : 0u;
      };
      uint32_t j[2] = {col(c, 0), col(c, 1)};
      for (; c < nsl; c += int(kProducers)) {
        // this slot's messages, validity words and edge values, and the next
        // slot's column ids, all in flight before the slot wait
        bool in[2], valid[2];
        uint32_t word[2];
        M m[2];
        E ed[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint64_t e = e0 + uint64_t(c) * kHubSlot + 32u * h + lane;
          in[h] = e < e1;
          GM_DCHECK(!in[h] || j[h] < nx);
          word[h] = in[h] ? xbits[j[h] >> 5] : 0u;
          m[h] = in[h] ? x[j[h]] : M{};
          ed[h] = in[h] ? load_edge<E>(val, e) : E{};
        }
        const int cn = c + int(kProducers);
        const uint32_t jn[2] = {col(cn, 0), col(cn, 1)};
        R r[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          valid[h] = in[h] && ((word[h] >> (j[h] & 31u)) & 1u);
          r[h] = R{};
          if (valid[h]) r[h] = p.process_message(m[h], ed[h], vk);
        }
        const unsigned slot = unsigned(c) % kHubRing;
        if (c >= int(kHubRing)) {
          // a full ring: sleep long -- spinning producers took the consumer's
          // issue slots (163 cycles per folded entry at 32 ns sleeps)
          if (lane == 0)
            while (ld_acquire_cta(&s_consumed) <= c - int(kHubRing)) __nanosleep(1000);
          __syncwarp();
        }
        // valid contributions packed to the front of the slot, in entry
        // order: the consumer folds a count, with no per-entry predicate
        const unsigned vm0 = __ballot_sync(0xffffffffu, valid[0]);
        const unsigned vm1 = __ballot_sync(0xffffffffu, valid[1]);
        const unsigned below = (1u << lane) - 1u;
        R* rs = ring + slot * kHubSlot;
        if (valid[0]) rs[__popc(vm0 & below)] = r[0];
        if (valid[1]) rs[__popc(vm0) + __popc(vm1 & below)] = r[1];
        __threadfence_block();
        __syncwarp();
        if (lane == 0) {
          s_cnt[slot] = unsigned(__popc(vm0) + __popc(vm1));
          st_release_cta(&s_ready[slot], c + 1);
        }
        j[0] = jn[0];
        j[1] = jn[1];
      }
    } else if (lane == 0) {
      R acc = p.reduce_identity();
      bool any = false;
      for (int c = 0; c < nsl; ++c) {
        const unsigned slot = unsigned(c) % kHubRing;
        // no sleep: the consumer is the critical path
        while (ld_acquire_cta(&s_ready[slot]) != c + 1) {
        }
        const int cnt = int(s_cnt[slot]);
        const R* rs = ring + slot * kHubSlot;
        if (any && cnt == int(kHubSlot)) {
          // the common full slot: one straight-line chain, so the compiler
          // issues each value's shared load several reduces ahead of its use
          // (the dynamic-count loop below waits on every group's loads)
#pragma unroll
          for (int u = 0; u < int(kHubSlot); ++u) acc = p.reduce(acc, rs[u]);
          if ((c & 1) == 1 || c + 1 == nsl) st_release_cta(&s_consumed, c + 1);
          continue;
        }
        int t = 0;
        if (!any && cnt) {
          acc = p.reduce(p.reduce_identity(), rs[0]);  // the row's first fold (S4)
          any = true;
          t = 1;
        }
        // branch-free groups of 8 (a predicate or branch per entry cost more
        // than the reduce itself)
        for (; t + 8 <= cnt; t += 8) {
          R v8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v8[u] = rs[t + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = p.reduce(acc, v8[u]);
        }
        for (; t < cnt; ++t) acc = p.reduce(acc, rs[t]);
        if ((c & 1) == 1 || c + 1 == nsl) st_release_cta(&s_consumed, c + 1);
      }
      if (any) {
        y[k] = acc;
        atomicOr(&ybits[k >> 5], 1u << (k & 31u));
      }
    }
    __syncthreads();  // the ring is reused by the next row
  }
}

// Entry counts of listed rows (hub selection on the host).
__global__ void k_row_lens(const uint32_t* rows, uint64_t nrows, const uint64_t* ptr,
                           uint32_t* lens);

// Row ids with more than kLongRow entries (order irrelevant: rows are independent).
__global__ void k_long_rows(uint64_t n, const uint64_t* ptr, uint32_t* rows,
                            unsigned long long* cnt);

// BOTH merge, engine.hpp:113-126: y_in folded into y_out, out-route first.
template <typename P>
__global__ void k_merge(P p, uint64_t n, typename P::reduced_t* y, uint32_t* ybits,
                        const typename P::reduced_t* y2, const uint32_t* y2bits) {
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t w = warp; w < words; w += nwarps) {
    const uint64_t v = w * 32 + lane_id();
    if (v < n) {
      const bool o = bit_test(ybits, uint32_t(v)), i = bit_test(y2bits, uint32_t(v));
      if (o && i)
        y[v] = p.reduce(y[v], y2[v]);
      else if (i)
        y[v] = y2[v];
    }
    __syncwarp();
    if (lane_id() == 0) ybits[w] |= y2bits[w];
  }
}

// Phase 3, engine.hpp:139-172: clear every flag, apply where y is valid,
// re-activate iff the state changed.
template <typename P>
__global__ void k_apply(P p, uint64_t n, typename P::reduced_t* y, const uint32_t* ybits,
                        typename P::vertex_t* props, uint32_t* active, const uint32_t* iperm,
                        unsigned long long* ctr, DevError* err) {
  // 32 consecutive validity words per warp step (coalesced), then the nonzero
  // ones lane = vertex; every activity word is rewritten (all flags cleared,
  // changed vertices set)
  const uint64_t words = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  unsigned long long nu = 0;  // lane 0's running count
  for (uint64_t w0 = warp * 32; w0 < words; w0 += nwarps * 32) {
    const uint64_t wl = w0 + lane;
    uint32_t yw = wl < words ? ybits[wl] : 0u;
    if (wl == words - 1 && (n & 31u)) yw &= (1u << (n & 31u)) - 1u;
    unsigned todo = __ballot_sync(0xffffffffu, yw != 0u);
    uint32_t mine = 0;  // this lane's word of the new activity
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t word = __shfl_sync(0xffffffffu, yw, j);
      const uint64_t v = (w0 + uint64_t(j)) * 32 + lane;
      bool upd = false;
      if ((word >> lane) & 1u) {
        const typename P::vertex_t old = props[v];
        typename P::vertex_t fresh;
        bool okv = true;
        const typename P::reduced_t yv = y[v];
        if constexpr (can_push<P>::value) y[v] = p.reduce_identity();  // the push's invariant
        if constexpr (can_fail<P>::value) {
          int ec = 0;
          fresh = p.apply(yv, old, ec);
          if (ec) {
            record_error(err, ec, kPhaseApply, ext_id(iperm, v), 0, 0);
            okv = false;
          }
        } else {
          fresh = p.apply(yv, old);
        }
        if (okv && !p.equal(fresh, old)) {
          props[v] = fresh;
          upd = true;
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, upd);
      if (lane == unsigned(j)) mine = b;
      if (lane == 0) nu += __popc(b);
    }
    if (wl < words) active[wl] = mine;
  }
  block_add_u64(ctr + 2, nu, 0);
}

__global__ void k_bytes_to_bits(const uint8_t* bytes, uint64_t n, uint32_t* bits);
__global__ void k_bits_to_bytes(const uint32_t* bits, uint64_t n, uint8_t* bytes);

// ------------------------------------------------------------------ host side
template <typename P>
class Engine {
 public:
  using V = typename P::vertex_t;
  using M = typename P::message_t;
  using R = typename P::reduced_t;

  Engine(Graph& g, const P& p) : g_(g), p_(p), s_(g.stream) {
    if constexpr (!std::is_same_v<typename P::edge_t, NoEdge>) {
      if (g.value_type != P::kEdgeType)
        fail(GM_EUSAGE, std::string("program reads ") + value_name(P::kEdgeType) +
                            " edge values but the graph stores " + value_name(g.value_type));
    }
    const Direction d = p_.direction();
    if (d != Direction::OUT) ensure_forward(g_);  // engine.hpp:107, 195
    const uint64_t n = g_.n, words = (n + 31) / 32;
    props_.alloc(n, s_);
    active_.alloc(words + 1, s_);
    active_.zero(s_);
    x_.alloc(n, s_);
    xbits_.alloc(words + 1, s_);
    y_.alloc(n, s_);
    ybits_.alloc(words + 1, s_);
    if (d == Direction::BOTH) {
      y2_.alloc(n, s_);
      y2bits_.alloc(words + 1, s_);
    }
    ctr_.alloc(3, s_);
    ctr_.zero(s_);
    err_.alloc(1, s_);
    err_.zero(s_);
    if constexpr (can_push<P>::value) {
      if (d == Direction::OUT && n) {  // y = identity wherever invalid (the push's invariant)
        k_fill_identity<P><<<grid_for(n, 256), 256, 0, s_>>>(p_, n, y_.get());
        GM_LAUNCH_CHECK();
      }
    }
    GM_CUDA(cudaEventCreate(&e0_));
    GM_CUDA(cudaEventCreate(&e1_));
    GM_CUDA(cudaEventCreate(&e2_));
    GM_CUDA(cudaEventCreate(&e3_));
  }
  ~Engine() {
    if (side_) {
      cudaStreamSynchronize(side_);
      cudaStreamDestroy(side_);
      cudaEventDestroy(fork_);
      cudaEventDestroy(join_);
    }
    if (hub_) {
      cudaStreamSynchronize(hub_);
      cudaStreamDestroy(hub_);
      cudaEventDestroy(hfork_);
      cudaEventDestroy(hjoin_);
    }
    cudaEventDestroy(e0_);
    cudaEventDestroy(e1_);
    cudaEventDestroy(e2_);
    cudaEventDestroy(e3_);
  }

  // Caller-order host arrays -> internal device state.
  void load(const void* props_host, const uint8_t* active_host) {
    const uint64_t n = g_.n;
    if (!n) return;
    DevBuf<V> tmp(n, s_);
    GM_CUDA(cudaMemcpyAsync(tmp.get(), props_host, n * sizeof(V), cudaMemcpyHostToDevice, s_));
    to_internal(g_, tmp.get(), props_.get(), sizeof(V));
    DevBuf<uint8_t> a(n, s_), ai(n, s_);
    GM_CUDA(cudaMemcpyAsync(a.get(), active_host, n, cudaMemcpyHostToDevice, s_));
    to_internal(g_, a.get(), ai.get(), 1);
    k_bytes_to_bits<<<grid_for((n + 31) / 32, 256), 256, 0, s_>>>(ai.get(), n, active_.get());
    GM_LAUNCH_CHECK();
    GM_CUDA(cudaStreamSynchronize(s_));
  }

  void store(void* props_host, uint8_t* active_host) {
    const uint64_t n = g_.n;
    if (!n) return;
    DevBuf<V> tmp(n, s_);
    to_external(g_, props_.get(), tmp.get(), sizeof(V));
    GM_CUDA(cudaMemcpyAsync(props_host, tmp.get(), n * sizeof(V), cudaMemcpyDeviceToHost, s_));
    bits_out(active_.get(), active_host);
  }

  void bits_out(const uint32_t* bits, uint8_t* host) {
    const uint64_t n = g_.n;
    DevBuf<uint8_t> b(n, s_), be(n, s_);
    k_bits_to_bytes<<<grid_for(n, 256), 256, 0, s_>>>(bits, n, b.get());
    GM_LAUNCH_CHECK();
    to_external(g_, b.get(), be.get(), 1);
    GM_CUDA(cudaMemcpyAsync(host, be.get(), n, cudaMemcpyDeviceToHost, s_));
    GM_CUDA(cudaStreamSynchronize(s_));
  }

  void send() {
    const uint64_t n = g_.n;
    const unsigned grid = grid_for((n + 31) / 32, 256);  // a warp per 32 words
    k_send<P><<<grid, 256, 0, s_>>>(p_, n, props_.get(), active_.get(), iperm(), x_.get(),
                                     xbits_.get(), ctr_.get(), err_.get());
    GM_LAUNCH_CHECK();
  }

  // rows of `c` with more than kLongRow entries, once per engine and CSR
  uint64_t long_rows(const Csr& c, DevBuf<uint32_t>& rows) {
    const uint64_t n = g_.n;
    rows.alloc(n + 1, s_);
    DevBuf<unsigned long long> cnt(1, s_);
    cnt.zero(s_);
    if (n) {
      k_long_rows<<<grid_for(n, 256), 256, 0, s_>>>(n, c.ptr.get(), rows.get(), cnt.get());
      GM_LAUNCH_CHECK();
    }
    unsigned long long h = 0;
    GM_CUDA(cudaMemcpyAsync(&h, cnt.get(), 8, cudaMemcpyDeviceToHost, s_));
    GM_CUDA(cudaStreamSynchronize(s_));
    return h;
  }

  // Order-sensitive programs without failing callbacks fold hub rows with
  // k_pull_hub (one CTA per row, a sequential consumer fed by producer warps).
  static constexpr bool kHubPath = !exact_reorder<P>::value && !can_fail<P>::value;

  // Move the rows above kHubRow entries from `lrows` to `hrows`, longest first
  // (the longest row's fold is the superstep's critical path, so it starts in
  // the first wave).  Once per engine and route.
  void split_hubs(const Csr& c, DevBuf<uint32_t>& lrows, uint64_t& nlong, DevBuf<uint32_t>& hrows,
                  uint64_t& nhub) {
    nhub = 0;
    if (!nlong) return;
    DevBuf<uint32_t> lens(nlong + 1, s_);
    k_row_lens<<<grid_for(nlong, 256), 256, 0, s_>>>(lrows.get(), nlong, c.ptr.get(), lens.get());
    GM_LAUNCH_CHECK();
    std::vector<uint32_t> rows(nlong), len(nlong);
    GM_CUDA(cudaMemcpyAsync(rows.data(), lrows.get(), nlong * 4, cudaMemcpyDeviceToHost, s_));
    GM_CUDA(cudaMemcpyAsync(len.data(), lens.get(), nlong * 4, cudaMemcpyDeviceToHost, s_));
    GM_CUDA(cudaStreamSynchronize(s_));
    std::vector<uint32_t> mid;
    std::vector<std::pair<uint32_t, uint32_t>> hub;
    mid.reserve(nlong);
    for (uint64_t i = 0; i < nlong; ++i) {
      if (len[i] > kHubRow)
        hub.emplace_back(len[i], rows[i]);
      else
        mid.push_back(rows[i]);
    }
    if (hub.empty()) return;
    std::sort(hub.begin(), hub.end(), [](const auto& a, const auto& b) {
      return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    std::vector<uint32_t> h(hub.size());
    for (size_t i = 0; i < hub.size(); ++i) h[i] = hub[i].second;
    nhub = h.size();
    hrows.alloc(nhub + 1, s_);
    GM_CUDA(cudaMemcpyAsync(hrows.get(), h.data(), nhub * 4, cudaMemcpyHostToDevice, s_));
    nlong = mid.size();
    if (nlong)
      GM_CUDA(cudaMemcpyAsync(lrows.get(), mid.data(), nlong * 4, cudaMemcpyHostToDevice, s_));
    GM_CUDA(cudaStreamSynchronize(s_));
  }

  void pull(const Csr& c, DevBuf<uint32_t>& lrows, uint64_t& nlong, DevBuf<uint32_t>& hrows,
            uint64_t& nhub, bool& have, R* y, uint32_t* ybits) {
    const uint64_t n = g_.n;
    if (!have) {
      nlong = long_rows(c, lrows);
      nhub = 0;
      if constexpr (kHubPath) {
        static const bool hub_on = !(getenv("GM_GENERIC_HUB") && getenv("GM_GENERIC_HUB")[0] == '0');
        if (hub_on) split_hubs(c, lrows, nlong, hrows, nhub);
      }
      have = true;
    }
    const unsigned grid = grid_for((n + 31) / 32 * 32, 256);
    // The long rows (the hubs: their in-order fold is the superstep's
    // critical path) run on a side stream concurrently with the short rows;
    // both OR their validity bits into the zeroed words.
    GM_CUDA(cudaMemsetAsync(ybits, 0, (n + 31) / 32 * 4, s_));
    if constexpr (kHubPath) {
      if (nhub) {
        if (!hub_) {
          GM_CUDA(cudaStreamCreateWithFlags(&hub_, cudaStreamNonBlocking));
          GM_CUDA(cudaEventCreateWithFlags(&hfork_, cudaEventDisableTiming));
          GM_CUDA(cudaEventCreateWithFlags(&hjoin_, cudaEventDisableTiming));
          int dev = 0;
          GM_CUDA(cudaGetDevice(&dev));
          GM_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
        }
        GM_CUDA(cudaEventRecord(hfork_, s_));
        GM_CUDA(cudaStreamWaitEvent(hub_, hfork_, 0));
        // two 512-thread CTAs per SM: half the SM's threads, the rest for the
        // short- and mid-row kernels running beside it
        const unsigned hgrid = unsigned(std::min<uint64_t>(nhub, uint64_t(2 * sms_)));
        if (!hclaim_) hclaim_.alloc(1, s_);
        GM_CUDA(cudaMemsetAsync(hclaim_.get(), 0, 4, hub_));
        k_pull_hub<P><<<hgrid, kHubThreads, 0, hub_>>>(p_, hrows.get(), nhub, hclaim_.get(), c.ptr.get(),
                                                        c.idx.get(), c.val.get(), x_.get(),
                                                        xbits_.get(), n, props_.get(), y, ybits);
        GM_LAUNCH_CHECK();
      }
    }
    if (nlong) {
      if (!side_) {
        GM_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
        GM_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
        GM_CUDA(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));
      }
      GM_CUDA(cudaEventRecord(fork_, s_));
      GM_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
      bool pieces = false;
      if constexpr (can_push<P>::value) pieces = p_.direction() == Direction::OUT && y == y_.get();
      if constexpr (can_push<P>::value) {
       if (pieces) {
        if (!npieces_) {  // once per engine: pieces of <= kPiece entries of every long row
          DevBuf<uint64_t> cnt(nlong + 1, s_);
          k_piece_counts<<<grid_for(nlong + 1, 256), 256, 0, s_>>>(lrows.get(), nlong, c.ptr.get(),
                                                                  cnt.get());
          GM_LAUNCH_CHECK();
          exclusive_scan_u64(cnt.get(), nlong + 1, s_);
          GM_CUDA(cudaMemcpyAsync(&npieces_, cnt.get() + nlong, 8, cudaMemcpyDeviceToHost, s_));
          GM_CUDA(cudaStreamSynchronize(s_));
          prow_.alloc(npieces_ + 1, s_);
          pbeg_.alloc(npieces_ + 1, s_);
          k_piece_fill<<<grid_for(nlong, 256), 256, 0, s_>>>(lrows.get(), nlong, c.ptr.get(),
                                                            cnt.get(), prow_.get(), pbeg_.get());
          GM_LAUNCH_CHECK();
          GM_CUDA(cudaEventRecord(fork_, s_));
          GM_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
        }
        k_pull_pieces<P><<<grid_for(npieces_ * 32, 256), 256, 0, side_>>>(
            p_, prow_.get(), pbeg_.get(), npieces_, c.ptr.get(), c.idx.get(), c.val.get(), x_.get(),
            xbits_.get(), props_.get(), y, ybits);
       }
      }
      if (!pieces) {
        k_pull_long<P><<<grid_for(nlong * 32, kLongThreads), kLongThreads, 0, side_>>>(
            p_, lrows.get(), nlong, c.ptr.get(), c.idx.get(), c.val.get(), x_.get(), xbits_.get(),
            props_.get(), iperm(), y, ybits, err_.get());
      }
      GM_LAUNCH_CHECK();
    }
    if constexpr (exact_reorder<P>::value && !can_fail<P>::value)
      k_pull_group<P><<<grid, 256, 0, s_>>>(p_, n, c.ptr.get(), c.idx.get(), c.val.get(), x_.get(),
                                            xbits_.get(), props_.get(), y, ybits);
    else
      k_pull<P><<<grid, 256, 0, s_>>>(p_, n, c.ptr.get(), c.idx.get(), c.val.get(), x_.get(),
                                       xbits_.get(), props_.get(), iperm(), y, ybits, err_.get());
    GM_LAUNCH_CHECK();
    if (nlong) {
      GM_CUDA(cudaEventRecord(join_, side_));
      GM_CUDA(cudaStreamWaitEvent(s_, join_, 0));
    }
    if (nhub) {
      GM_CUDA(cudaEventRecord(hjoin_, hub_));
      GM_CUDA(cudaStreamWaitEvent(s_, hjoin_, 0));
    }
  }

  // After send(): the valid messages as a queue plus their out-edge count;
  // push when those edges are under 1/kPushDiv of the stored entries (the
  // pull visits every entry).  One host read per superstep.
  static constexpr uint64_t kPushDiv = 10;
  bool decide_push() {
    if constexpr (!can_push<P>::value) {
      return false;
    } else {
      if (p_.direction() != Direction::OUT || g_.n == 0) return false;
      ensure_forward(g_);
      const uint64_t n = g_.n;
      if (!q_) {
        q_.alloc(n + 1, s_);
        qctr_.alloc(2, s_);
      }
      qctr_.zero(s_);
      k_msg_queue<<<grid_for((n + 31) / 32, 256), 256, 0, s_>>>(n, xbits_.get(), g_.fwd().ptr.get(),
                                                                   q_.get(), qctr_.get());
      GM_LAUNCH_CHECK();
      unsigned long long h[2];
      GM_CUDA(cudaMemcpyAsync(h, qctr_.get(), 16, cudaMemcpyDeviceToHost, s_));
      GM_CUDA(cudaStreamSynchronize(s_));
      nq_ = h[0];
      push_edges_ = h[1];
      return h[1] * kPushDiv < g_.m;
    }
  }

  void push() {
    if constexpr (can_push<P>::value) {
      const uint64_t words = (g_.n + 31) / 32;
      GM_CUDA(cudaMemsetAsync(ybits_.get(), 0, words * 4, s_));
      const Csr& fw = g_.fwd();
      if (!qoff_) qoff_.alloc(g_.n + 2, s_);
      k_queue_degrees<<<grid_for(nq_ + 1, 256), 256, 0, s_>>>(q_.get(), qctr_.get(), fw.ptr.get(),
                                                          qoff_.get());
      GM_LAUNCH_CHECK();
      exclusive_scan_u64(qoff_.get(), nq_ + 1, s_);
      if (push_edges_)
        k_push<P><<<grid_for(push_edges_, 256), 256, 0, s_>>>(
            p_, q_.get(), qctr_.get(), qoff_.get(), fw.ptr.get(), fw.idx.get(), fw.val.get(),
            x_.get(), props_.get(), y_.get(), ybits_.get());
      GM_LAUNCH_CHECK();
    }
  }

  void spmv() {
    const uint64_t n = g_.n;
    const unsigned grid = grid_for((n + 31) / 32 * 32, 256);
    const Direction d = p_.direction();
    if (pushing_) {
      push();
      return;
    }
    const Csr& first = d == Direction::IN ? g_.fwd() : g_.in;
    pull(first, long1_, nlong1_, hub1_, nhub1_, have1_, y_.get(), ybits_.get());
    if (d == Direction::BOTH) {
      pull(g_.fwd(), long2_, nlong2_, hub2_, nhub2_, have2_, y2_.get(), y2bits_.get());
      k_merge<P><<<grid, 256, 0, s_>>>(p_, n, y_.get(), ybits_.get(), y2_.get(), y2bits_.get());
      GM_LAUNCH_CHECK();
    }
  }

  void apply() {
    const uint64_t n = g_.n;
    const unsigned grid = grid_for((n + 31) / 32, 256);  // a warp per 32 words
    k_apply<P><<<grid, 256, 0, s_>>>(p_, n, y_.get(), ybits_.get(), props_.get(), active_.get(),
                                      iperm(), ctr_.get(), err_.get());
    GM_LAUNCH_CHECK();
  }

  // Engine::step (engine.hpp:176-189).
  gm_iteration_stats step() {
    gm_iteration_stats st{};
    if (g_.n == 0) return st;
    ctr_.zero(s_);
    err_.zero(s_);
    GM_CUDA(cudaEventRecord(e0_, s_));
    send();
    pushing_ = decide_push();
    pushed_ = pushing_;
    GM_CUDA(cudaEventRecord(e1_, s_));
    spmv();
    pushing_ = false;
    GM_CUDA(cudaEventRecord(e2_, s_));
    // a failed SpMV aborts before apply (engine.hpp:251-257); programs without
    // failing callbacks cannot set the error word, so they skip both reads
    // (each was a host round trip per superstep)
    if constexpr (can_fail<P>::value) check_error();
    apply();
    GM_CUDA(cudaEventRecord(e3_, s_));
    unsigned long long c[3];
    GM_CUDA(cudaMemcpyAsync(c, ctr_.get(), sizeof(c), cudaMemcpyDeviceToHost, s_));
    GM_CUDA(cudaStreamSynchronize(s_));
    if constexpr (can_fail<P>::value) check_error();
    float spmv_ms = 0, total_ms = 0;
    GM_CUDA(cudaEventElapsedTime(&spmv_ms, e1_, e2_));
    GM_CUDA(cudaEventElapsedTime(&total_ms, e0_, e3_));
    st.active_before = int64_t(c[0]);
    st.messages_generated = int64_t(c[1]);
    st.vertices_updated = int64_t(c[2]);
    st.spmv_seconds = spmv_ms * 1e-3;
    st.total_seconds = total_ms * 1e-3;
    const Direction d = p_.direction();
    st.edges_processed = int64_t(d == Direction::BOTH ? 2 * g_.m : g_.m);
    st.direction = 0;
    if (pushed_) {
      st.edges_processed = int64_t(push_edges_);
      st.direction = 1;
    }
    return st;
  }

  // Engine::run_graph_program (engine.hpp:193-213).
  std::vector<gm_iteration_stats> run(int64_t max_iters) {
    std::vector<gm_iteration_stats> out;
    for (int64_t it = 1; it <= max_iters; ++it) {
      gm_iteration_stats st = step();
      st.iteration = it;
      out.push_back(st);
      if (st.vertices_updated == 0) break;
    }
    return out;
  }

  void check_error() {
    DevError h{};
    GM_CUDA(cudaMemcpyAsync(&h, err_.get(), sizeof(h), cudaMemcpyDeviceToHost, s_));
    GM_CUDA(cudaStreamSynchronize(s_));
    if (!h.code) return;
    const std::string what = P::error_message(h.code);
    switch (h.phase) {
      case kPhaseSend:
        fail(GM_EENGINE, "send_message failed at vertex " + std::to_string(h.vertex) + ": " + what);
      case kPhaseApply:
        fail(GM_EENGINE, "apply failed at vertex " + std::to_string(h.vertex) + ": " + what);
      default:
        fail(GM_EENGINE, "vertex program callback failed at (column " + std::to_string(h.col) +
                             ", row " + std::to_string(h.row) + "): " + what);
    }
  }

  const uint32_t* iperm() const { return g_.relabeled ? g_.iperm.get() : nullptr; }
  Graph& graph() { return g_; }
  DevBuf<M>& x() { return x_; }
  DevBuf<R>& y() { return y_; }
  DevBuf<uint32_t>& xbits() { return xbits_; }
  DevBuf<uint32_t>& ybits() { return ybits_; }
  cudaStream_t stream() const { return s_; }

 private:
  Graph& g_;
  P p_;
  cudaStream_t s_;
  DevBuf<V> props_;
  DevBuf<uint32_t> active_;
  DevBuf<M> x_;
  DevBuf<uint32_t> xbits_;
  DevBuf<R> y_, y2_;
  DevBuf<uint32_t> ybits_, y2bits_;
  DevBuf<uint32_t> long1_, long2_;  // long rows of the first / second route's CSR
  uint64_t nlong1_ = 0, nlong2_ = 0;
  DevBuf<uint32_t> hub1_, hub2_;    // hub rows (k_pull_hub), longest first
  DevBuf<unsigned> hclaim_;         // k_pull_hub's row counter
  uint64_t nhub1_ = 0, nhub2_ = 0;
  bool have1_ = false, have2_ = false;
  DevBuf<unsigned long long> ctr_;
  DevBuf<DevError> err_;
  DevBuf<uint32_t> q_;                 // push: valid message sources
  DevBuf<unsigned long long> qctr_;    // push: [count, their out-edges]
  DevBuf<uint64_t> qoff_;              // push: exclusive out-edge offsets over the queue
  DevBuf<uint32_t> prow_;              // pull pieces of the long rows (order-free programs)
  DevBuf<uint64_t> pbeg_;
  uint64_t npieces_ = 0;
  uint64_t push_edges_ = 0, nq_ = 0;
  bool pushing_ = false, pushed_ = false;
  cudaStream_t side_ = nullptr;  // long rows, concurrent with the short-row kernel
  cudaEvent_t fork_{}, join_{};
  cudaStream_t hub_ = nullptr;   // hub rows, concurrent with both
  cudaEvent_t hfork_{}, hjoin_{};
  int sms_ = 148;
  cudaEvent_t e0_{}, e1_{}, e2_{}, e3_{};
};

}  // namespace gm
