// ingest.cu -- GPU graph ingest: generators, preprocess, relabel, CSR build.
//
// Replaces, on the device:
//   io::rmat_generate / bipartite_generate   src/io.cpp:224-288  (counter-based, seeded)
//   io::preprocess                           src/io.cpp:184-222  (drop loops, dedup keep-first,
//                                                                 SYMMETRIZE)
//   build_graph / build_dcsc_partitions      include/semigraph/dcsc.hpp:110-164, 243-274
//   Graph::ensure_forward                    include/semigraph/dcsc.hpp:201-215
//   degree_vector                            include/semigraph/engine.hpp:295-312
// Sorting uses CUB radix sort on packed (row << nb | col) keys; CUB's sort is
// stable, which gives the reference's "keep the first of each duplicate".
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>
#include <string>
#include <vector>

#include "graph.cuh"

namespace gm {
namespace {

constexpr unsigned kBlock = 256;

// ------------------------------------------------------------ CUB wrappers
void sort_pairs(DevBuf<uint64_t>& keys, DevBuf<uint32_t>& vals, int64_t m, int end_bit,
                cudaStream_t s) {
  if (m <= 1) return;
  DevBuf<uint64_t> k2(m, s);
  DevBuf<uint32_t> v2(m, s);
  cub::DoubleBuffer<uint64_t> dk(keys.get(), k2.get());
  cub::DoubleBuffer<uint32_t> dv(vals.get(), v2.get());
  size_t tmp = 0;
  GM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, m, 0, end_bit, s));
  DevBuf<uint8_t> t(tmp, s);
  GM_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, dk, dv, m, 0, end_bit, s));
  if (dk.Current() != keys.get()) {
    keys.swap(k2);
    vals.swap(v2);
  }
}

void sort_keys(DevBuf<uint64_t>& keys, int64_t m, int end_bit, cudaStream_t s) {
  if (m <= 1) return;
  DevBuf<uint64_t> k2(m, s);
  cub::DoubleBuffer<uint64_t> dk(keys.get(), k2.get());
  size_t tmp = 0;
  GM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, dk, m, 0, end_bit, s));
  DevBuf<uint8_t> t(tmp, s);
  GM_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, dk, m, 0, end_bit, s));
  if (dk.Current() != keys.get()) keys.swap(k2);
}

// In-place stable compaction (no second m-sized buffer: at scale 28 the key
// array alone is 34-69 GB).
template <typename T>
int64_t select_flagged(DevBuf<T>& data, const uint8_t* flags, int64_t m, cudaStream_t s) {
  if (m == 0) return 0;
  DevBuf<int64_t> cnt(1, s);
  size_t tmp = 0;
  GM_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, data.get(), flags, cnt.get(), m, s));
  DevBuf<uint8_t> t(tmp, s);
  GM_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, data.get(), flags, cnt.get(), m, s));
  int64_t h = 0;
  GM_CUDA(cudaMemcpyAsync(&h, cnt.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

void exclusive_scan_to_ptr(const uint32_t* counts, uint64_t* ptr, uint64_t n, cudaStream_t s);

// ------------------------------------------------------------------ kernels
__global__ void k_ids_u64(const uint64_t* s, const uint64_t* d, int64_t m, uint64_t n,
                          uint32_t* s32, uint32_t* d32, unsigned long long* bad) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t a = s[e], b = d[e];
    if (a >= n || b >= n) atomicMin(bad, (unsigned long long)e);
    s32[e] = uint32_t(a);
    d32[e] = uint32_t(b);
  }
}

__global__ void k_check_u32(const uint32_t* s, const uint32_t* d, int64_t m, uint64_t n,
                            unsigned long long* bad) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
       e += int64_t(gridDim.x) * blockDim.x)
    if (s[e] >= n || d[e] >= n) atomicMin(bad, (unsigned long long)e);
}

__global__ void k_make_keys(const uint32_t* s, const uint32_t* d, int64_t m, unsigned nb,
                            uint64_t* keys, uint32_t* idx, uint8_t* keep, int drop_loops) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
       e += int64_t(gridDim.x) * blockDim.x) {
    keys[e] = (uint64_t(s[e]) << nb) | d[e];
    if (idx) idx[e] = uint32_t(e);
    keep[e] = drop_loops ? (s[e] != d[e]) : 1;
  }
}

__global__ void k_unique_flags(const uint64_t* keys, int64_t m, uint8_t* flag,
                               unsigned long long* first_dup) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool u = i == 0 || keys[i] != keys[i - 1];
    flag[i] = u;
    if (!u && first_dup) atomicMin(first_dup, (unsigned long long)i);
  }
}

__global__ void k_append_reverse(uint64_t* keys, uint32_t* idx, int64_t m, unsigned nb) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    keys[m + i] = ((k & mask) << nb) | (k >> nb);
    if (idx) idx[m + i] = idx[i];
  }
}

// DAGIFY (io.cpp:206): keep src < dst.
__global__ void k_dag_flags(const uint64_t* keys, int64_t m, unsigned nb, uint8_t* keep) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    keep[i] = (keys[i] >> nb) < (keys[i] & mask);
}

// BIPARTITE_CHECK (io.cpp:208-219): the first edge (sorted order) whose source
// is some edge's destination or whose destination is some edge's source.
__global__ void k_bipartite_first(const uint64_t* keys, int64_t m, unsigned nb,
                                  const uint32_t* outdeg, const uint32_t* indeg,
                                  unsigned long long* first) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    if (indeg[keys[i] >> nb] || outdeg[keys[i] & mask]) atomicMin(first, (unsigned long long)i);
}

__global__ void k_degrees(const uint64_t* keys, int64_t m, unsigned nb, uint32_t* outdeg,
                          uint32_t* indeg) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    atomicAdd(&outdeg[keys[i] >> nb], 1u);
    atomicAdd(&indeg[keys[i] & mask], 1u);
  }
}

__global__ void k_relabel_keys(const uint32_t* outdeg, uint64_t n, uint64_t* keys) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    keys[v] = (uint64_t(0xFFFFFFFFu - outdeg[v]) << 32) | v;
}

// Degree rank k -> internal id; with P shards the ranks are dealt round-robin
// over P contiguous blocks of n/P ids (each block hub-first, nnz-balanced).
__global__ void k_perm_from_keys(const uint64_t* keys, uint64_t n, uint32_t shards, uint32_t* perm,
                                 uint32_t* iperm) {
  const uint64_t block = n / shards;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = uint32_t(keys[k]);
    const uint64_t i = (k % shards) * block + k / shards;
    iperm[i] = v;
    perm[v] = uint32_t(i);
  }
}

template <typename T>
__global__ void k_gather(const T* in, const uint32_t* idx, uint64_t n, T* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = in[idx[i]];
}

// Transposed key: (col_src, row_dst) of an external (s<<nb|d) key -> internal
// CSR(G^T) key (perm(d) << nb | perm(s)).
__global__ void k_transpose_keys(uint64_t* keys, int64_t m, unsigned nb, const uint32_t* perm) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t s = keys[i] >> nb, d = keys[i] & mask;
    if (perm) {
      s = perm[s];
      d = perm[d];
    }
    keys[i] = (d << nb) | s;
  }
}

__global__ void k_low_bits(const uint64_t* keys, int64_t m, uint64_t mask, uint32_t* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(keys[i] & mask);
}

// For every CSR entry: key = (col << nb) | row, payload = entry index.
__global__ void k_entry_keys_transposed(const uint64_t* ptr, const uint32_t* idx, uint64_t n,
                                        int64_t nnz, unsigned nb, uint64_t* keys,
                                        uint32_t* payload) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x) {
    // row = last r with ptr[r] <= e
    uint64_t lo = 0, hi = n;  // search in [0, n)
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (ptr[mid] <= uint64_t(e))
        lo = mid;
      else
        hi = mid;
    }
    keys[e] = (uint64_t(idx[e]) << nb) | lo;
    payload[e] = uint32_t(e);
  }
}

__global__ void k_export_keys(const uint64_t* ptr, const uint32_t* idx, uint64_t n, int64_t nnz,
                              unsigned nb, const uint32_t* iperm, uint64_t* keys,
                              uint32_t* payload) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (ptr[mid] <= uint64_t(e))
        lo = mid;
      else
        hi = mid;
    }
    uint32_t src = idx[e], dst = uint32_t(lo);
    if (iperm) {
      src = iperm[src];
      dst = iperm[dst];
    }
    keys[e] = (uint64_t(src) << nb) | dst;
    payload[e] = uint32_t(e);
  }
}

template <typename In, typename Out>
__global__ void k_convert(const In* in, int64_t m, Out* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<Out>(in[i]);
}

__global__ void k_rmat(uint64_t count, unsigned scale, uint64_t ta, uint64_t tab, uint64_t tabc,
                       uint32_t k0, uint32_t k1, PermKeys pk, int permute, uint32_t* src,
                       uint32_t* dst, uint64_t t0 = 0) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t t = t0 + i;  // tuple id: counter of the generator
    uint32_t s = 0, d = 0;
    for (unsigned l = 0; l < scale; l += 4) {
      uint32_t out[4];
      philox4x32_10(uint32_t(t), uint32_t(t >> 32), l >> 2, 0x524D4154u, k0, k1, out);
#pragma unroll
      for (unsigned q = 0; q < 4; ++q) {
        if (l + q >= scale) break;
        const uint64_t r = out[q];
        const uint32_t bit = 1u << (scale - 1 - (l + q));
        if (r < ta) {
        } else if (r < tab) {
          d |= bit;
        } else if (r < tabc) {
          s |= bit;
        } else {
          s |= bit;
          d |= bit;
        }
      }
    }
    if (permute) {
      s = perm_apply(pk, s);
      d = perm_apply(pk, d);
    }
    src[i] = s;
    dst[i] = d;
  }
}

__global__ void k_bip_degree(uint32_t users, double c, uint32_t cap, uint32_t* deg) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < users; u += gridDim.x * blockDim.x) {
    double dd = floor(c / double(u + 1));
    if (dd < 1.0) dd = 1.0;
    if (dd > double(cap)) dd = double(cap);
    deg[u] = uint32_t(dd);
  }
}

__global__ void k_bip_draw(const uint64_t* off, uint32_t users, uint32_t items,
                           const uint64_t* thr, uint32_t k0, uint32_t k1, uint32_t* src,
                           uint32_t* dst, uint64_t t0 = 0, uint64_t t1 = ~0ull) {
  const uint64_t total = off[users] < t1 ? off[users] : t1;
  for (uint64_t t = t0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t lo = 0, hi = users;  // last u with off[u] <= t
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (off[mid] <= t)
        lo = mid;
      else
        hi = mid;
    }
    const uint32_t u = lo;
    const uint32_t k = uint32_t(t - off[u]);
    uint32_t w[4];
    philox4x32_10(u, k >> 2, 0, 0x42495054u, k0, k1, w);
    const uint64_t r = w[k & 3u];
    uint32_t a = 0, b = items - 1;
    while (a < b) {
      const uint32_t mid = a + (b - a) / 2;
      if (r < thr[mid])
        b = mid;
      else
        a = mid + 1;
    }
    src[t - t0] = u;
    dst[t - t0] = users + a;
  }
}

// Per CSR(G^T) entry values derived from caller ids (weights / ratings).
__global__ void k_entry_weights(const uint64_t* ptr, const uint32_t* idx, uint64_t n, int64_t nnz,
                                const uint32_t* iperm, uint64_t seed_w, int mode, uint8_t* out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (ptr[mid] <= uint64_t(e))
        lo = mid;
      else
        hi = mid;
    }
    uint32_t dst = uint32_t(lo), src = idx[e];
    if (iperm) {
      dst = iperm[dst];
      src = iperm[src];
    }
    out[e] = mode == 0 ? edge_weight(seed_w, src, dst) : rating_of(seed_w, src, dst);
  }
}

template <typename T>
__global__ void k_gather_ext(const T* in, const uint32_t* perm, uint64_t n, T* out) {
  // out[v] = in[perm[v]]  (internal -> caller order)
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    out[v] = in[perm[v]];
}

__global__ void k_count_nonzero(const uint32_t* deg, uint64_t n, unsigned long long* cnt) {
  unsigned long long c = 0;
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    c += deg[v] > 0;
  warp_add_u64(cnt, c);
}

__global__ void k_widen(const uint32_t* in, uint64_t n, uint64_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

void exclusive_scan_to_ptr(const uint32_t* counts, uint64_t* ptr, uint64_t n, cudaStream_t s) {
  // ptr[0] = 0, ptr[i+1] = sum counts[0..i].  The counts are widened to u64
  // first: CUB accumulates in the input type, and above 2^32 stored entries
  // (scale-28 R-MAT) a u32 running sum wraps.
  GM_CUDA(cudaMemsetAsync(ptr, 0, sizeof(uint64_t), s));
  if (n == 0) return;
  k_widen<<<grid_for(n, 256), 256, 0, s>>>(counts, n, ptr + 1);
  GM_LAUNCH_CHECK();
  size_t tmp = 0;
  GM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, ptr + 1, ptr + 1, int64_t(n), s));
  DevBuf<uint8_t> t(tmp, s);
  GM_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, ptr + 1, ptr + 1, int64_t(n), s));
}

template <typename F>
void launch(uint64_t work, cudaStream_t s, F&& f) {
  if (work == 0) return;
  f(grid_for(work, kBlock), kBlock);
  GM_LAUNCH_CHECK();
}

uint64_t read_u64(const unsigned long long* p, cudaStream_t s) {
  unsigned long long h = 0;
  GM_CUDA(cudaMemcpyAsync(&h, p, sizeof(h), cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Convert caller values (any gm_value_type) to the storage type, on device.
void convert_values(const void* in, int in_type, int64_t m, void* out, int out_type,
                    cudaStream_t s) {
  if (out_type == GM_VAL_NONE || m == 0) return;
#define GM_CONV_OUT(InT)                                                                         \
  switch (out_type) {                                                                            \
    case GM_VAL_F64: launch(m, s, [&](unsigned g, unsigned b) { k_convert<<<g, b, 0, s>>>((const InT*)in, m, (double*)out); }); break; \
    case GM_VAL_F32: launch(m, s, [&](unsigned g, unsigned b) { k_convert<<<g, b, 0, s>>>((const InT*)in, m, (float*)out); }); break; \
    case GM_VAL_U8: launch(m, s, [&](unsigned g, unsigned b) { k_convert<<<g, b, 0, s>>>((const InT*)in, m, (uint8_t*)out); }); break; \
    case GM_VAL_I64: launch(m, s, [&](unsigned g, unsigned b) { k_convert<<<g, b, 0, s>>>((const InT*)in, m, (int64_t*)out); }); break; \
    case GM_VAL_U32: launch(m, s, [&](unsigned g, unsigned b) { k_convert<<<g, b, 0, s>>>((const InT*)in, m, (uint32_t*)out); }); break; \
    default: fail(GM_EUSAGE, "unsupported value storage type");                                \
  }
  switch (in_type) {
    case GM_VAL_F64: GM_CONV_OUT(double) break;
    case GM_VAL_F32: GM_CONV_OUT(float) break;
    case GM_VAL_U8: GM_CONV_OUT(uint8_t) break;
    case GM_VAL_I64: GM_CONV_OUT(int64_t) break;
    case GM_VAL_U32: GM_CONV_OUT(uint32_t) break;
    default: fail(GM_EUSAGE, "unsupported input value type");
  }
#undef GM_CONV_OUT
}

void gather_values(const uint8_t* in, const uint32_t* idx, int64_t m, size_t vs, uint8_t* out,
                   cudaStream_t s) {
  switch (vs) {
    case 8: launch(m, s, [&](unsigned g, unsigned b) { k_gather<<<g, b, 0, s>>>((const uint64_t*)in, idx, m, (uint64_t*)out); }); break;
    case 4: launch(m, s, [&](unsigned g, unsigned b) { k_gather<<<g, b, 0, s>>>((const uint32_t*)in, idx, m, (uint32_t*)out); }); break;
    case 1: launch(m, s, [&](unsigned g, unsigned b) { k_gather<<<g, b, 0, s>>>(in, idx, m, out); }); break;
    default: break;
  }
}

// Core pipeline on device edge arrays (caller ids, already range-checked).
// values: storage-typed, parallel to the input edges, or null.
void build(Graph& g, DevBuf<uint32_t>& s32, DevBuf<uint32_t>& d32, int64_t m,
           DevBuf<uint8_t>& values) {
  cudaStream_t s = g.stream;
  const unsigned nb = g.nb;
  const int end_bit = int(2 * nb);
  const bool pre = (g.flags & (GM_PREPROCESS | GM_SYMMETRIZE | GM_DAGIFY | GM_BIPARTITE_CHECK)) != 0;
  const size_t vs = value_size(g.value_type);
  // The payload (input position of each edge, to carry its value through the
  // sorts) exists only when there are values: value-less graphs sort bare keys,
  // which is what lets scale-28 R-MAT (4.3e9 raw, 8.6e9 symmetrised) fit.
  const bool payload = vs && values;

  DevBuf<uint64_t> keys(m, s);
  DevBuf<uint32_t> idx(payload ? m : 0, s);
  {
    DevBuf<uint8_t> keep(m, s);
    launch(m, s, [&](unsigned gr, unsigned b) {
      k_make_keys<<<gr, b, 0, s>>>(s32.get(), d32.get(), m, nb, keys.get(),
                                   payload ? idx.get() : nullptr, keep.get(), pre ? 1 : 0);
    });
    s32.reset();
    d32.reset();
    if (pre) {
      if (payload) select_flagged(idx, keep.get(), m, s);
      m = select_flagged(keys, keep.get(), m, s);
    }
  }
  auto sort = [&]() {
    if (payload)
      sort_pairs(keys, idx, m, end_bit, s);
    else
      sort_keys(keys, m, end_bit, s);
  };
  auto dedup = [&](bool allow_dups) {
    sort();
    DevBuf<uint8_t> flag(m, s);
    DevBuf<unsigned long long> dup(1, s);
    GM_CUDA(cudaMemsetAsync(dup.get(), 0xFF, sizeof(unsigned long long), s));
    launch(m, s, [&](unsigned gr, unsigned b) {
      k_unique_flags<<<gr, b, 0, s>>>(keys.get(), m, flag.get(), dup.get());
    });
    const uint64_t first = read_u64(dup.get(), s);
    if (first != ~0ull) {
      if (!allow_dups) {
        uint64_t k = 0;
        GM_CUDA(cudaMemcpy(&k, keys.get() + first, sizeof(k), cudaMemcpyDeviceToHost));
        const uint64_t mask = (uint64_t(1) << nb) - 1;
        fail(GM_EINPUT, "duplicate edge " + std::to_string((k >> nb) + 1) + " -> " +
                            std::to_string((k & mask) + 1) +
                            " (1-based); deduplicate before building");
      }
      if (payload) select_flagged(idx, flag.get(), m, s);
      m = select_flagged(keys, flag.get(), m, s);
    }
  };
  dedup(pre);
  if (g.flags & (GM_SYMMETRIZE | GM_DAGIFY)) {
    DevBuf<uint64_t> k2(2 * m, s);
    DevBuf<uint32_t> i2(payload ? 2 * m : 0, s);
    if (m) {
      GM_CUDA(cudaMemcpyAsync(k2.get(), keys.get(), m * 8, cudaMemcpyDeviceToDevice, s));
      if (payload) GM_CUDA(cudaMemcpyAsync(i2.get(), idx.get(), m * 4, cudaMemcpyDeviceToDevice, s));
    }
    keys.reset();
    idx.reset();
    launch(m, s, [&](unsigned gr, unsigned b) {
      k_append_reverse<<<gr, b, 0, s>>>(k2.get(), payload ? i2.get() : nullptr, m, nb);
    });
    keys.swap(k2);
    idx.swap(i2);
    k2.reset();
    i2.reset();
    m *= 2;
    dedup(true);
    if (g.flags & GM_DAGIFY) {
      DevBuf<uint8_t> keep(m, s);
      launch(m, s, [&](unsigned gr, unsigned b) { k_dag_flags<<<gr, b, 0, s>>>(keys.get(), m, nb, keep.get()); });
      if (payload) select_flagged(idx, keep.get(), m, s);
      m = select_flagged(keys, keep.get(), m, s);
    }
  }
  g.m = uint64_t(m);

  // Degrees in caller order.
  const uint64_t n = g.n;
  DevBuf<uint32_t> outdeg(n, s), indeg(n, s);
  outdeg.zero(s);
  indeg.zero(s);
  launch(m, s, [&](unsigned gr, unsigned b) {
    k_degrees<<<gr, b, 0, s>>>(keys.get(), m, nb, outdeg.get(), indeg.get());
  });
  if (g.flags & GM_BIPARTITE_CHECK) {
    DevBuf<unsigned long long> first(1, s);
    GM_CUDA(cudaMemsetAsync(first.get(), 0xFF, sizeof(unsigned long long), s));
    launch(m, s, [&](unsigned gr, unsigned b) {
      k_bipartite_first<<<gr, b, 0, s>>>(keys.get(), m, nb, outdeg.get(), indeg.get(), first.get());
    });
    const uint64_t e = read_u64(first.get(), s);
    if (e != ~0ull) {
      uint64_t k = 0;
      GM_CUDA(cudaMemcpy(&k, keys.get() + e, sizeof(k), cudaMemcpyDeviceToHost));
      const uint64_t mask = (uint64_t(1) << nb) - 1;
      fail(GM_EINPUT, "not bipartite: edge " + std::to_string((k >> nb) + 1) + " -> " +
                          std::to_string((k & mask) + 1) + " (1-based) mixes the user and item sides");
    }
  }

  // Relabel: internal id = rank by (out-degree desc, caller id asc).
  if (g.flags & GM_RELABEL) {
    g.relabeled = true;
    DevBuf<uint64_t> rk(n, s);
    launch(n, s, [&](unsigned gr, unsigned b) { k_relabel_keys<<<gr, b, 0, s>>>(outdeg.get(), n, rk.get()); });
    sort_keys(rk, int64_t(n), 64, s);
    g.perm.alloc(n, s);
    g.iperm.alloc(n, s);
    const uint32_t shards = g.shards;
    launch(n, s, [&](unsigned gr, unsigned b) {
      k_perm_from_keys<<<gr, b, 0, s>>>(rk.get(), n, shards, g.perm.get(), g.iperm.get());
    });
    g.outdeg.alloc(n, s);
    g.indeg.alloc(n, s);
    launch(n, s, [&](unsigned gr, unsigned b) {
      k_gather<<<gr, b, 0, s>>>(outdeg.get(), g.iperm.get(), n, g.outdeg.get());
      k_gather<<<gr, b, 0, s>>>(indeg.get(), g.iperm.get(), n, g.indeg.get());
    });
  } else {
    g.outdeg = std::move(outdeg);
    g.indeg = std::move(indeg);
  }
  {
    DevBuf<unsigned long long> c(1, s);
    c.zero(s);
    launch(n, s, [&](unsigned gr, unsigned b) { k_count_nonzero<<<gr, b, 0, s>>>(g.outdeg.get(), n, c.get()); });
    g.nonzero_outdeg = read_u64(c.get(), s);
  }

  // CSR(G^T): key (dst_int << nb | src_int), payload = value index.
  launch(m, s, [&](unsigned gr, unsigned b) {
    k_transpose_keys<<<gr, b, 0, s>>>(keys.get(), m, nb, g.relabeled ? g.perm.get() : nullptr);
  });
  sort();
  g.in.n = n;
  g.in.nnz = uint64_t(m);
  g.in.ptr.alloc(n + 1, s);
  exclusive_scan_to_ptr(g.indeg.get(), g.in.ptr.get(), n, s);
  g.in.idx.alloc(m, s);
  launch(m, s, [&](unsigned gr, unsigned b) {
    k_low_bits<<<gr, b, 0, s>>>(keys.get(), m, (uint64_t(1) << nb) - 1, g.in.idx.get());
  });
  keys.reset();
  if (payload) {
    g.in.val.alloc(size_t(m) * vs, s);
    gather_values(values.get(), idx.get(), m, vs, g.in.val.get(), s);
  }
  idx.reset();
  values.reset();
  g.out_alias = g.symmetric && vs == 0;
  if (g.out_alias) g.out_built = true;
  GM_CUDA(cudaStreamSynchronize(s));
}

Graph* new_graph(uint64_t n, uint32_t flags, int storage) {
  if (n > 0xFFFFFFFFull) fail(GM_EUSAGE, "graphs above 2^32-1 vertices are not supported");
  uint32_t shards = (flags >> 16) & 0xFFu;
  if (shards == 0) shards = 1;
  if (shards > 1 && !(flags & GM_RELABEL)) fail(GM_EUSAGE, "GM_SHARDS needs GM_RELABEL");
  if (shards > 1 && n % shards != 0)
    fail(GM_EUSAGE, "GM_SHARDS(" + std::to_string(shards) + "): vertex count " + std::to_string(n) +
                        " is not a multiple of the shard count");
  if ((flags & GM_SYMMETRIZE) && (flags & (GM_DAGIFY | GM_BIPARTITE_CHECK)))
    fail(GM_EUSAGE, "SYMMETRIZE, DAGIFY and BIPARTITE_CHECK are exclusive preprocessing modes");
  if ((flags & GM_DAGIFY) && (flags & GM_BIPARTITE_CHECK))
    fail(GM_EUSAGE, "SYMMETRIZE, DAGIFY and BIPARTITE_CHECK are exclusive preprocessing modes");
  auto* g = new Graph();
  g->shards = shards;
  GM_CUDA(cudaGetDevice(&g->device));
  GM_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  {  // Keep up to 4 GB of freed stream-ordered allocations mapped: with the
     // default threshold (0) every per-call scratch buffer (e.g. the result
     // permutation of a 33 MB rank vector) is unmapped at each synchronize and
     // remapped by the next call, which made end-to-end calls erratic.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
      uint64_t keep = 4ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  g->n = n;
  g->flags = flags;
  if (flags & (GM_SYMMETRIZE | GM_DAGIFY | GM_BIPARTITE_CHECK)) g->flags |= GM_PREPROCESS;
  g->symmetric = (flags & GM_SYMMETRIZE) != 0;
  g->value_type = storage;
  g->nb = bits_for(n);
  return g;
}

}  // namespace

uint64_t Graph::device_bytes() const {
  return perm.bytes() + iperm.bytes() + outdeg.bytes() + indeg.bytes() + in.ptr.bytes() +
         in.idx.bytes() + in.val.bytes() + out.ptr.bytes() + out.idx.bytes() + out.val.bytes();
}

Graph* graph_create(const gm_edge_list& e, uint64_t n, uint32_t flags, int storage) {
  if (e.count < 0) fail(GM_EUSAGE, "negative edge count");
  if (e.count > 0 && (!e.src || !e.dst)) fail(GM_EUSAGE, "null edge arrays");
  if (e.count >= int64_t(0xFFFFFFFFll)) fail(GM_EUSAGE, "more than 2^32-2 input edges");
  if (n == 0 && e.count > 0)
    fail(GM_EINPUT, "build_graph: zero vertices but " + std::to_string(e.count) + " edges");
  if (value_size(storage) == 0 && storage != GM_VAL_NONE) fail(GM_EUSAGE, "bad value storage type");
  std::unique_ptr<Graph> g(new_graph(n, flags, storage));
  cudaStream_t s = g->stream;
  const int64_t m = e.count;
  DevBuf<uint32_t> s32(m, s), d32(m, s);
  DevBuf<unsigned long long> bad(1, s);
  GM_CUDA(cudaMemsetAsync(bad.get(), 0xFF, sizeof(unsigned long long), s));
  const cudaMemcpyKind kind = e.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (e.id_type == GM_ID_U64) {
    DevBuf<uint64_t> s64(m, s), d64(m, s);
    if (m) {
      GM_CUDA(cudaMemcpyAsync(s64.get(), e.src, m * 8, kind, s));
      GM_CUDA(cudaMemcpyAsync(d64.get(), e.dst, m * 8, kind, s));
    }
    launch(m, s, [&](unsigned gr, unsigned b) {
      k_ids_u64<<<gr, b, 0, s>>>(s64.get(), d64.get(), m, n, s32.get(), d32.get(), bad.get());
    });
  } else if (e.id_type == GM_ID_U32) {
    if (m) {
      GM_CUDA(cudaMemcpyAsync(s32.get(), e.src, m * 4, kind, s));
      GM_CUDA(cudaMemcpyAsync(d32.get(), e.dst, m * 4, kind, s));
    }
    launch(m, s, [&](unsigned gr, unsigned b) { k_check_u32<<<gr, b, 0, s>>>(s32.get(), d32.get(), m, n, bad.get()); });
  } else {
    fail(GM_EUSAGE, "bad id type");
  }
  const uint64_t first_bad = read_u64(bad.get(), s);
  if (first_bad != ~0ull) {
    uint64_t a = 0, b = 0;
    if (e.id_type == GM_ID_U64) {
      if (e.on_device) {
        GM_CUDA(cudaMemcpy(&a, (const uint64_t*)e.src + first_bad, 8, cudaMemcpyDeviceToHost));
        GM_CUDA(cudaMemcpy(&b, (const uint64_t*)e.dst + first_bad, 8, cudaMemcpyDeviceToHost));
      } else {
        a = ((const uint64_t*)e.src)[first_bad];
        b = ((const uint64_t*)e.dst)[first_bad];
      }
    } else {
      uint32_t a32 = 0, b32 = 0;
      GM_CUDA(cudaMemcpy(&a32, s32.get() + first_bad, 4, cudaMemcpyDeviceToHost));
      GM_CUDA(cudaMemcpy(&b32, d32.get() + first_bad, 4, cudaMemcpyDeviceToHost));
      a = a32;
      b = b32;
    }
    fail(GM_EINPUT, "build_graph: edge " + std::to_string(a + 1) + " -> " + std::to_string(b + 1) +
                        " (1-based) exceeds vertex count " + std::to_string(n));
  }
  DevBuf<uint8_t> vals;
  const size_t vs = value_size(storage);
  if (vs && m) {
    vals.alloc(size_t(m) * vs, s);
    if (e.values) {
      const size_t ivs = value_size(e.value_type);
      if (!ivs) fail(GM_EUSAGE, "values given with value_type none");
      DevBuf<uint8_t> raw;
      const void* src_vals = e.values;
      if (!e.on_device) {
        raw.alloc(size_t(m) * ivs, s);
        GM_CUDA(cudaMemcpyAsync(raw.get(), e.values, size_t(m) * ivs, cudaMemcpyHostToDevice, s));
        src_vals = raw.get();
      }
      convert_values(src_vals, e.value_type, m, vals.get(), storage, s);
      GM_CUDA(cudaStreamSynchronize(s));
    } else {
      // Unweighted input: every edge carries value 1 (io.hpp:26-28).
      DevBuf<uint8_t> ones(m, s);
      GM_CUDA(cudaMemsetAsync(ones.get(), 1, m, s));
      convert_values(ones.get(), GM_VAL_U8, m, vals.get(), storage, s);
      GM_CUDA(cudaStreamSynchronize(s));
    }
  }
  build(*g, s32, d32, m, vals);
  if (flags & GM_NEED_FORWARD) ensure_forward(*g);
  return g.release();
}

// ---- helpers shared with the sharded ingest (dist.cu, ingest.cuh) ----------
void rmat_range(unsigned scale, double a, double b, double c, uint64_t seed, int permute,
                uint64_t t0, uint64_t count, uint32_t* src, uint32_t* dst, cudaStream_t s) {
  const PermKeys pk = make_perm_keys(scale, seed);
  const uint64_t ta = prob_threshold(a), tab = prob_threshold(a + b), tabc = prob_threshold(a + b + c);
  launch(count, s, [&](unsigned gr, unsigned bl) {
    k_rmat<<<gr, bl, 0, s>>>(count, scale, ta, tab, tabc, uint32_t(seed), uint32_t(seed >> 32), pk,
                             permute, src, dst, t0);
  });
}

// The seeded Zipf bipartite stream (graph_generate_bipartite below): total
// raw ratings, and the ratings [t0, t1) of it (user-major, counter based).
struct BipStream {
  DevBuf<uint64_t> thr, off;
  uint64_t total = 0;
};

static BipStream bip_stream(uint32_t users, uint32_t items, double c_num, uint32_t cap,
                            cudaStream_t s) {
  BipStream b;
  std::vector<uint64_t> thr(items);
  double tot = 0.0;
  for (uint32_t j = 1; j <= items; ++j) tot += std::pow(double(j), -0.8);
  double cum = 0.0;
  for (uint32_t j = 1; j <= items; ++j) {
    cum += std::pow(double(j), -0.8);
    thr[j - 1] = j == items ? (1ull << 32) : uint64_t(cum / tot * 4294967296.0);
  }
  b.thr.alloc(items, s);
  GM_CUDA(cudaMemcpyAsync(b.thr.get(), thr.data(), items * 8, cudaMemcpyHostToDevice, s));
  DevBuf<uint32_t> deg(users, s);
  launch(users, s, [&](unsigned gr, unsigned bl) { k_bip_degree<<<gr, bl, 0, s>>>(users, c_num, cap, deg.get()); });
  b.off.alloc(uint64_t(users) + 1, s);
  exclusive_scan_to_ptr(deg.get(), b.off.get(), users, s);
  GM_CUDA(cudaMemcpyAsync(&b.total, b.off.get() + users, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return b;
}

uint64_t bipartite_range(uint32_t users, uint32_t items, double c_num, uint32_t cap, uint64_t seed,
                         uint64_t part, uint64_t parts, uint32_t* src, uint32_t* dst,
                         uint64_t* total_out, cudaStream_t s) {
  BipStream b = bip_stream(users, items, c_num, cap, s);
  const uint64_t t0 = b.total * part / parts, t1 = b.total * (part + 1) / parts;
  if (total_out) *total_out = b.total;
  if (src && t1 > t0)
    launch(t1 - t0, s, [&](unsigned gr, unsigned bl) {
      k_bip_draw<<<gr, bl, 0, s>>>(b.off.get(), users, items, b.thr.get(), uint32_t(seed),
                                   uint32_t(seed >> 32), src, dst, t0, t1);
    });
  GM_CUDA(cudaStreamSynchronize(s));
  return t1 - t0;
}

void sort_keys_u64(DevBuf<uint64_t>& keys, int64_t m, int end_bit, cudaStream_t s) {
  sort_keys(keys, m, end_bit, s);
}

int64_t unique_keys_u64(DevBuf<uint64_t>& keys, int64_t m, cudaStream_t s) {
  if (m <= 1) return m;
  DevBuf<uint8_t> flag(m, s);
  launch(uint64_t(m), s, [&](unsigned gr, unsigned bl) {
    k_unique_flags<<<gr, bl, 0, s>>>(keys.get(), m, flag.get(), nullptr);
  });
  return select_flagged(keys, flag.get(), m, s);
}

void scan_counts_to_ptr(const uint32_t* counts, uint64_t* ptr, uint64_t n, cudaStream_t s) {
  exclusive_scan_to_ptr(counts, ptr, n, s);
}

Graph* graph_generate_rmat(uint32_t scale, uint32_t ef, double a, double b, double c,
                           uint64_t seed, int permute, uint32_t flags, int weights) {
  if (scale == 0 || scale > 31) fail(GM_EUSAGE, "rmat: scale must be in [1, 31]");
  if (!(a >= 0.0 && b >= 0.0 && c >= 0.0 && a + b + c <= 1.0))
    fail(GM_EINPUT, "rmat: quadrant probabilities must be non-negative and sum to at most 1");
  const uint64_t count = uint64_t(ef) << scale;
  // no payload (weights are derived from ids after the build): 2^36 raw edges
  if (count > (uint64_t(1) << 36)) fail(GM_EUSAGE, "rmat: more than 2^36 raw edges");
  if (weights != GM_VAL_NONE && weights != GM_VAL_U8) fail(GM_EUSAGE, "rmat: weights must be none or u8");
  const uint64_t n = uint64_t(1) << scale;
  std::unique_ptr<Graph> g(new_graph(n, flags, weights));
  cudaStream_t s = g->stream;
  DevBuf<uint32_t> s32(count, s), d32(count, s);
  const PermKeys pk = make_perm_keys(scale, seed);
  const uint64_t ta = prob_threshold(a), tab = prob_threshold(a + b), tabc = prob_threshold(a + b + c);
  launch(count, s, [&](unsigned gr, unsigned bl) {
    k_rmat<<<gr, bl, 0, s>>>(count, scale, ta, tab, tabc, uint32_t(seed), uint32_t(seed >> 32), pk,
                             permute, s32.get(), d32.get());
  });
  DevBuf<uint8_t> none;
  const int storage = g->value_type;
  g->value_type = GM_VAL_NONE;  // structure first; weights derived from caller ids below
  build(*g, s32, d32, int64_t(count), none);
  if (weights == GM_VAL_U8) {
    g->value_type = storage;
    g->out_alias = false;
    if (g->symmetric) g->out_built = false;
    g->in.val.alloc(g->in.nnz, s);
    const uint64_t seed_w = mix64(seed ^ 0x57E16475ull);
    launch(g->in.nnz, s, [&](unsigned gr, unsigned bl) {
      k_entry_weights<<<gr, bl, 0, s>>>(g->in.ptr.get(), g->in.idx.get(), g->n, int64_t(g->in.nnz),
                                        g->relabeled ? g->iperm.get() : nullptr, seed_w, 0,
                                        g->in.val.get());
    });
    GM_CUDA(cudaStreamSynchronize(s));
  }
  if (flags & GM_NEED_FORWARD) ensure_forward(*g);
  return g.release();
}

Graph* graph_generate_bipartite(uint32_t users, uint32_t items, double c_num, uint32_t cap,
                                uint64_t seed, uint32_t flags) {
  if (users == 0 || items == 0) fail(GM_EUSAGE, "bipartite: need users and items");
  const uint64_t n = uint64_t(users) + items;
  std::unique_ptr<Graph> g(new_graph(n, flags | GM_PREPROCESS, GM_VAL_NONE));
  cudaStream_t s = g->stream;
  // Zipf(0.8) CDF thresholds over item ranks (same definition as the oracle).
  std::vector<uint64_t> thr(items);
  double total = 0.0;
  for (uint32_t j = 1; j <= items; ++j) total += std::pow(double(j), -0.8);
  double cum = 0.0;
  for (uint32_t j = 1; j <= items; ++j) {
    cum += std::pow(double(j), -0.8);
    thr[j - 1] = j == items ? (1ull << 32) : uint64_t(cum / total * 4294967296.0);
  }
  DevBuf<uint64_t> dthr(items, s);
  GM_CUDA(cudaMemcpyAsync(dthr.get(), thr.data(), items * 8, cudaMemcpyHostToDevice, s));
  DevBuf<uint32_t> deg(users, s);
  launch(users, s, [&](unsigned gr, unsigned bl) { k_bip_degree<<<gr, bl, 0, s>>>(users, c_num, cap, deg.get()); });
  DevBuf<uint64_t> off(uint64_t(users) + 1, s);
  exclusive_scan_to_ptr(deg.get(), off.get(), users, s);
  uint64_t total_raw = 0;
  GM_CUDA(cudaMemcpyAsync(&total_raw, off.get() + users, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  if (total_raw >= 0xFFFFFFFFull) fail(GM_EUSAGE, "bipartite: more than 2^32-2 raw ratings");
  DevBuf<uint32_t> s32(total_raw, s), d32(total_raw, s);
  launch(total_raw, s, [&](unsigned gr, unsigned bl) {
    k_bip_draw<<<gr, bl, 0, s>>>(off.get(), users, items, dthr.get(), uint32_t(seed),
                                 uint32_t(seed >> 32), s32.get(), d32.get());
  });
  DevBuf<uint8_t> none;
  build(*g, s32, d32, int64_t(total_raw), none);
  g->value_type = GM_VAL_U8;
  g->in.val.alloc(g->in.nnz, s);
  const uint64_t seed_r = mix64(seed ^ 0x0DA7A5EEDull);
  launch(g->in.nnz, s, [&](unsigned gr, unsigned bl) {
    k_entry_weights<<<gr, bl, 0, s>>>(g->in.ptr.get(), g->in.idx.get(), g->n, int64_t(g->in.nnz),
                                      g->relabeled ? g->iperm.get() : nullptr, seed_r, 1,
                                      g->in.val.get());
  });
  GM_CUDA(cudaStreamSynchronize(s));
  ensure_forward(*g);
  return g.release();
}

void graph_destroy(Graph* g) {
  if (!g) return;
  cudaStream_t s = g->stream;
  cudaStreamSynchronize(s);
  delete g;  // buffers free stream-ordered on s
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}

// Transpose CSR(G^T) into CSR(G) (rows = sources, entries = destinations
// ascending), carrying values.  Graph::ensure_forward, dcsc.hpp:201-215.
void ensure_forward(Graph& g) {
  if (g.out_built) return;
  cudaStream_t s = g.stream;
  const uint64_t n = g.n;
  const int64_t m = int64_t(g.in.nnz);
  DevBuf<uint64_t> keys(m, s);
  DevBuf<uint32_t> pay(m, s);
  launch(m, s, [&](unsigned gr, unsigned b) {
    k_entry_keys_transposed<<<gr, b, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), n, m, g.nb, keys.get(),
                                             pay.get());
  });
  sort_pairs(keys, pay, m, int(2 * g.nb), s);
  g.out.n = n;
  g.out.nnz = uint64_t(m);
  g.out.ptr.alloc(n + 1, s);
  exclusive_scan_to_ptr(g.outdeg.get(), g.out.ptr.get(), n, s);
  g.out.idx.alloc(m, s);
  launch(m, s, [&](unsigned gr, unsigned b) {
    k_low_bits<<<gr, b, 0, s>>>(keys.get(), m, (uint64_t(1) << g.nb) - 1, g.out.idx.get());
  });
  const size_t vs = value_size(g.value_type);
  if (vs && g.in.val) {
    g.out.val.alloc(size_t(m) * vs, s);
    gather_values(g.in.val.get(), pay.get(), m, vs, g.out.val.get(), s);
  }
  g.out_built = true;
  g.out_alias = false;
  GM_CUDA(cudaStreamSynchronize(s));
}

void export_edges(Graph& g, uint32_t* src, uint32_t* dst, void* values) {
  cudaStream_t s = g.stream;
  const int64_t m = int64_t(g.in.nnz);
  if (m == 0) return;
  // caller-id key (src << nb | dst) of every G^T entry, payload = entry index
  DevBuf<uint64_t> keys(m, s);
  DevBuf<uint32_t> pay(m, s);
  launch(m, s, [&](unsigned gr, unsigned b) {
    k_export_keys<<<gr, b, 0, s>>>(g.in.ptr.get(), g.in.idx.get(), g.n, m, g.nb,
                                   g.relabeled ? g.iperm.get() : nullptr, keys.get(), pay.get());
  });
  sort_pairs(keys, pay, m, int(2 * g.nb), s);
  std::vector<uint64_t> hk(m);
  GM_CUDA(cudaMemcpyAsync(hk.data(), keys.get(), m * 8, cudaMemcpyDeviceToHost, s));
  const size_t vs = value_size(g.value_type);
  std::vector<uint8_t> hv;
  if (values && vs && g.in.val) {
    DevBuf<uint8_t> v(size_t(m) * vs, s);
    gather_values(g.in.val.get(), pay.get(), m, vs, v.get(), s);
    GM_CUDA(cudaMemcpyAsync(values, v.get(), size_t(m) * vs, cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
  const uint64_t mask = (uint64_t(1) << g.nb) - 1;
  for (int64_t i = 0; i < m; ++i) {
    src[i] = uint32_t(hk[i] >> g.nb);
    dst[i] = uint32_t(hk[i] & mask);
  }
}

void to_external(Graph& g, const void* int_dev, void* ext_dev, size_t eb) {
  cudaStream_t s = g.stream;
  const uint64_t n = g.n;
  if (n == 0) return;
  if (!g.relabeled) {
    if (int_dev != ext_dev) GM_CUDA(cudaMemcpyAsync(ext_dev, int_dev, n * eb, cudaMemcpyDeviceToDevice, s));
    return;
  }
  switch (eb) {
    case 8: launch(n, s, [&](unsigned gr, unsigned b) { k_gather_ext<<<gr, b, 0, s>>>((const uint64_t*)int_dev, g.perm.get(), n, (uint64_t*)ext_dev); }); break;
    case 4: launch(n, s, [&](unsigned gr, unsigned b) { k_gather_ext<<<gr, b, 0, s>>>((const uint32_t*)int_dev, g.perm.get(), n, (uint32_t*)ext_dev); }); break;
    case 1: launch(n, s, [&](unsigned gr, unsigned b) { k_gather_ext<<<gr, b, 0, s>>>((const uint8_t*)int_dev, g.perm.get(), n, (uint8_t*)ext_dev); }); break;
    default: {
      std::vector<uint32_t> hp(n);
      GM_CUDA(cudaMemcpyAsync(hp.data(), g.perm.get(), n * 4, cudaMemcpyDeviceToHost, s));
      std::vector<uint8_t> hi(n * eb), ho(n * eb);
      GM_CUDA(cudaMemcpyAsync(hi.data(), int_dev, n * eb, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
      for (uint64_t v = 0; v < n; ++v) std::memcpy(&ho[v * eb], &hi[size_t(hp[v]) * eb], eb);
      GM_CUDA(cudaMemcpyAsync(ext_dev, ho.data(), n * eb, cudaMemcpyHostToDevice, s));
      GM_CUDA(cudaStreamSynchronize(s));
    }
  }
}

void to_internal(Graph& g, const void* ext_dev, void* int_dev, size_t eb) {
  cudaStream_t s = g.stream;
  const uint64_t n = g.n;
  if (n == 0) return;
  if (!g.relabeled) {
    if (int_dev != ext_dev) GM_CUDA(cudaMemcpyAsync(int_dev, ext_dev, n * eb, cudaMemcpyDeviceToDevice, s));
    return;
  }
  switch (eb) {
    case 8: launch(n, s, [&](unsigned gr, unsigned b) { k_gather_ext<<<gr, b, 0, s>>>((const uint64_t*)ext_dev, g.iperm.get(), n, (uint64_t*)int_dev); }); break;
    case 4: launch(n, s, [&](unsigned gr, unsigned b) { k_gather_ext<<<gr, b, 0, s>>>((const uint32_t*)ext_dev, g.iperm.get(), n, (uint32_t*)int_dev); }); break;
    case 1: launch(n, s, [&](unsigned gr, unsigned b) { k_gather_ext<<<gr, b, 0, s>>>((const uint8_t*)ext_dev, g.iperm.get(), n, (uint8_t*)int_dev); }); break;
    default: {
      std::vector<uint32_t> hp(n);
      GM_CUDA(cudaMemcpyAsync(hp.data(), g.iperm.get(), n * 4, cudaMemcpyDeviceToHost, s));
      std::vector<uint8_t> hi(n * eb), ho(n * eb);
      GM_CUDA(cudaMemcpyAsync(hi.data(), ext_dev, n * eb, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
      for (uint64_t v = 0; v < n; ++v) std::memcpy(&ho[v * eb], &hi[size_t(hp[v]) * eb], eb);
      GM_CUDA(cudaMemcpyAsync(int_dev, ho.data(), n * eb, cudaMemcpyHostToDevice, s));
      GM_CUDA(cudaStreamSynchronize(s));
    }
  }
}

void degree_vector(Graph& g, int kind, uint64_t* out) {
  cudaStream_t s = g.stream;
  const uint64_t n = g.n;
  if (n == 0) return;
  DevBuf<uint32_t> ext(n, s);
  to_external(g, kind == 0 ? g.indeg.get() : g.outdeg.get(), ext.get(), 4);
  std::vector<uint32_t> h(n);
  GM_CUDA(cudaMemcpyAsync(h.data(), ext.get(), n * 4, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  for (uint64_t v = 0; v < n; ++v) out[v] = h[v];
}

uint64_t pick_source(Graph& g, uint64_t seed) {
  const uint64_t n = g.n;
  if (n == 0) fail(GM_EUSAGE, "pick_source on an empty graph");
  std::vector<uint64_t> deg(n);
  degree_vector(g, 1, deg.data());
  const uint64_t base = mix64(seed ^ 0x50C0FFEEull);
  for (uint64_t i = 0; i < 1024; ++i) {
    const uint64_t cand = mix64(base + i) % n;
    if (deg[cand] > 0) return cand;
  }
  for (uint64_t v = 0; v < n; ++v)
    if (deg[v] > 0) return v;
  return 0;
}

}  // namespace gm
