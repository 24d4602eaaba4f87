// dist.cu -- row-sharded graph ingest and the multi-GPU supersteps.
//
// Ingest (replaces build_dcsc_partitions + balanced_row_boundaries,
// include/semigraph/dcsc.hpp:77-164, and io::preprocess, src/io.cpp:184-222,
// for a graph no single GPU has to hold):
//   1. every shard draws its 1/P of the edge stream (R-MAT tuples are counter
//      based, so shard r generates tuples [r*M/P, (r+1)*M/P) of the same
//      stream a single GPU would);
//   2. a coarse histogram of destination rows, summed over the shards, gives
//      row boundaries balanced by entries (the rule of dcsc.hpp:81-105 at a
//      granularity of 2^kBucketBits rows, so every boundary is 32-aligned);
//   3. each shard sorts its packed (row << nb | col) keys and sends the run of
//      every destination shard to it (all-to-all: peer copies or NCCL);
//   4. the owner sorts what it received, removes duplicates (keep-first is moot
//      for value-less keys) and builds the CSR of its rows -- entries ascending
//      by caller id, the reference's fold order (engine.hpp:59-66);
//   5. directed graphs: out-degrees summed over the shards; the columns of
//      CSR(G^T) are renumbered to "packed" ids (rank among the vertices with
//      out-edges, ascending caller id), so the exchanged message vector holds
//      only vertices that send (SURVEY 8e mitigation 1) and its block per shard
//      is contiguous;  out-rows (CSR(G), for pushes) come from a second
//      all-to-all of the swapped keys.
// Each shard keeps only its rows: device memory ~ 1/P of one GPU's.
#include <algorithm>
#include <string>

#include "dist.cuh"
#include "ingest.cuh"

namespace gm {

struct DBfsState {
  std::vector<DevBuf<int32_t>> level;      // [l] owned rows
  std::vector<DevBuf<uint32_t>> vis, nxt;  // [l] owned words
  std::vector<DevBuf<uint32_t>> queue;     // [l] local frontier rows (push)
  std::vector<DevBuf<uint64_t>> qdeg;      // [l] their degrees -> exclusive offsets
  std::vector<DevBuf<uint32_t>> iso;       // [l] isolated-row bitmap (owned words)
  std::vector<DevBuf<uint32_t>> deg;       // [l] owned rows' degrees (pull)
  std::vector<DevBuf<unsigned long long>> ctr, sum;  // [l] counters / summed
  std::vector<void*> fb[2], claims;        // [l] peer-visible full bitmaps
  std::vector<std::vector<void*>> fb_tab[2], claims_tab;
  Comm* c = nullptr;
  ~DBfsState() {
    if (!c) return;
    for (int b = 0; b < 2; ++b) c->unshare(fb_tab[b]);
    c->unshare(claims_tab);
    for (int l = 0; l < c->L; ++l) {
      c->set(l);
      cudaStreamSynchronize(c->st[size_t(l)]);
      c->peer_free(l, fb[0][size_t(l)]);
      c->peer_free(l, fb[1][size_t(l)]);
      c->peer_free(l, claims[size_t(l)]);
      level[size_t(l)].reset();
      vis[size_t(l)].reset();
      nxt[size_t(l)].reset();
      queue[size_t(l)].reset();
      qdeg[size_t(l)].reset();
      iso[size_t(l)].reset();
      deg[size_t(l)].reset();
      ctr[size_t(l)].reset();
      sum[size_t(l)].reset();
    }
  }
};

void exclusive_scan_u64(uint64_t* data, uint64_t n, cudaStream_t s);  // generic_programs.cu

struct DPrState {
  std::vector<DevBuf<float>> rank, inv;               // [l] owned rows
  std::vector<DevBuf<uint32_t>> rows_short;           // [l] rows with <= kPrShort entries
  std::vector<DevBuf<uint32_t>> rows_long;            // [l] longer rows
  std::vector<DevBuf<uint64_t>> chunk_beg;            // [l] chunk c: entries [beg[c], beg[c+1])
  std::vector<DevBuf<uint32_t>> long_chunk0;          // [l] first chunk of long row i (+1 end)
  std::vector<DevBuf<float>> chunk_sum;               // [l] per-chunk partial sums
  std::vector<uint64_t> n_short, n_long, n_chunks;
  std::vector<DevBuf<unsigned long long>> part, sum;  // [l] 2 parities x 4 words
  DevBuf<unsigned long long> trace;                   // shard 0: summed words per superstep
  std::vector<void*> x[2];                            // [l] peer-visible packed messages
  std::vector<std::vector<void*>> x_tab[2];
  Comm* c = nullptr;
  ~DPrState() {
    if (!c) return;
    for (int b = 0; b < 2; ++b) c->unshare(x_tab[b]);
    for (int l = 0; l < c->L; ++l) {
      c->set(l);
      cudaStreamSynchronize(c->st[size_t(l)]);
      c->peer_free(l, x[0][size_t(l)]);
      c->peer_free(l, x[1][size_t(l)]);
      rank[size_t(l)].reset();
      inv[size_t(l)].reset();
      rows_short[size_t(l)].reset();
      rows_long[size_t(l)].reset();
      chunk_beg[size_t(l)].reset();
      long_chunk0[size_t(l)].reset();
      chunk_sum[size_t(l)].reset();
      part[size_t(l)].reset();
      sum[size_t(l)].reset();
      if (l == 0) trace.reset();
    }
  }
};

namespace {

constexpr unsigned kBlock = 256;
constexpr int kMaxPeers = 64;

template <typename T>
struct PeerTab {
  T* p[kMaxPeers];
};

template <typename F>
void launch(uint64_t work, cudaStream_t s, F&& f, unsigned block = kBlock) {
  if (work == 0) return;
  f(grid_for(work, block), block);
  GM_LAUNCH_CHECK();
}

// ---- ingest kernels -----------------------------------------------------------
// Packed keys row << nb | col of the generated edges; self loops dropped
// (io::preprocess); symmetric graphs add the reverse of every edge.
__global__ void k_edge_keys(const uint32_t* s, const uint32_t* d, uint64_t m, unsigned nb, int sym,
                            uint64_t* keys, unsigned long long* cnt) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = s[e], b = d[e];
    if (a == b) continue;
    const unsigned long long k = atomicAdd(cnt, sym ? 2ull : 1ull);
    keys[k] = (uint64_t(b) << nb) | a;  // row = destination (G^T)
    if (sym) keys[k + 1] = (uint64_t(a) << nb) | b;
  }
}

__global__ void k_row_hist(const uint64_t* keys, uint64_t m, unsigned shift,
                           unsigned long long* hist) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(&hist[keys[e] >> shift], 1ull);
}

// Start of each shard's run in a sorted key array (rows [bounds[r], ...)).
__global__ void k_run_starts(const uint64_t* keys, uint64_t m, unsigned nb, const uint64_t* bounds,
                             int P, uint64_t* starts) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  const uint64_t x = bounds[r] << nb;
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  starts[r] = r == P ? m : lo;
}

// CSR of the rows [lo, lo + rows) from sorted unique keys.
__global__ void k_keys_to_csr(const uint64_t* keys, uint64_t m, unsigned nb, uint64_t lo,
                              uint64_t rows, uint64_t* ptr, uint32_t* idx) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i <= m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i < m ? (keys[i] >> nb) - lo : rows;
    const uint64_t p = i == 0 ? 0 : (keys[i - 1] >> nb) - lo + 1;
    for (uint64_t q = p; q <= r && q <= rows; ++q) ptr[q] = i;  // rows (prev, r] start at i
    if (i < m) idx[i] = uint32_t(keys[i] & mask);
  }
}

__global__ void k_swap_keys(const uint64_t* ptr, const uint32_t* idx, uint64_t lo, uint64_t rows,
                            unsigned nb, uint64_t* keys) {
  // one warp per row: (col << nb | row) for every entry
  const uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = w; r < rows; r += nw)
    for (uint64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32)
      keys[e] = (uint64_t(idx[e]) << nb) | (lo + r);
}

__global__ void k_src_degree(const uint32_t* idx, uint64_t nnz, uint32_t* deg) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(&deg[idx[e]], 1u);
}

__global__ void k_row_col_keys(const uint64_t* ptr, const uint32_t* idx, uint64_t rows, unsigned cb,
                               uint64_t* keys) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = wp; r < rows; r += nw)
    for (uint64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) keys[e] = (r << cb) | idx[e];
}

__global__ void k_rebase_ptr2(const uint64_t* ptr, uint64_t n, uint64_t base, uint64_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = ptr[i] - base;
}

__global__ void k_low_cols(const uint64_t* keys, uint64_t m, unsigned cb, uint32_t* idx) {
  const uint64_t mask = (uint64_t(1) << cb) - 1;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x)
    idx[e] = uint32_t(keys[e] & mask);
}

// Each row's entries ascending (a value-less CSR), in chunks of ~2^30 entries.
void sort_row_entries(Csr& a, unsigned cb, cudaStream_t s) {
  const uint64_t rows = a.n;
  if (a.nnz < 2) return;
  const uint64_t per = std::max<uint64_t>(1, rows * (uint64_t(1) << 30) / a.nnz);
  for (uint64_t r0 = 0; r0 < rows; r0 += per) {
    const uint64_t r1 = std::min(rows, r0 + per);
    uint64_t e[2];
    GM_CUDA(cudaMemcpyAsync(&e[0], a.ptr.get() + r0, 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaMemcpyAsync(&e[1], a.ptr.get() + r1, 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const uint64_t m = e[1] - e[0];
    unsigned rb = 1;
    while ((uint64_t(1) << rb) < (r1 - r0) + 1) ++rb;
    if (m < 2 || rb + cb > 64) continue;
    DevBuf<uint64_t> lptr(r1 - r0 + 1, s), keys(m, s);
    launch(r1 - r0 + 1, s, [&](unsigned gr, unsigned bl) {
      k_rebase_ptr2<<<gr, bl, 0, s>>>(a.ptr.get() + r0, r1 - r0 + 1, e[0], lptr.get());
    });
    launch((r1 - r0) * 32, s, [&](unsigned gr, unsigned bl) {
      k_row_col_keys<<<gr, bl, 0, s>>>(lptr.get(), a.idx.get() + e[0], r1 - r0, cb, keys.get());
    });
    sort_keys_u64(keys, int64_t(m), int(rb + cb), s);
    launch(m, s, [&](unsigned gr, unsigned bl) {
      k_low_cols<<<gr, bl, 0, s>>>(keys.get(), m, cb, a.idx.get() + e[0]);
    });
    GM_CUDA(cudaStreamSynchronize(s));
  }
}

__global__ void k_pack_keys(const uint32_t* od, uint64_t n, uint64_t* keys) {
  for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n;
       u += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t d = od[u];
    const uint64_t cls = d ? uint64_t(1 + 31 - __clz(int(d))) : 0;  // 0 = no out-edges: last
    keys[u] = ((63 - cls) << 32) | u;
  }
}

__global__ void k_pack_map(const uint64_t* keys, uint64_t n, uint64_t* pmap) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    pmap[keys[i] & 0xFFFFFFFFull] = i;
}

__global__ void k_count_senders(const uint32_t* od, uint64_t n, unsigned long long* cnt) {
  unsigned long long c = 0;
  for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n;
       u += uint64_t(gridDim.x) * blockDim.x)
    c += od[u] > 0;
  warp_add_u64(cnt, c);
}

__global__ void k_block_pids(const uint32_t* od, const uint64_t* pmap, uint64_t lo, uint64_t rows,
                             uint32_t* pid) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x)
    pid[r] = od[lo + r] ? uint32_t(pmap[lo + r]) : ~0u;
}

__global__ void k_remap_cols(uint32_t* idx, uint64_t nnz, const uint64_t* pmap) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += uint64_t(gridDim.x) * blockDim.x)
    idx[e] = uint32_t(pmap[idx[e]]);
}

__global__ void k_row_weights(const uint64_t* ptr, const uint32_t* idx, uint64_t lo, uint64_t rows,
                              uint64_t seed_w, int row_is_dst, uint8_t* w) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = wp; r < rows; r += nw)
    for (uint64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      const uint32_t row = uint32_t(lo + r), col = idx[e];
      w[e] = row_is_dst ? edge_weight(seed_w, col, row) : edge_weight(seed_w, row, col);
    }
}

__global__ void k_first_dup(const uint64_t* keys, uint64_t m, unsigned long long* first) {
  for (uint64_t i = 1 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (keys[i] == keys[i - 1]) atomicMin(first, (unsigned long long)i);
}

unsigned bucket_bits(uint64_t n, int P) {
  // >= 32 rows per bucket (aligned boundaries), ~>= 64 buckets per shard
  unsigned b = 5;
  while (b < 20 && (n >> (b + 1)) >= uint64_t(P) * 64) ++b;
  return b;
}

uint64_t dread_u64(const unsigned long long* p, cudaStream_t s) {
  unsigned long long h = 0;
  GM_CUDA(cudaMemcpyAsync(&h, p, 8, cudaMemcpyDeviceToHost, s));
  GM_CUDA(cudaStreamSynchronize(s));
  return h;
}

// keys[l] (packed row << nb | col, any order) -> the CSR of each shard's rows.
// Sets g.bounds from the key histogram when empty.  check_dups: the first
// duplicate is an InputError (build_graph without preprocess, dcsc.hpp:148-150).
void route_and_build(DGraph& g, std::vector<DevBuf<uint64_t>>& keys, std::vector<uint64_t>& m,
                     unsigned nb, bool forward, bool check_dups) {
  Comm& c = *g.comm;
  const int P = c.P, L = c.L;
  if (g.bounds.empty()) {
    const unsigned bb = bucket_bits(g.n, P);
    const uint64_t nbk = (g.n + (uint64_t(1) << bb) - 1) >> bb;
    std::vector<DevBuf<unsigned long long>> h(static_cast<size_t>(L)), hs(static_cast<size_t>(L));
    std::vector<const uint64_t*> hin;
    std::vector<uint64_t*> hout;
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      h[size_t(l)].alloc(nbk, s);
      hs[size_t(l)].alloc(nbk, s);
      h[size_t(l)].zero(s);
      launch(m[size_t(l)], s, [&](unsigned gr, unsigned bl) {
        k_row_hist<<<gr, bl, 0, s>>>(keys[size_t(l)].get(), m[size_t(l)], nb + bb, h[size_t(l)].get());
      });
      hin.push_back(reinterpret_cast<const uint64_t*>(h[size_t(l)].get()));
      hout.push_back(reinterpret_cast<uint64_t*>(hs[size_t(l)].get()));
    }
    c.allreduce_u64(hin, hout, nbk);
    std::vector<uint64_t> hh(nbk);
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(hh.data(), hout[0], nbk * 8, cudaMemcpyDeviceToHost, c.st[0]));
    GM_CUDA(cudaStreamSynchronize(c.st[0]));
    // balanced_row_boundaries (dcsc.hpp:81-105) over buckets
    std::vector<uint64_t> cum(nbk + 1, 0);
    for (uint64_t i = 0; i < nbk; ++i) cum[i + 1] = cum[i] + hh[i];
    const uint64_t total = cum[nbk];
    g.bounds.assign(size_t(P) + 1, 0);
    g.bounds[size_t(P)] = g.n;
    for (int p = 1; p < P; ++p) {
      uint64_t lo = g.bounds[size_t(p) - 1] >> bb, hi = nbk;
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (cum[mid] * uint64_t(P) >= uint64_t(p) * total)
          hi = mid;
        else
          lo = mid + 1;
      }
      g.bounds[size_t(p)] = std::min(g.n, lo << bb);
    }
    for (int l = 0; l < L; ++l) {
      g.sh[size_t(l)].lo = g.bounds[size_t(c.global(l))];
      g.sh[size_t(l)].hi = g.bounds[size_t(c.global(l)) + 1];
    }
  }
  std::vector<DevBuf<uint64_t>> recv(static_cast<size_t>(L));
  std::vector<uint64_t> mr(static_cast<size_t>(L));
  if (P == 1) {  // one shard: its keys are its rows (no sort + copy: scale 28 fits)
    recv[0].swap(keys[0]);
    mr[0] = m[0];
  } else {
  // sort locally, find every destination's run, exchange the runs
  std::vector<std::vector<uint64_t>> send_offs(static_cast<size_t>(L)), send_counts(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    sort_keys_u64(keys[size_t(l)], int64_t(m[size_t(l)]), int(2 * nb), s);
    DevBuf<uint64_t> db(size_t(P) + 1, s), st(size_t(P) + 1, s);
    GM_CUDA(cudaMemcpyAsync(db.get(), g.bounds.data(), (size_t(P) + 1) * 8, cudaMemcpyHostToDevice, s));
    k_run_starts<<<1, 128, 0, s>>>(keys[size_t(l)].get(), m[size_t(l)], nb, db.get(), P, st.get());
    GM_LAUNCH_CHECK();
    std::vector<uint64_t> hst(size_t(P) + 1);
    GM_CUDA(cudaMemcpyAsync(hst.data(), st.get(), (size_t(P) + 1) * 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < P; ++r) {
      send_offs[size_t(l)].push_back(hst[size_t(r)] * 8);
      send_counts[size_t(l)].push_back((hst[size_t(r) + 1] - hst[size_t(r)]) * 8);
    }
  }
  // (local mode: exchange_counts is a transpose; nccl: a count all-gather)
  const auto recv_counts = c.exchange_counts(send_counts);
  std::vector<std::vector<uint64_t>> recv_offs(static_cast<size_t>(L));
  std::vector<const uint8_t*> sp;
  std::vector<uint8_t*> rp;
  for (int l = 0; l < L; ++l) {
    uint64_t off = 0;
    for (int q = 0; q < P; ++q) {
      recv_offs[size_t(l)].push_back(off);
      off += recv_counts[size_t(l)][size_t(q)];
    }
    mr[size_t(l)] = off / 8;
    c.set(l);
    recv[size_t(l)].alloc(mr[size_t(l)] + 1, c.st[size_t(l)]);
    sp.push_back(reinterpret_cast<const uint8_t*>(keys[size_t(l)].get()));
    rp.push_back(reinterpret_cast<uint8_t*>(recv[size_t(l)].get()));
  }
  c.alltoallv(sp, send_offs, send_counts, rp, recv_offs);
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    GM_CUDA(cudaStreamSynchronize(s));
    keys[size_t(l)].reset();
  }
  }  // P > 1
  // owners: sort, check / remove duplicates, build the rows
  std::vector<uint64_t> bad(size_t(L), 0);
  std::vector<std::string> msg(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    DevBuf<uint64_t>& k = recv[size_t(l)];
    int64_t cnt = int64_t(mr[size_t(l)]);
    sort_keys_u64(k, cnt, int(2 * nb), s);
    if (check_dups) {
      DevBuf<unsigned long long> fd(1, s);
      GM_CUDA(cudaMemsetAsync(fd.get(), 0xFF, 8, s));
      launch(uint64_t(cnt), s, [&](unsigned gr, unsigned bl) {
        k_first_dup<<<gr, bl, 0, s>>>(k.get(), uint64_t(cnt), fd.get());
      });
      const uint64_t i = dread_u64(fd.get(), s);
      if (i != ~0ull) {
        uint64_t key = 0;
        GM_CUDA(cudaMemcpyAsync(&key, k.get() + i, 8, cudaMemcpyDeviceToHost, s));
        GM_CUDA(cudaStreamSynchronize(s));
        const uint64_t row = key >> nb, col = key & ((uint64_t(1) << nb) - 1);
        const uint64_t src = forward ? row : col, dst = forward ? col : row;
        bad[size_t(l)] = 1;
        msg[size_t(l)] = "build_graph: duplicate edge " + std::to_string(src + 1) + " -> " +
                         std::to_string(dst + 1) + " (1-based); deduplicate before building";
      }
    } else {
      cnt = unique_keys_u64(k, cnt, s);
    }
    Csr& a = forward ? sh.out : sh.in;
    const uint64_t rows = sh.hi - sh.lo;
    a.n = rows;
    a.nnz = uint64_t(cnt);
    a.ptr.alloc(rows + 1, s);
    a.idx.alloc(uint64_t(cnt) + 1, s);
    launch(uint64_t(cnt) + 1, s, [&](unsigned gr, unsigned bl) {
      k_keys_to_csr<<<gr, bl, 0, s>>>(k.get(), uint64_t(cnt), nb, sh.lo, rows, a.ptr.get(), a.idx.get());
    });
    GM_CUDA(cudaStreamSynchronize(s));
    k.reset();
  }
  uint64_t nbad = 0;
  for (uint64_t b : bad) nbad += b;
  if (c.sum_host({nbad})) {
    for (int l = 0; l < L; ++l)
      if (bad[size_t(l)]) fail(GM_EINPUT, msg[size_t(l)]);
    fail(GM_EINPUT, "build_graph: duplicate edge on another shard; deduplicate before building");
  }
}

// CSR(G) rows of the owned vertices from everybody's CSR(G^T) rows.
void build_forward(DGraph& g, unsigned nb) {
  Comm& c = *g.comm;
  std::vector<DevBuf<uint64_t>> keys(static_cast<size_t>(c.L));
  std::vector<uint64_t> m(static_cast<size_t>(c.L));
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    m[size_t(l)] = sh.in.nnz;
    keys[size_t(l)].alloc(sh.in.nnz + 1, s);
    launch(sh.in.n * 32, s, [&](unsigned gr, unsigned bl) {
      k_swap_keys<<<gr, bl, 0, s>>>(sh.in.ptr.get(), sh.in.idx.get(), sh.lo, sh.in.n, nb,
                                    keys[size_t(l)].get());
    });
  }
  route_and_build(g, keys, m, nb, /*forward=*/true, /*check_dups=*/false);
}

// Directed graphs: global out-degrees (summed over the shards), the owned
// rows' out-degrees, and the packed renumbering of CSR(G^T)'s columns.
void finish_directed(DGraph& g) {
  Comm& c = *g.comm;
  const uint64_t n = g.n;
  std::vector<DevBuf<uint32_t>> deg(static_cast<size_t>(c.L)), degs(static_cast<size_t>(c.L));
  std::vector<const uint64_t*> din;
  std::vector<uint64_t*> dout;
  // u32 counts travel as u64 pairs: the sum of two shards' u32 never carries
  // across the 32-bit halves because a vertex's out-degree is < 2^32
  const uint64_t words = (n + 1) / 2;
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    deg[size_t(l)].alloc(2 * words, s);
    degs[size_t(l)].alloc(2 * words, s);
    deg[size_t(l)].zero(s);
    launch(sh.in.nnz, s, [&](unsigned gr, unsigned bl) {
      k_src_degree<<<gr, bl, 0, s>>>(sh.in.idx.get(), sh.in.nnz, deg[size_t(l)].get());
    });
    din.push_back(reinterpret_cast<const uint64_t*>(deg[size_t(l)].get()));
    dout.push_back(reinterpret_cast<uint64_t*>(degs[size_t(l)].get()));
  }
  c.allreduce_u64(din, dout, words);
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    deg[size_t(l)].reset();
    const uint32_t* od = degs[size_t(l)].get();
    sh.outdeg.alloc(sh.hi - sh.lo + 1, s);
    if (sh.hi > sh.lo)
      GM_CUDA(cudaMemcpyAsync(sh.outdeg.get(), od + sh.lo, (sh.hi - sh.lo) * 4,
                              cudaMemcpyDeviceToDevice, s));
    // packed id of u = its rank among the vertices with out-edges, hub-first:
    // by out-degree class (floor(log2 d), descending), then caller id -- a
    // P-independent order (every shard computes the same map from the summed
    // degrees) that puts the hubs' messages together at the front of x
    DevBuf<uint64_t> pmap(n + 1, s);
    {
      DevBuf<uint64_t> keys(n, s);
      launch(n, s, [&](unsigned gr, unsigned bl) { k_pack_keys<<<gr, bl, 0, s>>>(od, n, keys.get()); });
      sort_keys_u64(keys, int64_t(n), 38, s);
      launch(n, s, [&](unsigned gr, unsigned bl) { k_pack_map<<<gr, bl, 0, s>>>(keys.get(), n, pmap.get()); });
      DevBuf<unsigned long long> cnt(1, s);
      cnt.zero(s);
      launch(n, s, [&](unsigned gr, unsigned bl) { k_count_senders<<<gr, bl, 0, s>>>(od, n, cnt.get()); });
      GM_CUDA(cudaMemcpyAsync(pmap.get() + n, cnt.get(), 8, cudaMemcpyDeviceToDevice, s));
    }
    launch(sh.in.nnz, s, [&](unsigned gr, unsigned bl) {
      k_remap_cols<<<gr, bl, 0, s>>>(sh.in.idx.get(), sh.in.nnz, pmap.get());
    });
    // rows of a value-less graph re-sorted by packed id: hub-first gathers
    // (and a P-independent fold order, as the ids are)
    if (!sh.in.val) sort_row_entries(sh.in, bits_for(n + 1), s);
    sh.pid.alloc(sh.hi - sh.lo + 1, s);
    launch(sh.hi - sh.lo, s, [&](unsigned gr, unsigned bl) {
      k_block_pids<<<gr, bl, 0, s>>>(od, pmap.get(), sh.lo, sh.hi - sh.lo, sh.pid.get());
    });
    uint64_t nz = 0;
    GM_CUDA(cudaMemcpyAsync(&nz, pmap.get() + n, 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    g.nonzero_outdeg = nz;
    degs[size_t(l)].reset();
  }
}

}  // namespace

// ---- DGraph -----------------------------------------------------------------
DGraph::~DGraph() {
  bfs.reset();
  pr.reset();
  sssp.reset();
  cf.reset();
  if (!comm) return;
  struct Release {  // the graph's reference on its communicator, dropped last
    Comm* c;
    ~Release() { comm_release(c); }
  } rel{comm};
  for (int l = 0; l < comm->L && size_t(l) < sh.size(); ++l) {
    comm->set(l);
    cudaStreamSynchronize(comm->st[size_t(l)]);
    DShard& s = sh[size_t(l)];
    s.in.ptr.reset();
    s.in.idx.reset();
    s.in.val.reset();
    s.out.ptr.reset();
    s.out.idx.reset();
    s.out.val.reset();
    s.outdeg.reset();
    s.pid.reset();
    cudaStreamSynchronize(comm->st[size_t(l)]);
  }
}

uint64_t DGraph::owner(uint64_t v) const {
  return uint64_t(std::upper_bound(bounds.begin(), bounds.end(), v) - bounds.begin()) - 1;
}

uint64_t DGraph::device_bytes(int l) const {
  const DShard& s = sh[size_t(l)];
  uint64_t b = s.in.ptr.bytes() + s.in.idx.bytes() + s.in.val.bytes() + s.outdeg.bytes() +
               s.pid.bytes();
  if (!s.out_alias) b += s.out.ptr.bytes() + s.out.idx.bytes() + s.out.val.bytes();
  return b;
}

namespace {

DGraph* new_dgraph(Comm* c, uint64_t n, uint32_t flags) {
  std::unique_ptr<DGraph> g(new DGraph());
  comm_retain(c);
  g->comm = c;
  g->n = n;
  g->flags = flags;
  g->symmetric = (flags & GM_SYMMETRIZE) != 0;
  g->sh.resize(static_cast<size_t>(c->L));
  for (int l = 0; l < c->L; ++l) g->sh[size_t(l)].l = l;
  return g.release();
}

// Symmetric graphs: every row's neighbours ordered hub-first -- by degree
// class (floor(log2(degree)), descending), then caller id -- so a pull finds
// a frontier neighbour in its first probes (the role the degree relabel plays
// on one GPU).  The classes are global (an OR of every shard's slice of a
// byte per vertex), so the order, and every result, is the same for any P.
__global__ void k_deg_class(const uint64_t* ptr, uint64_t lo, uint64_t rows, uint8_t* cls) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t d = ptr[r + 1] - ptr[r];
    cls[lo + r] = d ? uint8_t(1 + 63 - __clzll((long long)d)) : 0;  // 0: isolated
  }
}

__global__ void k_hub_keys(const uint64_t* ptr, const uint32_t* idx, uint64_t rows, unsigned nb,
                           const uint8_t* cls, uint64_t* keys) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = wp; r < rows; r += nw)
    for (uint64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      const uint32_t u = idx[e];
      keys[e] = (r << (nb + 6)) | (uint64_t(63 - cls[u]) << nb) | u;
    }
}

__global__ void k_rebase_ptr(const uint64_t* ptr, uint64_t n, uint64_t base, uint64_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = ptr[i] - base;
}

__global__ void k_low_ids(const uint64_t* keys, uint64_t m, unsigned nb, uint32_t* idx) {
  const uint64_t mask = (uint64_t(1) << nb) - 1;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x)
    idx[e] = uint32_t(keys[e] & mask);
}

void hub_first_rows(DGraph& g, unsigned nb) {
  Comm& c = *g.comm;
  const uint64_t words = (g.n + 7) / 8;
  std::vector<DevBuf<uint64_t>> cl(static_cast<size_t>(c.L)), cls(static_cast<size_t>(c.L));
  std::vector<const uint64_t*> in;
  std::vector<uint64_t*> out;
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    cl[size_t(l)].alloc(words + 1, s);
    cls[size_t(l)].alloc(words + 1, s);
    cl[size_t(l)].zero(s);
    launch(sh.hi - sh.lo, s, [&](unsigned gr, unsigned bl) {
      k_deg_class<<<gr, bl, 0, s>>>(sh.in.ptr.get(), sh.lo, sh.hi - sh.lo,
                                    reinterpret_cast<uint8_t*>(cl[size_t(l)].get()));
    });
    in.push_back(cl[size_t(l)].get());
    out.push_back(cls[size_t(l)].get());
  }
  c.allreduce_u64(in, out, words);  // one writer per byte: the sum is an OR
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    cl[size_t(l)].reset();
    const uint64_t rows = sh.hi - sh.lo;
    if (!sh.in.nnz) continue;
    // rows in chunks of ~2^30 entries: the sort's key buffers stay ~16 GB
    // (one GPU holding a whole scale-28 graph has ~140 GB free, not 2 x 68)
    const uint64_t per = std::max<uint64_t>(1, rows * (uint64_t(1) << 30) / sh.in.nnz);
    for (uint64_t r0 = 0; r0 < rows; r0 += per) {
      const uint64_t r1 = std::min(rows, r0 + per);
      uint64_t e[2];
      GM_CUDA(cudaMemcpyAsync(&e[0], sh.in.ptr.get() + r0, 8, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaMemcpyAsync(&e[1], sh.in.ptr.get() + r1, 8, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
      const uint64_t m = e[1] - e[0];
      if (m < 2) continue;
      unsigned rb = 1;
      while ((uint64_t(1) << rb) < (r1 - r0) + 1) ++rb;
      if (rb + nb + 6 > 64) continue;  // keys too wide: keep caller-id order for these rows
      DevBuf<uint64_t> keys(m, s);
      // k_hub_keys numbers rows from r0 (pointer offset) and entries from e[0]
      DevBuf<uint64_t> lptr(r1 - r0 + 1, s);
      launch(r1 - r0 + 1, s, [&](unsigned gr, unsigned bl) {
        k_rebase_ptr<<<gr, bl, 0, s>>>(sh.in.ptr.get() + r0, r1 - r0 + 1, e[0], lptr.get());
      });
      launch((r1 - r0) * 32, s, [&](unsigned gr, unsigned bl) {
        k_hub_keys<<<gr, bl, 0, s>>>(lptr.get(), sh.in.idx.get() + e[0], r1 - r0, nb,
                                     reinterpret_cast<const uint8_t*>(cls[size_t(l)].get()),
                                     keys.get());
      });
      sort_keys_u64(keys, int64_t(m), int(rb + nb + 6), s);
      launch(m, s, [&](unsigned gr, unsigned bl) {
        k_low_ids<<<gr, bl, 0, s>>>(keys.get(), m, nb, sh.in.idx.get() + e[0]);
      });
      GM_CUDA(cudaStreamSynchronize(s));
    }
    cls[size_t(l)].reset();
  }
}

void finish_build(DGraph& g, unsigned nb, int weights, uint64_t seed) {
  Comm& c = *g.comm;
  if (g.symmetric) {
    for (auto& s : g.sh) s.out_alias = true;
    hub_first_rows(g, nb);
  } else {
    if ((g.flags & GM_NEED_FORWARD) || weights == GM_VAL_U8) build_forward(g, nb);
    if (weights == GM_VAL_U8) {
      g.value_type = GM_VAL_U8;
      const uint64_t seed_w = mix64(seed ^ 0x57E16475ull);
      for (int l = 0; l < c.L; ++l) {
        c.set(l);
        cudaStream_t s = c.st[size_t(l)];
        DShard& sh = g.sh[size_t(l)];
        for (int f = 0; f < 2; ++f) {
          Csr& a = f ? sh.out : sh.in;
          a.val.alloc(a.nnz + 1, s);
          launch(a.n * 32, s, [&](unsigned gr, unsigned bl) {
            k_row_weights<<<gr, bl, 0, s>>>(a.ptr.get(), a.idx.get(), sh.lo, a.n, seed_w, f == 0,
                                            a.val.get());
          });
        }
      }
    }
    finish_directed(g);  // after the forward build: it renumbers CSR(G^T) columns
  }
  uint64_t mm = 0;
  std::vector<uint64_t> nnz;
  for (auto& s : g.sh) nnz.push_back(s.in.nnz);
  mm = c.sum_host(nnz);
  g.m = mm;
  if (g.symmetric) {
    g.nonzero_outdeg = 0;  // not needed by the symmetric programs
  }
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    GM_CUDA(cudaStreamSynchronize(c.st[size_t(l)]));
  }
}

}  // namespace

DGraph* dgraph_generate_rmat(Comm* c, uint32_t scale, uint32_t ef, double a, double b, double cc,
                             uint64_t seed, uint32_t flags, int weights) {
  if (scale == 0 || scale > 31) fail(GM_EUSAGE, "rmat: scale must be in [1, 31]");
  if (!(a >= 0.0 && b >= 0.0 && cc >= 0.0 && a + b + cc <= 1.0))
    fail(GM_EINPUT, "rmat: quadrant probabilities must be non-negative and sum to at most 1");
  if (weights != GM_VAL_NONE && weights != GM_VAL_U8) fail(GM_EUSAGE, "rmat: weights must be none or u8");
  if ((flags & GM_SYMMETRIZE) && weights != GM_VAL_NONE)
    fail(GM_EUSAGE, "rmat: weighted symmetric sharded graphs are not supported");
  const uint64_t n = uint64_t(1) << scale;
  std::unique_ptr<DGraph> g(new_dgraph(c, n, flags | GM_PREPROCESS));
  const uint64_t count = uint64_t(ef) << scale;
  const unsigned nb = scale;
  const int sym = g->symmetric ? 1 : 0;
  std::vector<DevBuf<uint64_t>> keys(static_cast<size_t>(c->L));
  std::vector<uint64_t> m(static_cast<size_t>(c->L));
  for (int l = 0; l < c->L; ++l) {
    c->set(l);
    cudaStream_t s = c->st[size_t(l)];
    const int r = c->global(l);
    const uint64_t t0 = count * uint64_t(r) / uint64_t(c->P);
    const uint64_t t1 = count * uint64_t(r + 1) / uint64_t(c->P);
    DevBuf<uint32_t> s32(t1 - t0 + 1, s), d32(t1 - t0 + 1, s);
    rmat_range(scale, a, b, cc, seed, 1, t0, t1 - t0, s32.get(), d32.get(), s);
    keys[size_t(l)].alloc((t1 - t0) * (sym ? 2 : 1) + 1, s);
    DevBuf<unsigned long long> cnt(1, s);
    cnt.zero(s);
    launch(t1 - t0, s, [&](unsigned gr, unsigned bl) {
      k_edge_keys<<<gr, bl, 0, s>>>(s32.get(), d32.get(), t1 - t0, nb, sym, keys[size_t(l)].get(),
                                    cnt.get());
    });
    m[size_t(l)] = dread_u64(cnt.get(), s);
  }
  route_and_build(*g, keys, m, nb, /*forward=*/false, /*check_dups=*/false);
  finish_build(*g, nb, weights, seed);
  return g.release();
}

DGraph* dgraph_create(Comm* c, const gm_edge_list& e, uint64_t n, uint32_t flags, int storage) {
  if (storage != GM_VAL_NONE) fail(GM_EUSAGE, "dgraph: edge values are not supported yet");
  if (flags & (GM_DAGIFY | GM_BIPARTITE_CHECK))
    fail(GM_EUSAGE, "dgraph: DAGIFY / BIPARTITE_CHECK are single-GPU ingest modes");
  if (n == 0 || n > (uint64_t(1) << 32)) fail(GM_EUSAGE, "dgraph: 1 <= n <= 2^32");
  std::unique_ptr<DGraph> g(new_dgraph(c, n, flags | ((flags & GM_SYMMETRIZE) ? GM_PREPROCESS : 0)));
  const bool pre = (g->flags & GM_PREPROCESS) != 0;
  const unsigned nb = bits_for(n);
  const int sym = g->symmetric ? 1 : 0;
  std::vector<DevBuf<uint64_t>> keys(static_cast<size_t>(c->L));
  std::vector<uint64_t> m(static_cast<size_t>(c->L));
  std::vector<uint64_t> bad(size_t(c->L), 0);
  std::string msg;
  for (int l = 0; l < c->L; ++l) {
    c->set(l);
    cudaStream_t s = c->st[size_t(l)];
    const uint64_t cnt = l == 0 ? uint64_t(e.count) : 0;
    DevBuf<uint32_t> s32(cnt + 1, s), d32(cnt + 1, s);
    if (cnt) {
      if (e.id_type != GM_ID_U32) fail(GM_EUSAGE, "dgraph: ids must be u32");
      const cudaMemcpyKind kd = e.on_device ? cudaMemcpyDefault : cudaMemcpyHostToDevice;
      GM_CUDA(cudaMemcpyAsync(s32.get(), e.src, cnt * 4, kd, s));
      GM_CUDA(cudaMemcpyAsync(d32.get(), e.dst, cnt * 4, kd, s));
    }
    // range check before packing (the reference message, dcsc.hpp:252-256)
    std::vector<uint32_t> hs(cnt), hd(cnt);
    if (cnt) {
      GM_CUDA(cudaMemcpyAsync(hs.data(), s32.get(), cnt * 4, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaMemcpyAsync(hd.data(), d32.get(), cnt * 4, cudaMemcpyDeviceToHost, s));
      GM_CUDA(cudaStreamSynchronize(s));
    }
    for (uint64_t i = 0; i < cnt && !bad[size_t(l)]; ++i)
      if (hs[i] >= n || hd[i] >= n) {
        bad[size_t(l)] = 1;
        msg = "build_graph: edge " + std::to_string(uint64_t(hs[i]) + 1) + " -> " +
              std::to_string(uint64_t(hd[i]) + 1) + " (1-based) exceeds vertex count " +
              std::to_string(n);
      }
    if (bad[size_t(l)]) continue;
    keys[size_t(l)].alloc(cnt * (sym ? 2 : 1) + 1, s);
    DevBuf<unsigned long long> k(1, s);
    k.zero(s);
    if (pre) {
      launch(cnt, s, [&](unsigned gr, unsigned bl) {
        k_edge_keys<<<gr, bl, 0, s>>>(s32.get(), d32.get(), cnt, nb, sym, keys[size_t(l)].get(), k.get());
      });
      m[size_t(l)] = dread_u64(k.get(), s);
    } else {
      // build_graph keeps self loops; rows = destinations
      std::vector<uint64_t> hk(cnt);
      for (uint64_t i = 0; i < cnt; ++i) hk[i] = (uint64_t(hd[i]) << nb) | hs[i];
      if (cnt)
        GM_CUDA(cudaMemcpyAsync(keys[size_t(l)].get(), hk.data(), cnt * 8, cudaMemcpyHostToDevice, s));
      GM_CUDA(cudaStreamSynchronize(s));
      m[size_t(l)] = cnt;
    }
  }
  // every rank learns whether any rank's input was bad before a collective
  if (c->sum_host(bad)) fail(GM_EINPUT, msg.empty() ? "build_graph: an edge on another rank exceeds "
                                                      "the vertex count" : msg);
  route_and_build(*g, keys, m, nb, false, /*check_dups=*/!pre);
  finish_build(*g, nb, GM_VAL_NONE, 0);
  return g.release();
}

// ============================================================================
// BFS over the row shards (algo::bfs, traversal.hpp:119-123; levels are the
// superstep that first reaches a vertex, engine.hpp:193-213).
//
// Per superstep, on every shard:
//   push (frontier small): expand the shard's own frontier rows (a local
//        queue); a neighbour in the shard's rows is claimed in its next-block
//        bitmap, any other one in the shard's full-N claims bitmap; after a
//        barrier each owner ORs its words of every shard's claims bitmap into
//        its next block (peer loads) and clears them (peer stores);
//   pull (frontier large): every unvisited owned row scans its neighbours for
//        a member of the replicated frontier bitmap (early exit).
// finish: new = next & ~visited -> level, visited, the next local queue and
// the (found, found edges) counters, which one u64 all-reduce sums; the host
// reads the sums (the only host synchronisation per superstep) and applies
// the single-GPU rule: pull once frontier edges > m/20, push again once the
// frontier < n/24.  Before a pull superstep the owners store their new-frontier
// words into every shard's replicated frontier bitmap (peer stores over
// NVLink); pushes need no replicated frontier at all.
// ============================================================================
namespace {

constexpr int kPush = 1, kPull = 0;

// the shard's isolated rows (no neighbours: never reached, never a parent)
__global__ void k_db_isolated(const uint64_t* ptr, uint64_t rows, uint32_t* iso) {
  const uint64_t words = (rows + 31) / 32;
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); w0 < words;
       w0 += uint64_t(gridDim.x) * blockDim.x) {
    for (unsigned j = 0; j < 32 && w0 + j < words; ++j) {
      const uint64_t r = (w0 + j) * 32 + lane_id();
      const unsigned b = __ballot_sync(0xffffffffu, r < rows && ptr[r + 1] == ptr[r]);
      if (lane_id() == 0) iso[w0 + j] = b;
    }
  }
}

__global__ void k_db_init(int32_t* level, uint64_t rows, uint32_t* vis, uint32_t* nxt,
                          uint64_t words, uint64_t root_local, int owns_root, uint32_t* queue,
                          unsigned long long* ctr, const uint64_t* ptr, const uint32_t* iso) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < rows || i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (i < rows) level[i] = owns_root && i == root_local ? 0 : -1;
    if (i < words) {
      // nxt doubles as the frontier block a pull superstep publishes: the
      // root; isolated rows count as visited (pulls skip them)
      const uint32_t rb = owns_root && i == (root_local >> 5) ? 1u << (root_local & 31u) : 0u;
      vis[i] = rb | iso[i];
      nxt[i] = rb;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr[0] = owns_root ? 1 : 0;                                     // found
    ctr[1] = owns_root ? ptr[root_local + 1] - ptr[root_local] : 0;  // their edges
    ctr[2] = 0;                                                      // examined (pull)
    ctr[3] = owns_root ? 1 : 0;                                      // queue length
    if (owns_root) queue[0] = uint32_t(root_local);
  }
}

// Before a push: the frontier rows (set bits of the frontier block) as a
// queue with their degrees; one atomicAdd per warp of 32 words.
__global__ void k_db_queue(const uint32_t* fr, uint64_t words, const uint64_t* ptr, uint32_t* q,
                           uint64_t* qdeg, unsigned long long* qn) {
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); w0 < words;
       w0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t w = w0 + lane_id();
    uint32_t bits = w < words ? fr[w] : 0u;
    const unsigned c = __popc(bits);
    unsigned incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane_id() >= unsigned(o)) incl += t;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) continue;
    unsigned long long base = 0;
    if (lane_id() == 31) base = atomicAdd(qn, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 31) + (incl - c);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint64_t r = w * 32 + uint64_t(b);
      q[base] = uint32_t(r);
      qdeg[base] = ptr[r + 1] - ptr[r];
      ++base;
    }
  }
}

// push: edge-balanced -- thread t takes the t-th frontier edge (its row found
// by a binary search over the queue's degree offsets), so a hub row's edges
// spread over the grid; an owned neighbour is claimed in the next block,
// any other one in the shard's claims bitmap
__global__ void __launch_bounds__(256) k_db_push(const uint32_t* __restrict__ q,
                                                 const uint64_t* __restrict__ qoff, uint64_t nq,
                                                 const uint64_t* __restrict__ ptr,
                                                 const uint32_t* __restrict__ idx, uint64_t lo,
                                                 uint64_t hi, const uint32_t* __restrict__ vis,
                                                 uint32_t* nxt, uint32_t* claims, uint64_t n) {
  const uint64_t total = qoff[nq];
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = 0, b = nq;  // last i with qoff[i] <= t
    while (b - a > 1) {
      const uint64_t mid = (a + b) >> 1;
      if (qoff[mid] <= t)
        a = mid;
      else
        b = mid;
    }
    const uint32_t r = q[a];
    const uint32_t v = __ldg(&idx[ptr[r] + (t - qoff[a])]);
    GM_DCHECK(r < hi - lo && v < n);
    if (v >= lo && v < hi) {
      const uint64_t o = v - lo;
      const uint32_t ob = 1u << (o & 31u);
      if (!(vis[o >> 5] & ob) && !(nxt[o >> 5] & ob)) atomicOr(&nxt[o >> 5], ob);
    } else {
      const uint32_t bit = 1u << (v & 31u);
      if (!(claims[v >> 5] & bit)) atomicOr(&claims[v >> 5], bit);
    }
  }
}

// Row degrees of the owned rows (once per graph), for the pull's frontier
// edge count.
__global__ void k_db_deg(const uint64_t* ptr, uint64_t rows, uint32_t* deg) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x)
    deg[r] = uint32_t(ptr[r + 1] - ptr[r]);
}

// pull: a warp takes 32 consecutive words (one coalesced load of their
// visited bits), then each word with open rows in turn, lane = row, early
// exit at the first frontier neighbour.  Found rows get their level, next-
// frontier and visited bits here (each word is owned by one warp: one ballot,
// no atomics) and the found count and their degrees are summed, so no finish
// pass follows a pull (it had cost ~0.8 ms per large pull at scale 28).
__global__ void __launch_bounds__(256) k_db_pull(const uint64_t* __restrict__ ptr,
                                                  const uint32_t* __restrict__ idx,
                                                  const uint32_t* __restrict__ deg, uint64_t rows,
                                                  uint32_t* vis, const uint32_t* __restrict__ fb,
                                                  uint32_t* nxt, int32_t* level, int32_t lvl,
                                                  uint64_t n, unsigned long long* ctr) {
  unsigned long long ex = 0, f = 0, fe = 0;
  const uint64_t words = (rows + 31) / 32;
  const unsigned lane = lane_id();
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); w0 < words;
       w0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t myvis = w0 + lane < words ? vis[w0 + lane] : 0xFFFFFFFFu;
    unsigned open = __ballot_sync(0xffffffffu, myvis != 0xFFFFFFFFu);
    while (open) {
      const int j = __ffs(open) - 1;
      open &= open - 1;
      const uint64_t w = w0 + uint64_t(j);
      const uint32_t vw = __shfl_sync(0xffffffffu, myvis, j);
      const uint64_t r = w * 32 + lane;
      bool found = false;
      uint32_t d = 0;
      if (r < rows && !((vw >> lane) & 1u)) {
        // the row's neighbours in order, one probe at a time (hub-first
        // rows: the first probe usually decides).  Measured alternatives at
        // scale 28 (superstep 3 / 4): a slot-major head of four neighbours
        // probed in one round 4.39 / 2.53 ms, slot 0 first then the other
        // three 4.76 / 1.70 ms, this walk 2.98 / 1.52 ms -- the frontier
        // bitmap is L2-resident and its random probes are request-bound, so
        // probes beyond the first hit cost more than the latency they hide.
        d = __ldg(&deg[r]);
        const uint64_t b = ptr[r], e1 = b + d;
        for (uint64_t k = b; k < e1; ++k) {
          const uint32_t u = __ldg(&idx[k]);
          GM_DCHECK(u < n);
          ++ex;
          if ((__ldg(&fb[u >> 5]) >> (u & 31u)) & 1u) {
            found = true;
            break;
          }
        }
      }
      const unsigned bits = __ballot_sync(0xffffffffu, found);
      if (found) {
        level[r] = lvl;
        ++f;
        fe += d;
      }
      if (lane == 0 && bits) {
        nxt[w] = bits;  // nxt was cleared for the pull
        vis[w] = vw | bits;
      }
    }
  }
  warp_add_u64(&ctr[0], f);
  warp_add_u64(&ctr[1], fe);
  warp_add_u64(&ctr[2], ex);
}

// owner side of a push: OR in (and clear) this block's words of every shard's claims
__global__ void k_db_claims(PeerTab<uint32_t> claims, int P, uint64_t w0, uint64_t words,
                            uint32_t* nxt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t x = 0;
    for (int q = 0; q < P; ++q) {
      uint32_t* p = claims.p[q] + w0 + i;
      const uint32_t c = *p;
      if (c) {
        x |= c;
        *p = 0;
      }
    }
    if (x) nxt[i] |= x;
  }
}

// new = next & ~visited: levels, visited, and nxt keeps the new bits (the
// frontier block of the next superstep: published before a pull, queued
// before a push); no queue appends here (one atomic per word of a 66 M-vertex
// level serialised on the counter: 6 ms at scale 28)
__global__ void k_db_finish(uint32_t* nxt, uint32_t* vis, uint64_t words, uint64_t rows,
                            int32_t lvl, int32_t* level, const uint64_t* ptr,
                            unsigned long long* ctr) {
  // a warp takes 32 consecutive words (coalesced), then each nonzero word in
  // turn with lane = row (coalesced level writes and degree reads)
  unsigned long long f = 0, fe = 0;
  const unsigned lane = lane_id();
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); w0 < words;
       w0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t wl = w0 + lane;
    uint32_t mine = 0;
    if (wl < words) {
      const uint32_t x = nxt[wl];
      if (x) {
        mine = x & ~vis[wl];
        if (wl * 32 + 32 > rows) mine &= rows > wl * 32 ? (~0u >> (32 - (rows - wl * 32))) : 0u;
        nxt[wl] = mine;
        vis[wl] |= mine;
      }
    }
    unsigned nz = __ballot_sync(0xffffffffu, mine != 0u);
    while (nz) {
      const int j = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t nw = __shfl_sync(0xffffffffu, mine, j);
      if ((nw >> lane) & 1u) {
        const uint64_t r = (w0 + uint64_t(j)) * 32 + lane;
        level[r] = lvl;
        fe += ptr[r + 1] - ptr[r];
        ++f;
      }
    }
  }
  warp_add_u64(&ctr[0], f);
  warp_add_u64(&ctr[1], fe);
}

// the new-frontier words of this block into every shard's frontier bitmap
__global__ void k_db_publish(const uint32_t* nxt, uint64_t w0, uint64_t words, PeerTab<uint32_t> fb,
                             int P) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t x = nxt[i];
    for (int q = 0; q < P; ++q) fb.p[q][w0 + i] = x;
  }
}

DBfsState& dbfs_state(DGraph& g) {
  if (g.bfs) return *g.bfs;
  Comm& c = *g.comm;
  g.bfs = std::unique_ptr<DBfsState, void (*)(DBfsState*)>(new DBfsState(),
                                                           [](DBfsState* p) { delete p; });
  DBfsState& st = *g.bfs;
  const int L = c.L;
  st.level.resize(static_cast<size_t>(L));
  st.vis.resize(static_cast<size_t>(L));
  st.nxt.resize(static_cast<size_t>(L));
  st.queue.resize(static_cast<size_t>(L));
  st.qdeg.resize(static_cast<size_t>(L));
  st.iso.resize(static_cast<size_t>(L));
  st.deg.resize(static_cast<size_t>(L));
  st.ctr.resize(static_cast<size_t>(L));
  st.sum.resize(static_cast<size_t>(L));
  const uint64_t words_all = (g.n + 31) / 32;
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    const uint64_t rows = g.sh[size_t(l)].hi - g.sh[size_t(l)].lo;
    const uint64_t words = (rows + 31) / 32;
    st.level[size_t(l)].alloc(rows + 1, s);
    st.vis[size_t(l)].alloc(words + 1, s);
    st.nxt[size_t(l)].alloc(words + 1, s);
    st.queue[size_t(l)].alloc(rows + 1, s);
    st.qdeg[size_t(l)].alloc(rows + 2, s);
    st.iso[size_t(l)].alloc(words + 1, s);
    launch(words, s, [&](unsigned gr, unsigned bl) {
      k_db_isolated<<<gr, bl, 0, s>>>(g.sh[size_t(l)].in.ptr.get(), rows, st.iso[size_t(l)].get());
    });
    st.deg[size_t(l)].alloc(rows + 1, s);
    if (rows)
      k_db_deg<<<grid_for(rows, 256), 256, 0, s>>>(g.sh[size_t(l)].in.ptr.get(), rows,
                                                  st.deg[size_t(l)].get());
    GM_LAUNCH_CHECK();
    st.ctr[size_t(l)].alloc(4, s);
    st.sum[size_t(l)].alloc(4, s);
    st.nxt[size_t(l)].zero(s);
    for (int b = 0; b < 2; ++b) st.fb[b].push_back(c.peer_alloc(l, words_all * 4));
    st.claims.push_back(c.peer_alloc(l, words_all * 4));
    GM_CUDA(cudaMemsetAsync(st.claims.back(), 0, words_all * 4, s));
    GM_CUDA(cudaStreamSynchronize(s));
  }
  st.c = &c;
  for (int b = 0; b < 2; ++b) st.fb_tab[b] = c.share(st.fb[b]);
  st.claims_tab = c.share(st.claims);
  return st;
}

template <typename T>
PeerTab<T> tab_of(const std::vector<void*>& row, int P) {
  PeerTab<T> t{};
  for (int q = 0; q < P; ++q) t.p[q] = static_cast<T*>(row[size_t(q)]);
  return t;
}

struct StepTimer {
  cudaEvent_t e[4]{};
  explicit StepTimer() {
    for (auto& x : e) GM_CUDA(cudaEventCreate(&x));
  }
  ~StepTimer() {
    for (auto& x : e) cudaEventDestroy(x);
  }
  double ms(int a, int b) const {
    float x = 0.f;
    if (cudaEventElapsedTime(&x, e[a], e[b]) != cudaSuccess) {
      (void)cudaGetLastError();
      return 0.0;
    }
    return x;
  }
};

}  // namespace

std::vector<gm_iteration_stats> dbfs(DGraph& g, uint64_t root, int64_t max_iters, int32_t* out,
                                     bool out_on_device) {
  Comm& c = *g.comm;
  if (!g.symmetric) fail(GM_EUSAGE, "dgraph bfs: needs a symmetric graph (GM_SYMMETRIZE)");
  if (root >= g.n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(g.n));
  DBfsState& st = dbfs_state(g);
  const int L = c.L, P = c.P;
  const uint64_t n = g.n, m = g.m;
  const uint64_t ro = g.owner(root);
  c.set(0);
  HostPinned<unsigned long long> h(4);
  std::vector<std::vector<gm_iteration_stats>> none;
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    const uint64_t rows = sh.hi - sh.lo, words = (rows + 31) / 32;
    const int owns = uint64_t(c.global(l)) == ro;
    k_db_init<<<grid_for(std::max(rows, words) + 1, kBlock), kBlock, 0, s>>>(
        st.level[size_t(l)].get(), rows, st.vis[size_t(l)].get(), st.nxt[size_t(l)].get(), words,
        owns ? root - sh.lo : 0,
        owns, st.queue[size_t(l)].get(), st.ctr[size_t(l)].get(), sh.in.ptr.get(),
        st.iso[size_t(l)].get());
    GM_LAUNCH_CHECK();
  }
  std::vector<const uint64_t*> cin;
  std::vector<uint64_t*> cout_;
  for (int l = 0; l < L; ++l) {
    cin.push_back(reinterpret_cast<const uint64_t*>(st.ctr[size_t(l)].get()));
    cout_.push_back(reinterpret_cast<uint64_t*>(st.sum[size_t(l)].get()));
  }
  StepTimer tm;
  std::vector<gm_iteration_stats> stats;
  uint64_t nf = 1, ef = 0;
  {
    // the root's degree: first summed counters
    c.allreduce_u64(cin, cout_, 4);
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(h.get(), st.sum[0].get(), 32, cudaMemcpyDeviceToHost, c.st[0]));
    GM_CUDA(cudaStreamSynchronize(c.st[0]));
    ef = h[1];
  }
  int dir = kPush;
  int cur = 0;
  for (int64_t it = 1; nf > 0 && it <= max_iters; ++it) {
    // direction (the single-GPU rule of k_bfs_coop)
    int nd = dir;
    if (dir == kPush && ef * 20 > m) nd = kPull;
    else if (dir == kPull && nf * 24 < n) nd = kPush;
    if (nd == kPull) {
      // publish the current frontier blocks into every shard's bitmap
      for (int l = 0; l < L; ++l) {
        c.set(l);
        cudaStream_t s = c.st[size_t(l)];
        DShard& sh = g.sh[size_t(l)];
        const uint64_t words = (sh.hi - sh.lo + 31) / 32;
        if (l == 0) GM_CUDA(cudaEventRecord(tm.e[2], s));
        launch(words, s, [&](unsigned gr, unsigned bl) {
          k_db_publish<<<gr, bl, 0, s>>>(st.nxt[size_t(l)].get(), sh.lo / 32, words,
                                         tab_of<uint32_t>(st.fb_tab[cur][size_t(l)], P), P);
        });
      }
      c.barrier();
    } else if (L > 0) {
      c.set(0);
      GM_CUDA(cudaEventRecord(tm.e[2], c.st[0]));
    }
    // push: every shard's frontier rows as a queue with degree offsets (one
    // host read of the queue lengths: the scan and the grid need them)
    std::vector<uint64_t> nq(static_cast<size_t>(L), 0);
    if (nd == kPush) {
      for (int l = 0; l < L; ++l) {
        c.set(l);
        cudaStream_t s = c.st[size_t(l)];
        DShard& sh = g.sh[size_t(l)];
        const uint64_t words = (sh.hi - sh.lo + 31) / 32;
        GM_CUDA(cudaMemsetAsync(st.ctr[size_t(l)].get() + 3, 0, 8, s));
        launch(words, s, [&](unsigned gr, unsigned bl) {
          k_db_queue<<<gr, bl, 0, s>>>(st.nxt[size_t(l)].get(), words, sh.in.ptr.get(),
                                       st.queue[size_t(l)].get(), st.qdeg[size_t(l)].get(),
                                       st.ctr[size_t(l)].get() + 3);
        });
        GM_CUDA(cudaMemcpyAsync(&h[3], st.ctr[size_t(l)].get() + 3, 8, cudaMemcpyDeviceToHost, s));
        GM_CUDA(cudaStreamSynchronize(s));
        nq[size_t(l)] = h[3];
        GM_CUDA(cudaMemsetAsync(st.qdeg[size_t(l)].get() + nq[size_t(l)], 0, 8, s));
        exclusive_scan_u64(st.qdeg[size_t(l)].get(), nq[size_t(l)] + 1, s);
      }
    }
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      const uint64_t rows = sh.hi - sh.lo, words = (rows + 31) / 32;
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[0], s));
      GM_CUDA(cudaMemsetAsync(st.ctr[size_t(l)].get(), 0, 32, s));
      if (nd == kPush) {
        if (nq[size_t(l)]) {
          k_db_push<<<grid_for(std::max<uint64_t>(ef, 1), 256), 256, 0, s>>>(
              st.queue[size_t(l)].get(), st.qdeg[size_t(l)].get(), nq[size_t(l)], sh.in.ptr.get(),
              sh.in.idx.get(), sh.lo, sh.hi, st.vis[size_t(l)].get(), st.nxt[size_t(l)].get(),
              static_cast<uint32_t*>(st.claims[size_t(l)]), n);
          GM_LAUNCH_CHECK();
        }
      } else {
        // nxt holds the published frontier block: clear it for the claims
        if (words) GM_CUDA(cudaMemsetAsync(st.nxt[size_t(l)].get(), 0, words * 4, s));
        launch(rows, s, [&](unsigned gr, unsigned bl) {
          k_db_pull<<<gr, bl, 0, s>>>(sh.in.ptr.get(), sh.in.idx.get(), st.deg[size_t(l)].get(), rows, st.vis[size_t(l)].get(),
                                       static_cast<const uint32_t*>(st.fb[cur][size_t(l)]),
                                       st.nxt[size_t(l)].get(), st.level[size_t(l)].get(),
                                       int32_t(it), n, st.ctr[size_t(l)].get());
        });
      }
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[1], s));
    }
    if (nd == kPush) {
      c.barrier();
      for (int l = 0; l < L; ++l) {
        c.set(l);
        cudaStream_t s = c.st[size_t(l)];
        DShard& sh = g.sh[size_t(l)];
        const uint64_t words = (sh.hi - sh.lo + 31) / 32;
        launch(words, s, [&](unsigned gr, unsigned bl) {
          k_db_claims<<<gr, bl, 0, s>>>(tab_of<uint32_t>(st.claims_tab[size_t(l)], P), P, sh.lo / 32,
                                        words, st.nxt[size_t(l)].get());
        });
      }
      // nobody expands into a claims bitmap before its owner cleared it
      c.barrier();
    }
    // a pull already wrote levels, visited and next-frontier bits and counted
    // what it found; a push's claims are resolved here
    for (int l = 0; l < L && nd == kPush; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      const uint64_t rows = sh.hi - sh.lo, words = (rows + 31) / 32;
      launch(words * 32, s, [&](unsigned gr, unsigned bl) {
        k_db_finish<<<gr, bl, 0, s>>>(st.nxt[size_t(l)].get(), st.vis[size_t(l)].get(), words, rows,
                                      int32_t(it), st.level[size_t(l)].get(), sh.in.ptr.get(),
                                      st.ctr[size_t(l)].get());
      });
    }
    c.allreduce_u64(cin, cout_, 4);
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(h.get(), st.sum[0].get(), 32, cudaMemcpyDeviceToHost, c.st[0]));
    GM_CUDA(cudaEventRecord(tm.e[3], c.st[0]));
    GM_CUDA(cudaStreamSynchronize(c.st[0]));
    gm_iteration_stats s{};
    s.iteration = it;
    s.active_before = int64_t(nf);
    s.messages_generated = int64_t(nf);
    s.vertices_updated = int64_t(h[0]);
    s.direction = nd == kPush ? 1 : 0;
    s.edges_processed = int64_t(nd == kPush ? ef : h[2]);
    s.spmv_seconds = tm.ms(0, 1) * 1e-3;
    s.total_seconds = tm.ms(2, 3) * 1e-3;
    s.comm_seconds = std::max(0.0, s.total_seconds - s.spmv_seconds);
    s.bytes_algorithmic = nd == kPush
                              ? int64_t(24 * nf + 4 * ef + 16 * h[0] + n / 8)
                              : int64_t(16 * n + 4 * h[2] + 4 * h[0] + 2 * n / 8);
    stats.push_back(s);
    nf = h[0];
    ef = h[1];
    dir = nd;
    cur ^= 1;
    (void)none;
  }
  // levels of the owned rows, concatenated in shard order
  if (out) {
    uint64_t off = 0;
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      const uint64_t rows = g.sh[size_t(l)].hi - g.sh[size_t(l)].lo;
      if (rows)
        GM_CUDA(cudaMemcpyAsync(out + off, st.level[size_t(l)].get(), rows * 4,
                                out_on_device ? cudaMemcpyDefault : cudaMemcpyDeviceToHost, s));
      off += rows;
    }
  }
  for (int l = 0; l < L; ++l) {
    c.set(l);
    GM_CUDA(cudaStreamSynchronize(c.st[size_t(l)]));
  }
  return stats;
}


// ============================================================================
// PageRank over the row shards (BASELINE configs[4]; the program of
// pagerank.hpp:36-63 driven like the CF driver, collaborative_filtering.hpp:
// 181-193 -- the same formula as gm_pagerank).
//
// Superstep t on shard r: every owned row v folds x_t over its in-entries in
// ascending caller-id order (a thread per row up to kPrShort entries; longer
// rows in fixed chunks of kPrChunk entries, a warp per chunk with a fixed
// shuffle tree, the chunks folded in order) -- the reduction tree depends only
// on the row, so ranks are bitwise identical for any number of shards.
// rank_{t+1}(v) = base_t + d * sum; a vertex with out-edges stores its message
// rank/outdeg at its packed id into EVERY shard's x_{t+1} (peer stores: the
// all-gather fused into the epilogue); a dangling vertex adds its rank to the
// dangling mass as a 63-bit fixed-point integer split in two 32-bit limbs, so
// the sum over shards is exact and order-free.  One u64 all-reduce of
// {limb0, limb1, updated} per superstep is the barrier; base_{t+1} =
// (1-d)/N + d*D/N is computed on the device from it.  No host synchronisation
// inside the 20 supersteps.
// ============================================================================
namespace {

constexpr uint32_t kPrShort = 32;
constexpr uint64_t kPrChunk = 4096;

struct DPrArgs {
  const uint64_t* ptr;
  const uint32_t* idx;
  const uint32_t* pid;
  const float* inv;
  const float* x;                 // x_t (packed, local copy)
  float* rank;
  PeerTab<float> xn;              // x_{t+1} of every shard
  int P;
  const unsigned long long* sum;  // summed {limb0, limb1, updated} of rank_t
  unsigned long long* part;       // this shard's words for rank_{t+1}
  double one_minus_d_over_n, d_over_n;
  float d;
  uint64_t nx;  // packed message ids < nx
};

__device__ __forceinline__ float dpr_base(const DPrArgs& a) {
  const double D = (double(a.sum[1]) * 4294967296.0 + double(a.sum[0])) * 0x1p-63;
  return float(a.one_minus_d_over_n + a.d_over_n * D);
}

struct DprAcc {
  unsigned long long l0 = 0, l1 = 0, upd = 0;
};

__device__ __forceinline__ void dpr_apply(const DPrArgs& a, uint32_t r, float sum, float base,
                                          bool has_in, DprAcc& acc) {
  const float nr = base + a.d * sum;
  const float old = a.rank[r];
  acc.upd += has_in && __float_as_uint(nr) != __float_as_uint(old);
  a.rank[r] = nr;
  const uint32_t p = a.pid[r];
  if (p != ~0u) {
    GM_DCHECK(p < a.nx);
    const float xv = nr * a.inv[r];
    for (int q = 0; q < a.P; ++q) a.xn.p[q][p] = xv;
  } else {
    const unsigned long long f = __float2ull_rz(nr * 9.223372036854775808e18f);
    acc.l0 += f & 0xFFFFFFFFull;
    acc.l1 += f >> 32;
  }
}

__device__ __forceinline__ void dpr_flush(const DPrArgs& a, const DprAcc& acc) {
  warp_add_u64(&a.part[0], acc.l0);
  warp_add_u64(&a.part[1], acc.l1);
  warp_add_u64(&a.part[2], acc.upd);
}

// Rows of <= kPrShort entries, a thread per row in row order (neighbouring
// threads read neighbouring offsets, ranks and packed ids), the entries
// folded in stored order with four gathers in flight.  Longer rows are left
// to the chunk path.  (A group of 8 lanes per row was slower: most rows have
// a few entries -- 79 -> 47 GTEPS at scale 28.)
__global__ void __launch_bounds__(256) k_dpr_short(DPrArgs a, uint64_t rows) {
  const float base = dpr_base(a);
  DprAcc acc;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = a.ptr[r], e = a.ptr[r + 1];
    if (e - b > kPrShort) continue;
    float s = 0.0f;
    uint64_t k = b;
    for (; k + 4 <= e; k += 4) {
      const uint32_t i0 = __ldg(&a.idx[k]), i1 = __ldg(&a.idx[k + 1]);
      const uint32_t i2 = __ldg(&a.idx[k + 2]), i3 = __ldg(&a.idx[k + 3]);
      GM_DCHECK(i0 < a.nx && i1 < a.nx && i2 < a.nx && i3 < a.nx);
      const float x0 = __ldg(&a.x[i0]), x1 = __ldg(&a.x[i1]);
      const float x2 = __ldg(&a.x[i2]), x3 = __ldg(&a.x[i3]);
      s += x0;
      s += x1;
      s += x2;
      s += x3;
    }
    for (; k < e; ++k) {
      GM_DCHECK(a.idx[k] < a.nx);
      s += __ldg(&a.x[__ldg(&a.idx[k])]);
    }
    dpr_apply(a, uint32_t(r), s, base, e > b, acc);
  }
  dpr_flush(a, acc);
}

// warp per chunk of a long row: lane-strided partials, fixed xor tree
__global__ void __launch_bounds__(256) k_dpr_chunks(DPrArgs a, const uint64_t* beg, uint64_t nc,
                                                    const uint64_t* row_end_of_chunk, float* out) {
  const uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t c = w; c < nc; c += nw) {
    const uint64_t b = beg[c], e = row_end_of_chunk[c];
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    uint64_t k = b + lane;
    for (; k + 96 < e; k += 128) {
      const uint32_t i0 = __ldg(&a.idx[k]), i1 = __ldg(&a.idx[k + 32]);
      const uint32_t i2 = __ldg(&a.idx[k + 64]), i3 = __ldg(&a.idx[k + 96]);
      s0 += __ldg(&a.x[i0]);
      s1 += __ldg(&a.x[i1]);
      s2 += __ldg(&a.x[i2]);
      s3 += __ldg(&a.x[i3]);
    }
    for (; k < e; k += 32) s0 += __ldg(&a.x[__ldg(&a.idx[k])]);
    float s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
  }
}

__global__ void __launch_bounds__(256) k_dpr_long(DPrArgs a, const uint32_t* rows, uint64_t nr,
                                                  const uint32_t* chunk0, const float* csum) {
  const float base = dpr_base(a);
  DprAcc acc;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nr;
       i += uint64_t(gridDim.x) * blockDim.x) {
    float s = 0.0f;
    for (uint32_t c = chunk0[i]; c < chunk0[i + 1]; ++c) s += csum[c];
    dpr_apply(a, rows[i], s, base, true, acc);
  }
  dpr_flush(a, acc);
}

__global__ void k_dpr_init(uint64_t rows, float r0, const uint32_t* pid, const float* inv,
                           float* rank, PeerTab<float> x0, int P, unsigned long long* part) {
  DprAcc acc;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    rank[r] = r0;
    const uint32_t p = pid[r];
    if (p != ~0u) {
      const float xv = r0 * inv[r];
      for (int q = 0; q < P; ++q) x0.p[q][p] = xv;
    } else {
      const unsigned long long f = __float2ull_rz(r0 * 9.223372036854775808e18f);
      acc.l0 += f & 0xFFFFFFFFull;
      acc.l1 += f >> 32;
    }
  }
  warp_add_u64(&part[0], acc.l0);
  warp_add_u64(&part[1], acc.l1);
}

__global__ void k_dpr_classify(const uint64_t* ptr, uint64_t rows, const uint32_t* od, float* inv,
                               uint32_t* rs, uint32_t* rl, uint32_t* nchunks,
                               unsigned long long* cnt) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    inv[r] = od[r] ? 1.0f / float(od[r]) : 0.0f;
    const uint64_t d = ptr[r + 1] - ptr[r];
    if (d <= kPrShort) {
      rs[atomicAdd(&cnt[0], 1ull)] = uint32_t(r);
    } else {
      const unsigned long long i = atomicAdd(&cnt[1], 1ull);
      rl[i] = uint32_t(r);
      nchunks[i] = uint32_t((d + kPrChunk - 1) / kPrChunk);
    }
  }
}

__global__ void k_dpr_chunk_ranges(const uint64_t* ptr, const uint32_t* rl, uint64_t nl,
                                   const uint64_t* c0, uint64_t* beg, uint64_t* end,
                                   uint32_t* chunk0) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i <= nl;
       i += uint64_t(gridDim.x) * blockDim.x) {
    chunk0[i] = uint32_t(c0[i]);
    if (i == nl) continue;
    const uint32_t r = rl[i];
    const uint64_t b = ptr[r], e = ptr[r + 1];
    uint64_t c = c0[i];
    for (uint64_t k = b; k < e; k += kPrChunk, ++c) {
      beg[c] = k;
      end[c] = k + kPrChunk < e ? k + kPrChunk : e;
    }
  }
}

DPrState& dpr_state(DGraph& g) {
  if (g.pr) return *g.pr;
  Comm& c = *g.comm;
  g.pr = std::unique_ptr<DPrState, void (*)(DPrState*)>(new DPrState(), [](DPrState* p) { delete p; });
  DPrState& st = *g.pr;
  const int L = c.L;
  for (auto* v : {&st.rank, &st.inv}) v->resize(static_cast<size_t>(L));
  st.rows_short.resize(static_cast<size_t>(L));
  st.rows_long.resize(static_cast<size_t>(L));
  st.chunk_beg.resize(static_cast<size_t>(L));
  st.long_chunk0.resize(static_cast<size_t>(L));
  st.chunk_sum.resize(static_cast<size_t>(L));
  st.part.resize(static_cast<size_t>(L));
  st.sum.resize(static_cast<size_t>(L));
  st.n_short.assign(size_t(L), 0);
  st.n_long.assign(size_t(L), 0);
  st.n_chunks.assign(size_t(L), 0);
  const uint64_t nx = std::max<uint64_t>(g.nonzero_outdeg, 1);
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    const uint64_t rows = sh.hi - sh.lo;
    st.rank[size_t(l)].alloc(rows + 1, s);
    st.inv[size_t(l)].alloc(rows + 1, s);
    st.rows_short[size_t(l)].alloc(rows + 1, s);
    st.rows_long[size_t(l)].alloc(rows + 1, s);
    DevBuf<uint32_t> nch(rows + 1, s);
    DevBuf<unsigned long long> cnt(2, s);
    cnt.zero(s);
    launch(rows, s, [&](unsigned gr, unsigned bl) {
      k_dpr_classify<<<gr, bl, 0, s>>>(sh.in.ptr.get(), rows, sh.outdeg.get(), st.inv[size_t(l)].get(),
                                       st.rows_short[size_t(l)].get(), st.rows_long[size_t(l)].get(),
                                       nch.get(), cnt.get());
    });
    unsigned long long hc[2];
    GM_CUDA(cudaMemcpyAsync(hc, cnt.get(), 16, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    st.n_short[size_t(l)] = hc[0];
    const uint64_t nl = hc[1];
    st.n_long[size_t(l)] = nl;
    DevBuf<uint64_t> c0(nl + 1, s);
    scan_counts_to_ptr(nch.get(), c0.get(), nl, s);
    uint64_t nc = 0;
    GM_CUDA(cudaMemcpyAsync(&nc, c0.get() + nl, 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    st.n_chunks[size_t(l)] = nc;
    st.chunk_beg[size_t(l)].alloc(2 * nc + 2, s);  // [beg | end]
    st.long_chunk0[size_t(l)].alloc(nl + 1, s);
    st.chunk_sum[size_t(l)].alloc(nc + 1, s);
    launch(nl + 1, s, [&](unsigned gr, unsigned bl) {
      k_dpr_chunk_ranges<<<gr, bl, 0, s>>>(sh.in.ptr.get(), st.rows_long[size_t(l)].get(), nl,
                                           c0.get(), st.chunk_beg[size_t(l)].get(),
                                           st.chunk_beg[size_t(l)].get() + nc + 1,
                                           st.long_chunk0[size_t(l)].get());
    });
    st.part[size_t(l)].alloc(8, s);
    st.sum[size_t(l)].alloc(8, s);
    for (int b = 0; b < 2; ++b) st.x[b].push_back(c.peer_alloc(l, nx * 4));
    GM_CUDA(cudaStreamSynchronize(s));
  }
  st.c = &c;
  for (int b = 0; b < 2; ++b) st.x_tab[b] = c.share(st.x[b]);
  return st;
}

}  // namespace

std::vector<gm_iteration_stats> dpagerank(DGraph& g, double damping, int64_t iters, float* out,
                                          bool out_on_device) {
  Comm& c = *g.comm;
  if (g.symmetric) fail(GM_EUSAGE, "dgraph pagerank: needs a directed graph");
  if (!(damping >= 0.0 && damping <= 1.0)) fail(GM_EINPUT, "pagerank: damping must be in [0, 1]");
  DPrState& st = dpr_state(g);
  const int L = c.L, P = c.P;
  const uint64_t n = g.n;
  const int64_t ni = std::max<int64_t>(iters, 0);
  c.set(0);
  st.trace.alloc(size_t(ni + 1) * 4, c.st[0]);
  std::vector<const uint64_t*> pin[2];
  std::vector<uint64_t*> pout[2];
  for (int b = 0; b < 2; ++b)
    for (int l = 0; l < L; ++l) {
      pin[b].push_back(reinterpret_cast<const uint64_t*>(st.part[size_t(l)].get() + 4 * b));
      pout[b].push_back(reinterpret_cast<uint64_t*>(st.sum[size_t(l)].get() + 4 * b));
    }
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    const uint64_t rows = sh.hi - sh.lo;
    st.part[size_t(l)].zero(s);
    launch(rows, s, [&](unsigned gr, unsigned bl) {
      k_dpr_init<<<gr, bl, 0, s>>>(rows, float(1.0 / double(n)), sh.pid.get(), st.inv[size_t(l)].get(),
                                   st.rank[size_t(l)].get(), tab_of<float>(st.x_tab[0][size_t(l)], P),
                                   P, st.part[size_t(l)].get());
    });
  }
  c.allreduce_u64(pin[0], pout[0], 4);
  std::vector<std::unique_ptr<StepTimer>> tms;
  for (int64_t t = 0; t < ni; ++t) {
    const int p = int(t & 1), q = p ^ 1;
    tms.emplace_back(new StepTimer());
    StepTimer& tm = *tms.back();
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[0], s));
      GM_CUDA(cudaMemsetAsync(st.part[size_t(l)].get() + 4 * q, 0, 32, s));
      DPrArgs a{};
      a.ptr = sh.in.ptr.get();
      a.idx = sh.in.idx.get();
      a.pid = sh.pid.get();
      a.inv = st.inv[size_t(l)].get();
      a.x = static_cast<const float*>(st.x[p][size_t(l)]);
      a.rank = st.rank[size_t(l)].get();
      a.xn = tab_of<float>(st.x_tab[q][size_t(l)], P);
      a.P = P;
      a.sum = st.sum[size_t(l)].get() + 4 * p;
      a.part = st.part[size_t(l)].get() + 4 * q;
      a.one_minus_d_over_n = (1.0 - damping) / double(n);
      a.d_over_n = damping / double(n);
      a.d = float(damping);
      a.nx = std::max<uint64_t>(g.nonzero_outdeg, 1);
      const uint64_t nc = st.n_chunks[size_t(l)];
      if (nc) {
        k_dpr_chunks<<<grid_for(nc * 32, 256), 256, 0, s>>>(
            a, st.chunk_beg[size_t(l)].get(), nc, st.chunk_beg[size_t(l)].get() + nc + 1,
            st.chunk_sum[size_t(l)].get());
        GM_LAUNCH_CHECK();
      }
      launch(sh.hi - sh.lo, s, [&](unsigned gr, unsigned bl) {
        k_dpr_short<<<gr, bl, 0, s>>>(a, sh.hi - sh.lo);
      });
      launch(st.n_long[size_t(l)], s, [&](unsigned gr, unsigned bl) {
        k_dpr_long<<<gr, bl, 0, s>>>(a, st.rows_long[size_t(l)].get(), st.n_long[size_t(l)],
                                     st.long_chunk0[size_t(l)].get(), st.chunk_sum[size_t(l)].get());
      });
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[1], s));
    }
    c.allreduce_u64(pin[q], pout[q], 4);
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(st.trace.get() + 4 * t, st.sum[0].get() + 4 * q, 32,
                            cudaMemcpyDeviceToDevice, c.st[0]));
    GM_CUDA(cudaEventRecord(tm.e[2], c.st[0]));
  }
  // ranks of the owned rows, concatenated in shard order
  if (out) {
    uint64_t off = 0;
    for (int l = 0; l < L; ++l) {
      c.set(l);
      const uint64_t rows = g.sh[size_t(l)].hi - g.sh[size_t(l)].lo;
      if (rows)
        GM_CUDA(cudaMemcpyAsync(out + off, st.rank[size_t(l)].get(), rows * 4,
                                out_on_device ? cudaMemcpyDefault : cudaMemcpyDeviceToHost,
                                c.st[size_t(l)]));
      off += rows;
    }
  }
  std::vector<unsigned long long> tr(size_t(ni + 1) * 4);
  c.set(0);
  if (ni)
    GM_CUDA(cudaMemcpyAsync(tr.data(), st.trace.get(), size_t(ni) * 32, cudaMemcpyDeviceToHost, c.st[0]));
  for (int l = 0; l < L; ++l) {
    c.set(l);
    GM_CUDA(cudaStreamSynchronize(c.st[size_t(l)]));
  }
  std::vector<gm_iteration_stats> stats;
  uint64_t nnz_local = 0;
  for (auto& sh : g.sh) nnz_local += sh.in.nnz;
  for (int64_t t = 0; t < ni; ++t) {
    gm_iteration_stats s{};
    s.iteration = t + 1;
    s.active_before = int64_t(n);
    s.messages_generated = int64_t(g.nonzero_outdeg);
    s.vertices_updated = int64_t(tr[size_t(t) * 4 + 2]);
    s.spmv_seconds = tms[size_t(t)]->ms(0, 1) * 1e-3;
    s.total_seconds = tms[size_t(t)]->ms(0, 2) * 1e-3;
    s.comm_seconds = std::max(0.0, s.total_seconds - s.spmv_seconds);
    s.edges_processed = int64_t(nnz_local);
    s.bytes_algorithmic = int64_t(4 * nnz_local + 8 * (n / uint64_t(P) + 1) + 16 * (n / uint64_t(P)));
    s.direction = 0;
    stats.push_back(s);
  }
  return stats;
}

}  // namespace gm

// ---- seed-chosen source on a sharded graph (the rule of pick_source, ingest.cu:
// the first of mix64(base + i) % n with out-edges; BASELINE configs[1..2]) ----
namespace gm {
namespace {

__global__ void k_cand_deg(const uint64_t* ptr, const uint32_t* outdeg, uint64_t lo, uint64_t hi,
                           uint64_t base, uint64_t n, uint64_t i0, int count,
                           unsigned long long* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t v = mix64(base + i0 + uint64_t(i)) % n;
  unsigned long long f = 0;
  if (v >= lo && v < hi) {
    const uint64_t r = v - lo;
    f = outdeg ? outdeg[r] > 0 : ptr[r + 1] > ptr[r];
  }
  flag[i] = f;
}

__global__ void k_first_nonempty(const uint64_t* ptr, const uint32_t* outdeg, uint64_t rows,
                                 uint64_t lo, unsigned long long* first) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x)
    if (outdeg ? outdeg[r] > 0 : ptr[r + 1] > ptr[r]) atomicMin(first, (unsigned long long)(lo + r));
}

}  // namespace

uint64_t dpick_source(DGraph& g, uint64_t seed) {
  Comm& c = *g.comm;
  const uint64_t n = g.n;
  const uint64_t base = mix64(seed ^ 0x50C0FFEEull);
  constexpr int kBatch = 1024;
  std::vector<DevBuf<unsigned long long>> f(static_cast<size_t>(c.L)), fs(static_cast<size_t>(c.L));
  std::vector<const uint64_t*> in;
  std::vector<uint64_t*> out;
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    const DShard& sh = g.sh[size_t(l)];
    f[size_t(l)].alloc(kBatch, s);
    fs[size_t(l)].alloc(kBatch, s);
    k_cand_deg<<<(kBatch + 255) / 256, 256, 0, s>>>(sh.in.ptr.get(), g.symmetric ? nullptr : sh.outdeg.get(),
                                                    sh.lo, sh.hi, base, n, 0, kBatch, f[size_t(l)].get());
    GM_LAUNCH_CHECK();
    in.push_back(reinterpret_cast<const uint64_t*>(f[size_t(l)].get()));
    out.push_back(reinterpret_cast<uint64_t*>(fs[size_t(l)].get()));
  }
  c.allreduce_u64(in, out, kBatch);
  std::vector<unsigned long long> h(kBatch);
  c.set(0);
  GM_CUDA(cudaMemcpyAsync(h.data(), fs[0].get(), kBatch * 8, cudaMemcpyDeviceToHost, c.st[0]));
  GM_CUDA(cudaStreamSynchronize(c.st[0]));
  for (int i = 0; i < kBatch; ++i)
    if (h[size_t(i)]) return mix64(base + uint64_t(i)) % n;
  // no candidate hit: the smallest vertex with out-edges (min over shards)
  std::vector<std::vector<uint64_t>> firsts(static_cast<size_t>(c.L));
  std::vector<DevBuf<unsigned long long>> m1(static_cast<size_t>(c.L)), ms(static_cast<size_t>(c.L));
  in.clear();
  out.clear();
  const size_t P = size_t(c.P);
  for (int l = 0; l < c.L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    const DShard& sh = g.sh[size_t(l)];
    m1[size_t(l)].alloc(P, s);
    ms[size_t(l)].alloc(P, s);
    m1[size_t(l)].zero(s);
    DevBuf<unsigned long long> first(1, s);
    GM_CUDA(cudaMemsetAsync(first.get(), 0xFF, 8, s));
    launch(sh.hi - sh.lo, s, [&](unsigned gr, unsigned bl) {
      k_first_nonempty<<<gr, bl, 0, s>>>(sh.in.ptr.get(), g.symmetric ? nullptr : sh.outdeg.get(),
                                         sh.hi - sh.lo, sh.lo, first.get());
    });
    unsigned long long v = 0;
    GM_CUDA(cudaMemcpyAsync(&v, first.get(), 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    const unsigned long long enc = v == ~0ull ? 0 : v + 1;  // 0 = none
    GM_CUDA(cudaMemcpyAsync(m1[size_t(l)].get() + c.global(l), &enc, 8, cudaMemcpyHostToDevice, s));
    GM_CUDA(cudaStreamSynchronize(s));
    in.push_back(reinterpret_cast<const uint64_t*>(m1[size_t(l)].get()));
    out.push_back(reinterpret_cast<uint64_t*>(ms[size_t(l)].get()));
  }
  c.allreduce_u64(in, out, P);
  std::vector<unsigned long long> hm(P);
  c.set(0);
  GM_CUDA(cudaMemcpyAsync(hm.data(), ms[0].get(), P * 8, cudaMemcpyDeviceToHost, c.st[0]));
  GM_CUDA(cudaStreamSynchronize(c.st[0]));
  for (size_t q = 0; q < P; ++q)
    if (hm[q]) return hm[q] - 1;
  return 0;
}

}  // namespace gm

// degree_vector (engine.hpp:295-312) of the owned rows: kind 0 = IN (row
// lengths of CSR(G^T)), 1 = OUT.
namespace gm {
namespace {
__global__ void k_row_lengths(const uint64_t* ptr, uint64_t rows, uint32_t* out) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x)
    out[r] = uint32_t(ptr[r + 1] - ptr[r]);
}
}  // namespace

void ddegrees(DGraph& g, int l, int kind, uint32_t* out_host) {
  Comm& c = *g.comm;
  if (l < 0 || l >= c.L) fail(GM_EUSAGE, "bad shard");
  if (kind != 0 && kind != 1) fail(GM_EUSAGE, "degree kind must be 0 (IN) or 1 (OUT)");
  c.set(l);
  cudaStream_t s = c.st[size_t(l)];
  const DShard& sh = g.sh[size_t(l)];
  const uint64_t rows = sh.hi - sh.lo;
  if (!rows) return;
  if (kind == 1 && !g.symmetric) {
    GM_CUDA(cudaMemcpyAsync(out_host, sh.outdeg.get(), rows * 4, cudaMemcpyDeviceToHost, s));
  } else {
    DevBuf<uint32_t> d(rows, s);
    launch(rows, s, [&](unsigned gr, unsigned bl) {
      k_row_lengths<<<gr, bl, 0, s>>>(sh.in.ptr.get(), rows, d.get());
    });
    GM_CUDA(cudaMemcpyAsync(out_host, d.get(), rows * 4, cudaMemcpyDeviceToHost, s));
  }
  GM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gm

namespace gm {

// ============================================================================
// SSSP over the row shards (algo::sssp, traversal.hpp:125-133; BSP
// Bellman-Ford on integer weights, the superstep-start distances of the
// frontier are the messages, rule S3).
//
// Per superstep, on every shard (direction: pull once the frontier's
// out-edges exceed m/6, the single-GPU rule):
//   push: the shard's own frontier rows (a local queue carrying their
//         superstep-start distances) relax their out-edges (CSR(G) rows of
//         the shard): an owned destination by atomicMin on its distance, any
//         other into the shard's full-N candidate array; after a barrier each
//         owner takes the min over every shard's candidates for its rows
//         (peer loads) and resets them (peer stores);
//   pull: every owned row takes the min over its in-entries of msg[u] + w,
//         msg being the replicated packed vector of the frontier's
//         distances (INF elsewhere) that the owners published before.
// finish: the improved rows form the next frontier; one u64 all-reduce of
// (improved, their out-edges) per superstep, read by the host.
// ============================================================================
struct DSsspState {
  std::vector<DevBuf<uint32_t>> dist, chg, queue, qd;   // [l]
  std::vector<DevBuf<unsigned long long>> ctr, sum;     // [l]
  std::vector<void*> msg, cand;                         // [l] peer-visible
  std::vector<std::vector<void*>> msg_tab, cand_tab;
  Comm* c = nullptr;
  ~DSsspState() {
    if (!c) return;
    c->unshare(msg_tab);
    c->unshare(cand_tab);
    for (int l = 0; l < c->L; ++l) {
      c->set(l);
      cudaStreamSynchronize(c->st[size_t(l)]);
      c->peer_free(l, msg[size_t(l)]);
      c->peer_free(l, cand[size_t(l)]);
      dist[size_t(l)].reset();
      chg[size_t(l)].reset();
      queue[size_t(l)].reset();
      qd[size_t(l)].reset();
      ctr[size_t(l)].reset();
      sum[size_t(l)].reset();
    }
  }
};

namespace {

constexpr uint32_t kInf = 0xFFFFFFFFu;
constexpr uint64_t kDSsspPullDiv = 6;

__global__ void k_ds_init(uint32_t* dist, uint32_t* chg, uint64_t rows, uint64_t words,
                          uint64_t root_local, int owns_root, uint32_t* queue, uint32_t* qd,
                          unsigned long long* ctr, const uint32_t* outdeg) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < rows || i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (i < rows) dist[i] = owns_root && i == root_local ? 0u : kInf;
    if (i < words) chg[i] = owns_root && i == (root_local >> 5) ? 1u << (root_local & 31u) : 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr[0] = owns_root ? 1 : 0;
    ctr[1] = owns_root ? outdeg[root_local] : 0;
    ctr[2] = 0;
    ctr[3] = owns_root ? 1 : 0;
    if (owns_root) {
      queue[0] = uint32_t(root_local);
      qd[0] = 0;
    }
  }
}

// this shard's rows of the message vector: the new distance of every row
// that improved in the last superstep, INF for the others, into every shard
__global__ void k_ds_publish(const uint32_t* dist, const uint32_t* chg, const uint32_t* pid,
                             uint64_t rows, PeerTab<uint32_t> msg, int P, uint64_t nx) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = pid[r];
    if (p == ~0u) continue;  // no out-edges: never read
    GM_DCHECK(p < nx);
    const uint32_t v = (chg[r >> 5] >> (r & 31u)) & 1u ? dist[r] : kInf;
    for (int q = 0; q < P; ++q) msg.p[q][p] = v;
  }
}

__device__ __forceinline__ void ds_improve(uint32_t* dist, uint32_t* chg, uint64_t r, uint32_t nd) {
  if (nd < dist[r] && atomicMin(&dist[r], nd) > nd) atomicOr(&chg[r >> 5], 1u << (r & 31u));
}

__global__ void __launch_bounds__(256) k_ds_push(const uint32_t* __restrict__ queue,
                                                 const uint32_t* __restrict__ qd,
                                                 const unsigned long long* qn,
                                                 const uint64_t* __restrict__ ptr,
                                                 const uint32_t* __restrict__ idx,
                                                 const uint8_t* __restrict__ w, uint64_t lo,
                                                 uint64_t hi, uint32_t* dist, uint32_t* chg,
                                                 uint32_t* cand, uint64_t n) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t nq = qn[3];
  for (uint64_t i = wp; i < nq; i += nw) {
    const uint32_t r = queue[i], du = qd[i];
    for (uint64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      const uint32_t v = __ldg(&idx[e]);
      GM_DCHECK(v < n);
      const uint32_t nd = du + __ldg(&w[e]);
      if (v >= lo && v < hi)
        ds_improve(dist, chg, v - lo, nd);
      else if (nd < cand[v])
        atomicMin(&cand[v], nd);
    }
  }
}

__global__ void k_ds_claims(PeerTab<uint32_t> cand, int P, uint64_t lo, uint64_t rows,
                            uint32_t* dist, uint32_t* chg) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t best = kInf;
    for (int q = 0; q < P; ++q) {
      uint32_t* p = cand.p[q] + lo + r;
      const uint32_t c = *p;
      if (c != kInf) {
        best = c < best ? c : best;
        *p = kInf;
      }
    }
    if (best != kInf) ds_improve(dist, chg, r, best);
  }
}

__global__ void __launch_bounds__(256) k_ds_pull(const uint64_t* __restrict__ ptr,
                                                 const uint32_t* __restrict__ idx,
                                                 const uint8_t* __restrict__ w, uint64_t rows,
                                                 const uint32_t* __restrict__ msg, uint32_t* dist,
                                                 uint32_t* chg, unsigned long long* ctr,
                                                 uint64_t nx) {
  unsigned long long ex = 0;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t best = kInf;
    const uint64_t e1 = ptr[r + 1];
    for (uint64_t e = ptr[r]; e < e1; ++e) {
      const uint32_t u = __ldg(&idx[e]);
      GM_DCHECK(u < nx);
      const uint32_t m = __ldg(&msg[u]);
      if (m != kInf) {
        const uint32_t nd = m + __ldg(&w[e]);
        best = nd < best ? nd : best;
      }
    }
    ex += e1 - ptr[r];
    if (best != kInf) ds_improve(dist, chg, r, best);
  }
  warp_add_u64(&ctr[2], ex);
}

__global__ void k_ds_finish(const uint32_t* chg, uint64_t words, uint64_t rows, const uint32_t* dist,
                            const uint32_t* outdeg, uint32_t* queue, uint32_t* qd,
                            unsigned long long* ctr) {
  // lanes = 32 consecutive words; one queue reservation per warp (an atomic
  // per word with changes serialised on the counter)
  unsigned long long f = 0, fe = 0;
  const unsigned lane = lane_id();
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~uint64_t(31); w0 < words;
       w0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t wd = w0 + lane;
    uint32_t b = wd < words ? chg[wd] : 0u;
    const unsigned c = __popc(b);
    unsigned incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= unsigned(o)) incl += t;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) continue;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(&ctr[3], (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 31) + (incl - c);
    while (b) {
      const int i = __ffs(b) - 1;
      b &= b - 1;
      const uint64_t r = wd * 32 + uint64_t(i);
      GM_DCHECK(r < rows);
      queue[base] = uint32_t(r);
      qd[base] = dist[r];
      ++base;
      ++f;
      fe += outdeg[r];
    }
  }
  warp_add_u64(&ctr[0], f);
  warp_add_u64(&ctr[1], fe);
}

DSsspState& dsssp_state(DGraph& g) {
  if (g.sssp) return *g.sssp;
  Comm& c = *g.comm;
  g.sssp = std::unique_ptr<DSsspState, void (*)(DSsspState*)>(new DSsspState(),
                                                              [](DSsspState* p) { delete p; });
  DSsspState& st = *g.sssp;
  const int L = c.L;
  for (auto* v : {&st.dist, &st.chg, &st.queue, &st.qd}) v->resize(static_cast<size_t>(L));
  st.ctr.resize(static_cast<size_t>(L));
  st.sum.resize(static_cast<size_t>(L));
  const uint64_t nx = std::max<uint64_t>(g.nonzero_outdeg, 1);
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    const uint64_t rows = g.sh[size_t(l)].hi - g.sh[size_t(l)].lo;
    st.dist[size_t(l)].alloc(rows + 1, s);
    st.chg[size_t(l)].alloc((rows + 31) / 32 + 1, s);
    st.queue[size_t(l)].alloc(rows + 1, s);
    st.qd[size_t(l)].alloc(rows + 1, s);
    st.ctr[size_t(l)].alloc(4, s);
    st.sum[size_t(l)].alloc(4, s);
    st.msg.push_back(c.peer_alloc(l, nx * 4));
    st.cand.push_back(c.peer_alloc(l, g.n * 4 + 4));
    GM_CUDA(cudaMemsetAsync(st.cand.back(), 0xFF, g.n * 4 + 4, s));
    GM_CUDA(cudaStreamSynchronize(s));
  }
  st.c = &c;
  st.msg_tab = c.share(st.msg);
  st.cand_tab = c.share(st.cand);
  return st;
}

}  // namespace

std::vector<gm_iteration_stats> dsssp(DGraph& g, uint64_t root, int64_t max_iters, uint32_t* out,
                                      bool out_on_device) {
  Comm& c = *g.comm;
  if (g.symmetric || g.value_type != GM_VAL_U8)
    fail(GM_EUSAGE, "dgraph sssp: needs a directed graph with u8 weights");
  if (root >= g.n)
    fail(GM_EINPUT, "source vertex " + std::to_string(root + 1) + " (1-based) exceeds vertex count " +
                        std::to_string(g.n));
  DSsspState& st = dsssp_state(g);
  const int L = c.L, P = c.P;
  const uint64_t m = g.m;
  const uint64_t nx = std::max<uint64_t>(g.nonzero_outdeg, 1);
  const uint64_t ro = g.owner(root);
  HostPinned<unsigned long long> h(4);
  std::vector<const uint64_t*> cin;
  std::vector<uint64_t*> cout_;
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    DShard& sh = g.sh[size_t(l)];
    const uint64_t rows = sh.hi - sh.lo, words = (rows + 31) / 32;
    const int owns = uint64_t(c.global(l)) == ro;
    k_ds_init<<<grid_for(std::max(rows, words) + 1, kBlock), kBlock, 0, s>>>(
        st.dist[size_t(l)].get(), st.chg[size_t(l)].get(), rows, words, owns ? root - sh.lo : 0,
        owns, st.queue[size_t(l)].get(), st.qd[size_t(l)].get(), st.ctr[size_t(l)].get(),
        sh.outdeg.get());
    GM_LAUNCH_CHECK();
    cin.push_back(reinterpret_cast<const uint64_t*>(st.ctr[size_t(l)].get()));
    cout_.push_back(reinterpret_cast<uint64_t*>(st.sum[size_t(l)].get()));
  }
  c.allreduce_u64(cin, cout_, 4);
  c.set(0);
  GM_CUDA(cudaMemcpyAsync(h.get(), st.sum[0].get(), 32, cudaMemcpyDeviceToHost, c.st[0]));
  GM_CUDA(cudaStreamSynchronize(c.st[0]));
  uint64_t nf = h[0], ef = h[1];
  StepTimer tm;
  std::vector<gm_iteration_stats> stats;
  for (int64_t it = 1; nf > 0 && it <= max_iters; ++it) {
    const bool pull = ef * kDSsspPullDiv > m;
    c.set(0);
    GM_CUDA(cudaEventRecord(tm.e[2], c.st[0]));
    if (pull) {  // the frontier's distances into every shard's message vector
      for (int l = 0; l < L; ++l) {
        c.set(l);
        cudaStream_t s = c.st[size_t(l)];
        DShard& sh = g.sh[size_t(l)];
        const uint64_t rows = sh.hi - sh.lo;
        launch(rows, s, [&](unsigned gr, unsigned bl) {
          k_ds_publish<<<gr, bl, 0, s>>>(st.dist[size_t(l)].get(), st.chg[size_t(l)].get(),
                                         sh.pid.get(), rows, tab_of<uint32_t>(st.msg_tab[size_t(l)], P),
                                         P, nx);
        });
      }
      c.barrier();
    }
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      const uint64_t rows = sh.hi - sh.lo, words = (rows + 31) / 32;
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[0], s));
      if (words) GM_CUDA(cudaMemsetAsync(st.chg[size_t(l)].get(), 0, words * 4, s));
      GM_CUDA(cudaMemsetAsync(st.ctr[size_t(l)].get(), 0, 24, s));  // keep ctr[3] (queue length)
      if (!pull) {
        k_ds_push<<<148 * 4, 256, 0, s>>>(st.queue[size_t(l)].get(), st.qd[size_t(l)].get(),
                                          st.ctr[size_t(l)].get(), sh.out.ptr.get(), sh.out.idx.get(),
                                          sh.out.val.get(), sh.lo, sh.hi, st.dist[size_t(l)].get(),
                                          st.chg[size_t(l)].get(),
                                          static_cast<uint32_t*>(st.cand[size_t(l)]), g.n);
        GM_LAUNCH_CHECK();
      } else {
        launch(rows, s, [&](unsigned gr, unsigned bl) {
          k_ds_pull<<<gr, bl, 0, s>>>(sh.in.ptr.get(), sh.in.idx.get(), sh.in.val.get(), rows,
                                      static_cast<const uint32_t*>(st.msg[size_t(l)]),
                                      st.dist[size_t(l)].get(), st.chg[size_t(l)].get(),
                                      st.ctr[size_t(l)].get(), nx);
        });
      }
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[1], s));
    }
    if (!pull) {
      c.barrier();
      for (int l = 0; l < L; ++l) {
        c.set(l);
        cudaStream_t s = c.st[size_t(l)];
        DShard& sh = g.sh[size_t(l)];
        const uint64_t rows = sh.hi - sh.lo;
        launch(rows, s, [&](unsigned gr, unsigned bl) {
          k_ds_claims<<<gr, bl, 0, s>>>(tab_of<uint32_t>(st.cand_tab[size_t(l)], P), P, sh.lo, rows,
                                        st.dist[size_t(l)].get(), st.chg[size_t(l)].get());
        });
      }
      c.barrier();  // nobody pushes into a candidate array before its owners reset it
    }
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      const uint64_t rows = sh.hi - sh.lo, words = (rows + 31) / 32;
      GM_CUDA(cudaMemsetAsync(st.ctr[size_t(l)].get() + 3, 0, 8, s));
      launch(words, s, [&](unsigned gr, unsigned bl) {
        k_ds_finish<<<gr, bl, 0, s>>>(st.chg[size_t(l)].get(), words, rows, st.dist[size_t(l)].get(),
                                      sh.outdeg.get(), st.queue[size_t(l)].get(),
                                      st.qd[size_t(l)].get(), st.ctr[size_t(l)].get());
      });
    }
    c.allreduce_u64(cin, cout_, 4);
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(h.get(), st.sum[0].get(), 32, cudaMemcpyDeviceToHost, c.st[0]));
    GM_CUDA(cudaEventRecord(tm.e[3], c.st[0]));
    GM_CUDA(cudaStreamSynchronize(c.st[0]));
    gm_iteration_stats s{};
    s.iteration = it;
    s.active_before = int64_t(nf);
    s.messages_generated = int64_t(nf);
    s.vertices_updated = int64_t(h[0]);
    s.direction = pull ? 0 : 1;
    s.edges_processed = int64_t(pull ? h[2] : ef);
    s.spmv_seconds = tm.ms(0, 1) * 1e-3;
    s.total_seconds = tm.ms(2, 3) * 1e-3;
    s.comm_seconds = std::max(0.0, s.total_seconds - s.spmv_seconds);
    s.bytes_algorithmic = pull ? int64_t(9 * m + 8 * nf + 4 * g.n + 20 * h[0])
                               : int64_t(28 * nf + 5 * ef + 20 * h[0] + g.n / 8);
    stats.push_back(s);
    nf = h[0];
    ef = h[1];
  }
  if (out) {
    uint64_t off = 0;
    for (int l = 0; l < L; ++l) {
      c.set(l);
      const uint64_t rows = g.sh[size_t(l)].hi - g.sh[size_t(l)].lo;
      if (rows)
        GM_CUDA(cudaMemcpyAsync(out + off, st.dist[size_t(l)].get(), rows * 4,
                                out_on_device ? cudaMemcpyDefault : cudaMemcpyDeviceToHost,
                                c.st[size_t(l)]));
      off += rows;
    }
  }
  for (int l = 0; l < L; ++l) {
    c.set(l);
    GM_CUDA(cudaStreamSynchronize(c.st[size_t(l)]));
  }
  return stats;
}

}  // namespace gm

// ============================================================================
// Collaborative filtering over the row shards (CfGdProgram,
// collaborative_filtering.hpp:51-90, driven like collaborative_filtering_gd,
// :134-211).  The bipartite graph is sharded by vertex (users and items
// alike); shard r stores CSR(G^T) rows (an item's raters) and CSR(G) rows (a
// user's items) of its vertices with the u8 ratings.  Every shard holds the
// whole superstep-start factor matrix (n x k fp32, 40 MB for configs[3]);
// a warp per owned vertex folds e*q over both routes (out-route first, the
// BOTH merge of engine.hpp:113-126; lane-strided partials and a fixed xor
// tree: the same result for any P), applies p' = p + gamma*(sum - lambda*p)
// to every vertex (un-messaged ones take the empty sum, :192-193) and stores
// p' into every shard's next factor matrix (peer stores).  Each rating's
// squared error is taken at its user's owner; one f64 all-reduce per
// superstep sums them (the RMSE of the factors the superstep read) and one
// u64 all-reduce the updated-vertex count.
// ============================================================================
namespace gm {

struct DCfState {
  std::vector<void*> f[2];  // [l] peer-visible factor matrices
  std::vector<std::vector<void*>> f_tab[2];
  std::vector<DevBuf<double>> sq, sqs;                 // [l] partial / summed
  std::vector<DevBuf<unsigned long long>> ctr, sum;    // [l] updated
  std::vector<DevBuf<uint32_t>> vbits;
  int64_t k = 0;
  Comm* c = nullptr;
  ~DCfState() {
    if (!c) return;
    for (int b = 0; b < 2; ++b) c->unshare(f_tab[b]);
    for (int l = 0; l < c->L; ++l) {
      c->set(l);
      cudaStreamSynchronize(c->st[size_t(l)]);
      c->peer_free(l, f[0][size_t(l)]);
      c->peer_free(l, f[1][size_t(l)]);
      sq[size_t(l)].reset();
      sqs[size_t(l)].reset();
      ctr[size_t(l)].reset();
      sum[size_t(l)].reset();
      vbits[size_t(l)].reset();
    }
  }
};

namespace {

__global__ void k_row_ratings(const uint64_t* ptr, const uint32_t* idx, uint64_t lo, uint64_t rows,
                              uint64_t seed_r, int row_is_item, uint8_t* out) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = wp; r < rows; r += nw)
    for (uint64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      const uint32_t row = uint32_t(lo + r), col = idx[e];
      out[e] = row_is_item ? rating_of(seed_r, col, row) : rating_of(seed_r, row, col);
    }
}

constexpr int kCfK = 20;

// one route of vertex v: acc += (r - p.q_u) q_u over the row's entries
__device__ __forceinline__ bool dcf_route(const uint64_t* ptr, const uint32_t* idx, const uint8_t* val,
                                          uint64_t r, const float* f, const float (&p)[kCfK],
                                          float (&acc)[kCfK], double& sq) {
  const uint64_t b = ptr[r], e1 = ptr[r + 1];
  for (uint64_t e = b + lane_id(); e < e1; e += 32) {
    const float4* q4 = reinterpret_cast<const float4*>(f + uint64_t(idx[e]) * kCfK);
    float q[kCfK];
#pragma unroll
    for (int i = 0; i < kCfK / 4; ++i) {
      const float4 t = q4[i];
      q[4 * i] = t.x;
      q[4 * i + 1] = t.y;
      q[4 * i + 2] = t.z;
      q[4 * i + 3] = t.w;
    }
    float dot = 0.0f;
#pragma unroll
    for (int i = 0; i < kCfK; ++i) dot += p[i] * q[i];
    const float err = float(val[e]) - dot;
    sq += double(err) * double(err);
#pragma unroll
    for (int i = 0; i < kCfK; ++i) acc[i] += err * q[i];
  }
#pragma unroll
  for (int i = 0; i < kCfK; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  return e1 > b;
}

__global__ void __launch_bounds__(256) k_dcf_step(const uint64_t* in_ptr, const uint32_t* in_idx,
                                                  const uint8_t* in_val, const uint64_t* out_ptr,
                                                  const uint32_t* out_idx, const uint8_t* out_val,
                                                  uint64_t lo, uint64_t rows, const float* f,
                                                  PeerTab<float> fn, int P, float gamma,
                                                  float lambda, uint32_t* vbits,
                                                  unsigned long long* upd, double* sq_out) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  double sq = 0.0;
  unsigned long long u = 0;
  for (uint64_t r = wp; r < rows; r += nw) {
    const uint64_t v = lo + r;
    float p[kCfK], so[kCfK], si[kCfK];
#pragma unroll
    for (int i = 0; i < kCfK; ++i) {
      p[i] = f[v * kCfK + i];
      so[i] = 0.0f;
      si[i] = 0.0f;
    }
    double dummy = 0.0;
    // out-route: v receives along its in-edges (CSR(G^T) row); in-route: along
    // its out-edges (CSR(G) row) -- each rating's error counted once, at the user
    const bool any_o = dcf_route(in_ptr, in_idx, in_val, r, f, p, so, dummy);
    const bool any_i = dcf_route(out_ptr, out_idx, out_val, r, f, p, si, sq);
    bool changed = false;
    float np[kCfK];
#pragma unroll
    for (int i = 0; i < kCfK; ++i) {
      const float s = any_o && any_i ? so[i] + si[i] : (any_o ? so[i] : si[i]);
      np[i] = p[i] + gamma * (s - lambda * p[i]);
      changed |= __float_as_uint(np[i]) != __float_as_uint(p[i]);
    }
    if (lane < kCfK) {
      float mine = np[0];
#pragma unroll
      for (int i = 1; i < kCfK; ++i)
        if (int(lane) == i) mine = np[i];
      for (int q = 0; q < P; ++q) fn.p[q][v * kCfK + lane] = mine;
    }
    if (lane == 0 && changed && (any_o || any_i)) {
      ++u;
      atomicOr(&vbits[r >> 5], 1u << (r & 31u));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0 && sq != 0.0) atomicAdd(sq_out, sq);
  warp_add_u64(upd, u);
}

// squared errors of the factors f over the ratings of the owned users
__global__ void __launch_bounds__(256) k_dcf_sq(const uint64_t* out_ptr, const uint32_t* out_idx,
                                                const uint8_t* out_val, uint64_t lo, uint64_t rows,
                                                const float* f, double* sq_out) {
  const uint64_t wp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  double sq = 0.0;
  for (uint64_t r = wp; r < rows; r += nw) {
    const uint64_t v = lo + r;
    float p[kCfK], acc[kCfK];
#pragma unroll
    for (int i = 0; i < kCfK; ++i) {
      p[i] = f[v * kCfK + i];
      acc[i] = 0.0f;
    }
    dcf_route(out_ptr, out_idx, out_val, r, f, p, acc, sq);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane_id() == 0 && sq != 0.0) atomicAdd(sq_out, sq);
}

DCfState& dcf_state(DGraph& g, int64_t k) {
  if (g.cf && g.cf->k == k) return *g.cf;
  g.cf.reset();
  Comm& c = *g.comm;
  g.cf = std::unique_ptr<DCfState, void (*)(DCfState*)>(new DCfState(), [](DCfState* p) { delete p; });
  DCfState& st = *g.cf;
  st.k = k;
  const int L = c.L;
  st.sq.resize(static_cast<size_t>(L));
  st.sqs.resize(static_cast<size_t>(L));
  st.ctr.resize(static_cast<size_t>(L));
  st.sum.resize(static_cast<size_t>(L));
  st.vbits.resize(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) {
    c.set(l);
    cudaStream_t s = c.st[size_t(l)];
    const uint64_t rows = g.sh[size_t(l)].hi - g.sh[size_t(l)].lo;
    for (int b = 0; b < 2; ++b) st.f[b].push_back(c.peer_alloc(l, g.n * uint64_t(k) * 4 + 16));
    st.sq[size_t(l)].alloc(1, s);
    st.sqs[size_t(l)].alloc(1, s);
    st.ctr[size_t(l)].alloc(1, s);
    st.sum[size_t(l)].alloc(1, s);
    st.vbits[size_t(l)].alloc((rows + 31) / 32 + 1, s);
  }
  st.c = &c;
  for (int b = 0; b < 2; ++b) st.f_tab[b] = c.share(st.f[b]);
  return st;
}

}  // namespace

DGraph* dgraph_generate_bipartite(Comm* c, uint32_t users, uint32_t items, double c_num,
                                  uint32_t cap, uint64_t seed) {
  if (users == 0 || items == 0) fail(GM_EUSAGE, "bipartite: need users and items");
  const uint64_t n = uint64_t(users) + items;
  std::unique_ptr<DGraph> g(new_dgraph(c, n, GM_PREPROCESS));
  g->bipartite = true;
  const unsigned nb = bits_for(n);
  std::vector<DevBuf<uint64_t>> keys(static_cast<size_t>(c->L));
  std::vector<uint64_t> m(static_cast<size_t>(c->L));
  for (int l = 0; l < c->L; ++l) {
    c->set(l);
    cudaStream_t s = c->st[size_t(l)];
    const uint64_t cnt = bipartite_range(users, items, c_num, cap, seed, uint64_t(c->global(l)),
                                         uint64_t(c->P), nullptr, nullptr, nullptr, s);
    DevBuf<uint32_t> s32(cnt + 1, s), d32(cnt + 1, s);
    bipartite_range(users, items, c_num, cap, seed, uint64_t(c->global(l)), uint64_t(c->P), s32.get(),
                    d32.get(), nullptr, s);
    keys[size_t(l)].alloc(cnt + 1, s);
    DevBuf<unsigned long long> k(1, s);
    k.zero(s);
    launch(cnt, s, [&](unsigned gr, unsigned bl) {
      k_edge_keys<<<gr, bl, 0, s>>>(s32.get(), d32.get(), cnt, nb, 0, keys[size_t(l)].get(), k.get());
    });
    m[size_t(l)] = dread_u64(k.get(), s);
  }
  route_and_build(*g, keys, m, nb, /*forward=*/false, /*check_dups=*/false);
  build_forward(*g, nb);
  g->value_type = GM_VAL_U8;
  const uint64_t seed_r = mix64(seed ^ 0x0DA7A5EEDull);
  for (int l = 0; l < c->L; ++l) {
    c->set(l);
    cudaStream_t s = c->st[size_t(l)];
    DShard& sh = g->sh[size_t(l)];
    for (int f = 0; f < 2; ++f) {
      Csr& a = f ? sh.out : sh.in;
      a.val.alloc(a.nnz + 1, s);
      launch(a.n * 32, s, [&](unsigned gr, unsigned bl) {
        k_row_ratings<<<gr, bl, 0, s>>>(a.ptr.get(), a.idx.get(), sh.lo, a.n, seed_r, f == 0,
                                        a.val.get());
      });
    }
  }
  std::vector<uint64_t> nnz;
  for (auto& s : g->sh) nnz.push_back(s.in.nnz);
  g->m = c->sum_host(nnz);
  for (int l = 0; l < c->L; ++l) {
    c->set(l);
    GM_CUDA(cudaStreamSynchronize(c->st[size_t(l)]));
  }
  return g.release();
}

std::vector<gm_iteration_stats> dcf(DGraph& g, int64_t k, float gamma, float lambda,
                                    int64_t iters, const float* init, float* out,
                                    double* rmse_trace) {
  Comm& c = *g.comm;
  if (!g.bipartite) fail(GM_EUSAGE, "dgraph cf: needs a bipartite rating graph");
  if (k != kCfK) fail(GM_EUSAGE, "dgraph cf: k = 20 (the BASELINE latent dimension) only");
  if (!(gamma > 0.0f)) fail(GM_EINPUT, "cf: gamma must be positive");
  if (!(lambda >= 0.0f)) fail(GM_EINPUT, "cf: lambda must be non-negative");
  if (!init) fail(GM_EUSAGE, "dgraph cf: init factors are required");
  DCfState& st = dcf_state(g, k);
  const int L = c.L, P = c.P;
  const uint64_t n = g.n, m = g.m;
  for (int l = 0; l < L; ++l) {  // every shard starts from the full init matrix
    c.set(l);
    GM_CUDA(cudaMemcpyAsync(st.f[0][size_t(l)], init, n * uint64_t(k) * 4, cudaMemcpyHostToDevice,
                            c.st[size_t(l)]));
  }
  std::vector<const double*> qin;
  std::vector<double*> qout;
  std::vector<const uint64_t*> cin;
  std::vector<uint64_t*> cout_;
  for (int l = 0; l < L; ++l) {
    qin.push_back(st.sq[size_t(l)].get());
    qout.push_back(st.sqs[size_t(l)].get());
    cin.push_back(reinterpret_cast<const uint64_t*>(st.ctr[size_t(l)].get()));
    cout_.push_back(reinterpret_cast<uint64_t*>(st.sum[size_t(l)].get()));
  }
  std::vector<gm_iteration_stats> stats;
  std::vector<std::unique_ptr<StepTimer>> tms;
  std::vector<unsigned long long> upd(size_t(std::max<int64_t>(iters, 0)));
  auto rmse_of = [&](int buf) {  // RMSE of factor matrix `buf` over all ratings
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      st.sq[size_t(l)].zero(s);
      launch((sh.hi - sh.lo) * 32, s, [&](unsigned gr, unsigned bl) {
        k_dcf_sq<<<gr, bl, 0, s>>>(sh.out.ptr.get(), sh.out.idx.get(), sh.out.val.get(), sh.lo,
                                   sh.hi - sh.lo, static_cast<const float*>(st.f[buf][size_t(l)]),
                                   st.sq[size_t(l)].get());
      });
    }
    c.allreduce_f64(qin, qout, 1);
    double h = 0.0;
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(&h, st.sqs[0].get(), 8, cudaMemcpyDeviceToHost, c.st[0]));
    GM_CUDA(cudaStreamSynchronize(c.st[0]));
    return m ? std::sqrt(h / double(m)) : 0.0;
  };
  int cur = 0;
  for (int64_t it = 1; it <= iters; ++it) {
    tms.emplace_back(new StepTimer());
    StepTimer& tm = *tms.back();
    for (int l = 0; l < L; ++l) {
      c.set(l);
      cudaStream_t s = c.st[size_t(l)];
      DShard& sh = g.sh[size_t(l)];
      const uint64_t rows = sh.hi - sh.lo;
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[0], s));
      st.sq[size_t(l)].zero(s);
      st.ctr[size_t(l)].zero(s);
      GM_CUDA(cudaMemsetAsync(st.vbits[size_t(l)].get(), 0, ((rows + 31) / 32 + 1) * 4, s));
      launch(rows * 32, s, [&](unsigned gr, unsigned bl) {
        k_dcf_step<<<gr, bl, 0, s>>>(sh.in.ptr.get(), sh.in.idx.get(), sh.in.val.get(), sh.out.ptr.get(),
                                     sh.out.idx.get(), sh.out.val.get(), sh.lo, rows,
                                     static_cast<const float*>(st.f[cur][size_t(l)]),
                                     tab_of<float>(st.f_tab[cur ^ 1][size_t(l)], P), P, gamma, lambda,
                                     st.vbits[size_t(l)].get(), st.ctr[size_t(l)].get(),
                                     st.sq[size_t(l)].get());
      });
      if (l == 0) GM_CUDA(cudaEventRecord(tm.e[1], s));
    }
    c.allreduce_u64(cin, cout_, 1);  // also the barrier: every shard's factors have landed
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(&upd[size_t(it - 1)], st.sum[0].get(), 8, cudaMemcpyDeviceToHost, c.st[0]));
    GM_CUDA(cudaEventRecord(tm.e[2], c.st[0]));
    cur ^= 1;
    if (rmse_trace) rmse_trace[it - 1] = rmse_of(cur);
  }
  if (out) {
    c.set(0);
    GM_CUDA(cudaMemcpyAsync(out, st.f[cur][0], n * uint64_t(k) * 4, cudaMemcpyDeviceToHost, c.st[0]));
  }
  for (int l = 0; l < L; ++l) {
    c.set(l);
    GM_CUDA(cudaStreamSynchronize(c.st[size_t(l)]));
  }
  for (int64_t it = 1; it <= iters; ++it) {
    gm_iteration_stats s{};
    s.iteration = it;
    s.active_before = int64_t(n);
    s.messages_generated = int64_t(n);
    s.vertices_updated = int64_t(upd[size_t(it - 1)]);
    s.spmv_seconds = tms[size_t(it - 1)]->ms(0, 1) * 1e-3;
    s.total_seconds = tms[size_t(it - 1)]->ms(0, 2) * 1e-3;
    s.comm_seconds = std::max(0.0, s.total_seconds - s.spmv_seconds);
    s.edges_processed = int64_t(2 * m);
    s.bytes_algorithmic = int64_t(2 * 5 * m + 2 * 8 * (n + 2) + 3 * 4 * uint64_t(k) * n);
    stats.push_back(s);
  }
  return stats;
}

}  // namespace gm
