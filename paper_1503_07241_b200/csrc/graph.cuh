// graph.cuh -- device-resident graph: CSR(G^T) (+ lazily CSR(G)) over internal ids.
//
// Replaces semigraph::Graph (include/semigraph/dcsc.hpp:183-238).  The reference
// keeps G^T as nnz-balanced DCSC row partitions (dcsc.hpp:43-65); here the whole
// transpose is one CSR with int64 offsets and int32 column ids (4 B/entry instead
// of the reference's 16 B), rows = destination, entries = sources ascending.
// Optional relabeling (GM_RELABEL) orders internal ids by out-degree, descending,
// so hot sources are contiguous (gather locality) -- results are always mapped
// back to caller ids.
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace gm {

struct Csr {
  uint64_t n = 0, nnz = 0;
  DevBuf<uint64_t> ptr;  // n + 1
  DevBuf<uint32_t> idx;  // nnz
  DevBuf<uint8_t> val;   // nnz * value_size(value_type)
};

// CUDA-event timing of a handle's dominant kernel (bench.py's roofline:
// algorithmic bytes per launch / average launch duration).  Off by default;
// gm_kernel_timer_start turns it on, the kernels' host drivers bracket their
// main launch with begin()/end(), gm_kernel_timer_stop sums the durations.
struct KernelTimer {
  bool on = false;
  const char* name = "";
  std::vector<cudaEvent_t> ev;  // begin/end pairs, reused across windows
  size_t used = 0;
  void begin(cudaStream_t s, const char* nm) {
    if (!on) return;
    name = nm;
    if (ev.size() < used + 2) {
      for (int i = 0; i < 2; ++i) {
        cudaEvent_t e;
        GM_CUDA(cudaEventCreate(&e));
        ev.push_back(e);
      }
    }
    GM_CUDA(cudaEventRecord(ev[used], s));
  }
  void end(cudaStream_t s) {
    if (!on) return;
    GM_CUDA(cudaEventRecord(ev[used + 1], s));
    used += 2;
  }
  ~KernelTimer() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

struct PrCache;    // pagerank.cu
struct PrHubCache; // pagerank_hub.cu
struct TravCache;  // traversal.cu
struct CfCache;    // cf.cu
struct BfsShardCache;  // bfs_shard.cu
struct SsspShardCache;  // sssp_shard.cu

struct Graph {
  uint64_t n = 0, m = 0;
  uint32_t flags = 0;
  uint32_t shards = 1;  // GM_SHARDS(P): row blocks of n / shards internal ids
  int value_type = GM_VAL_NONE;
  int device = 0;
  bool symmetric = false;
  bool relabeled = false;
  unsigned nb = 1;  // bits per vertex id
  cudaStream_t stream = nullptr;

  DevBuf<uint32_t> perm;   // caller id -> internal id (empty when identity)
  DevBuf<uint32_t> iperm;  // internal id -> caller id
  DevBuf<uint32_t> outdeg; // internal order
  DevBuf<uint32_t> indeg;  // internal order
  uint64_t nonzero_outdeg = 0;

  Csr in;    // CSR(G^T): row k lists sources j of edges j -> k
  Csr out;   // CSR(G):   row j lists destinations k of edges j -> k
  bool out_built = false;
  bool out_alias = false;  // symmetric and value-less: CSR(G) == CSR(G^T)

  KernelTimer ktimer;

  // GM_OUT_HOST_ASYNC: a host copy stream fed from two device staging
  // buffers; the compute stream waits for a buffer's previous copy before
  // writing it again (stage()), the copy stream waits for the write (issue()).
  struct HostAsync {
    cudaStream_t cs = nullptr;
    cudaEvent_t ready[2]{}, freed[2]{};
    DevBuf<uint8_t> buf[2];
    bool used[2]{};
    int i = 0;
    void* stage(cudaStream_t s, size_t bytes) {
      if (!cs) {
        GM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
          GM_CUDA(cudaEventCreateWithFlags(&ready[b], cudaEventDisableTiming));
          GM_CUDA(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
        }
      }
      if (buf[i].size() < bytes) {
        if (used[i]) GM_CUDA(cudaEventSynchronize(freed[i]));
        buf[i].alloc(bytes, s);
        used[i] = false;
      }
      if (used[i]) GM_CUDA(cudaStreamWaitEvent(s, freed[i], 0));
      return buf[i].get();
    }
    void issue(cudaStream_t s, void* host, size_t bytes) {
      GM_CUDA(cudaEventRecord(ready[i], s));
      GM_CUDA(cudaStreamWaitEvent(cs, ready[i], 0));
      GM_CUDA(cudaMemcpyAsync(host, buf[i].get(), bytes, cudaMemcpyDeviceToHost, cs));
      GM_CUDA(cudaEventRecord(freed[i], cs));
      used[i] = true;
      i ^= 1;
    }
    void sync() {
      if (cs) GM_CUDA(cudaStreamSynchronize(cs));
    }
    ~HostAsync() {
      if (!cs) return;
      cudaStreamSynchronize(cs);
      for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(ready[b]);
        cudaEventDestroy(freed[b]);
      }
      cudaStreamDestroy(cs);
    }
  } host_async;

  std::unique_ptr<PrCache, void (*)(PrCache*)> pr{nullptr, nullptr};
  std::unique_ptr<PrHubCache, void (*)(PrHubCache*)> prhub{nullptr, nullptr};
  std::unique_ptr<TravCache, void (*)(TravCache*)> trav{nullptr, nullptr};
  std::unique_ptr<CfCache, void (*)(CfCache*)> cf{nullptr, nullptr};
  std::unique_ptr<CfCache, void (*)(CfCache*)> cf_shard{nullptr, nullptr};
  std::unique_ptr<BfsShardCache, void (*)(BfsShardCache*)> bfs_shard{nullptr, nullptr};
  std::unique_ptr<SsspShardCache, void (*)(SsspShardCache*)> sssp_shard{nullptr, nullptr};

  const Csr& fwd() const { return out_alias ? in : out; }
  uint64_t device_bytes() const;
};

// ingest.cu
Graph* graph_create(const gm_edge_list& e, uint64_t n, uint32_t flags, int storage);
Graph* graph_generate_rmat(uint32_t scale, uint32_t ef, double a, double b, double c,
                           uint64_t seed, int permute, uint32_t flags, int weights);
Graph* graph_generate_bipartite(uint32_t users, uint32_t items, double c_num, uint32_t cap,
                                uint64_t seed, uint32_t flags);
void graph_destroy(Graph* g);
void ensure_forward(Graph& g);
void export_edges(Graph& g, uint32_t* src, uint32_t* dst, void* values);
void degree_vector(Graph& g, int kind, uint64_t* out);
uint64_t pick_source(Graph& g, uint64_t seed);

// Gather/scatter between caller order and internal order (elem_bytes wide).
void to_internal(Graph& g, const void* ext_dev, void* int_dev, size_t elem_bytes);
void to_external(Graph& g, const void* int_dev, void* ext_dev, size_t elem_bytes);

}  // namespace gm
