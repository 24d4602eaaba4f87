// dist.cuh -- multi-GPU layer: communicator + row-sharded graph.
//
// The reference runs every row partition of G^T from one run_graph_program
// call (include/semigraph/engine.hpp:193-213, partitions dispatched by
// pool_.run at :230, boundaries by detail::balanced_row_boundaries,
// dcsc.hpp:77-105).  Here a partition is a shard on a GPU:
//
//   Comm    P shards ("ranks").  One process drives L of them:
//           * local: one process, L = P shards on the devices it lists
//             (repeats allowed: virtual shards on one GPU), the exchange is
//             peer memory (NVLink loads/stores between the devices);
//           * nccl:  one process per GPU (L = 1), an NCCL communicator
//             (libnccl loaded at run time) for all-reduce / all-to-all and
//             CUDA IPC mappings of the peers' buffers for the peer stores.
//   DGraph  shard r owns the contiguous caller-id rows [lo_r, hi_r) (32-aligned,
//           balanced by stored entries like dcsc.hpp:81-105) and stores only
//           those rows: CSR(G^T) rows (in-edges) and, for programs that push
//           along out-edges, CSR(G) rows (out-edges).  Columns are global
//           caller ids, ascending -- the reference's per-row fold order
//           (engine.hpp:59-66) -- so results do not depend on P.
//
// Every collective is issued by the host thread once per process and runs on
// the shards' streams (stream-ordered: no host round trip inside it).
#pragma once

#include <memory>
#include <vector>

#include "graph.cuh"

namespace gm {

struct Comm {
  int P = 1;      // shards in the job
  int L = 1;      // shards this process drives
  int first = 0;  // global index of local shard 0
  bool use_nccl = false;
  std::vector<int> dev;           // [L] CUDA device of each local shard
  std::vector<cudaStream_t> st;   // [L] its stream
  void* nccl = nullptr;           // ncclComm_t when use_nccl
  std::vector<cudaEvent_t> ev;    // [L] scratch events for local barriers
  DevBuf<uint64_t> one;           // NCCL barrier word (L == 1)

  ~Comm();
  // Every shard's stream waits for the work issued on every other shard's
  // stream so far (peer stores issued before are visible after).
  void barrier();
  // out[l][i] = sum over shards q of in[q][i], count u64 words (in != out).
  void allreduce_u64(const std::vector<const uint64_t*>& in, const std::vector<uint64_t*>& out,
                     size_t count);
  // The same for doubles (local: summed in shard order).
  void allreduce_f64(const std::vector<const double*>& in, const std::vector<double*>& out,
                     size_t count);
  // dst[l] = concatenation over shards q (rank order) of src[q], bytes each.
  void allgather(const std::vector<const void*>& src, const std::vector<void*>& dst, size_t bytes);
  // All-to-all of byte runs: shard q sends send_counts[q][r] bytes starting at
  // send[q] + send_offs[q][r] to shard r, which receives them at recv[r] +
  // recv_offs[r][q].  Counts/offsets are host-side, known to the caller (for
  // nccl after a count exchange, see exchange_counts).
  void alltoallv(const std::vector<const uint8_t*>& send,
                 const std::vector<std::vector<uint64_t>>& send_offs,
                 const std::vector<std::vector<uint64_t>>& send_counts,
                 const std::vector<uint8_t*>& recv,
                 const std::vector<std::vector<uint64_t>>& recv_offs);
  // mine[l][r] (host, per local shard l, per destination r) -> theirs[l][q] =
  // what shard q sent to local shard l.  A small host-visible all-to-all.
  std::vector<std::vector<uint64_t>> exchange_counts(const std::vector<std::vector<uint64_t>>& mine);
  // Sum of a host value per local shard over all shards (host result,
  // synchronising).
  uint64_t sum_host(const std::vector<uint64_t>& mine);
  // Device buffers visible to every shard: local[l] (from peer_alloc) ->
  // table[l][q] = shard q's buffer as addressable from local shard l's device.
  std::vector<std::vector<void*>> share(const std::vector<void*>& local);
  void unshare(std::vector<std::vector<void*>>& table);
  void* peer_alloc(int l, size_t bytes);  // cudaMalloc on shard l's device (IPC-able)
  void peer_free(int l, void* p);
  void set(int l) const;                  // cudaSetDevice(dev[l])
  int global(int l) const { return first + l; }
  int refs = 1;  // the caller's handle + one per live DGraph
};
// gm_comm_destroy drops the caller's reference; graphs built on the
// communicator hold theirs until they are destroyed.
void comm_retain(Comm* c);
void comm_release(Comm* c);

Comm* comm_create_local(int ndev, const int* devices);
Comm* comm_create_nccl(int nranks, int rank, int device, const void* id128);
void comm_nccl_unique_id(void* id128);

// ---- row-sharded graph -------------------------------------------------------
struct DShard {
  int l = 0;             // local index
  uint64_t lo = 0, hi = 0;
  Csr in;                // rows [lo, hi) of CSR(G^T), local row index
  Csr out;               // rows [lo, hi) of CSR(G) (directed push / BOTH); aliases in if symmetric
  bool out_alias = false;
  DevBuf<uint32_t> outdeg;  // out-degree of the owned rows
  DevBuf<uint32_t> pid;     // directed: packed id of each owned row (~0u: no out-edges)
  const Csr& fwd() const { return out_alias ? in : out; }
};

struct DBfsState;
struct DPrState;
struct DSsspState;
struct DCfState;

struct DGraph {
  Comm* comm = nullptr;
  uint64_t n = 0, m = 0;
  uint32_t flags = 0;
  bool symmetric = false;
  bool bipartite = false;  // users -> items rating graph (CF): columns stay caller ids
  int value_type = GM_VAL_NONE;
  std::vector<uint64_t> bounds;  // P + 1 row boundaries
  std::vector<DShard> sh;        // L local shards
  uint64_t nonzero_outdeg = 0;   // global count of vertices with out-edges

  std::unique_ptr<DBfsState, void (*)(DBfsState*)> bfs{nullptr, nullptr};
  std::unique_ptr<DPrState, void (*)(DPrState*)> pr{nullptr, nullptr};
  std::unique_ptr<DSsspState, void (*)(DSsspState*)> sssp{nullptr, nullptr};
  std::unique_ptr<DCfState, void (*)(DCfState*)> cf{nullptr, nullptr};

  ~DGraph();
  uint64_t owner(uint64_t v) const;  // shard owning caller id v
  uint64_t device_bytes(int l) const;
};

DGraph* dgraph_generate_rmat(Comm* c, uint32_t scale, uint32_t ef, double a, double b, double cc,
                             uint64_t seed, uint32_t flags, int weights);
DGraph* dgraph_generate_bipartite(Comm* c, uint32_t users, uint32_t items, double c_num,
                                  uint32_t cap, uint64_t seed);
DGraph* dgraph_create(Comm* c, const gm_edge_list& local_edges, uint64_t n, uint32_t flags,
                      int storage);

uint64_t dpick_source(DGraph& g, uint64_t seed);
void ddegrees(DGraph& g, int local_shard, int kind, uint32_t* out_host);

// Drivers: the whole superstep loop in the library (counters stay on the
// devices; one host read per superstep at most).  Outputs: the owned rows of
// every local shard, concatenated in shard order (the full caller-order
// vector for a local comm).
std::vector<gm_iteration_stats> dbfs(DGraph& g, uint64_t root, int64_t max_iters, int32_t* out,
                                     bool out_on_device);
std::vector<gm_iteration_stats> dpagerank(DGraph& g, double damping, int64_t iters, float* out,
                                          bool out_on_device);
std::vector<gm_iteration_stats> dsssp(DGraph& g, uint64_t root, int64_t max_iters, uint32_t* out,
                                      bool out_on_device);
std::vector<gm_iteration_stats> dcf(DGraph& g, int64_t k, float gamma, float lambda,
                                    int64_t iters, const float* init, float* out,
                                    double* rmse_trace);

}  // namespace gm
