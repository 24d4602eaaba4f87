// comm.cu -- the communicator behind the sharded graph (dist.cuh).
//
// Local mode: one process, P shards on the listed devices; collectives are
// peer-memory kernels and copies ordered by cross-stream event waits.  NCCL
// mode: one process per GPU; libnccl is loaded at run time (the process's
// already-loaded copy, e.g. torch's, else the system one) and every
// collective is stream-ordered on the shard's stream.  Failures of NCCL calls
// are GM_ENCCL (include/graphmat_b200.h).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "dist.cuh"

namespace gm {
namespace {

// ---- libnccl, resolved at run time ------------------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // The process's own copy first (e.g. torch's, so both share one NCCL),
    // then GM_NCCL_LIB, then the system library.  RTLD_LOCAL: the symbols
    // must not shadow another NCCL a later library binds to.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
      if (const char* p = getenv("GM_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = "libnccl.so.2 not found (set GM_NCCL_LIB)";
      return;
    }
#define GM_NCCL_SYM(f)                                                          \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f));                \
  if (!api.f) {                                                                 \
    err = "libnccl.so.2 lacks nccl" #f;                                         \
    return;                                                                     \
  }
    GM_NCCL_SYM(GetUniqueId)
    GM_NCCL_SYM(CommInitRank)
    GM_NCCL_SYM(CommDestroy)
    GM_NCCL_SYM(AllReduce)
    GM_NCCL_SYM(AllGather)
    GM_NCCL_SYM(Send)
    GM_NCCL_SYM(Recv)
    GM_NCCL_SYM(GroupStart)
    GM_NCCL_SYM(GroupEnd)
    GM_NCCL_SYM(GetErrorString)
#undef GM_NCCL_SYM
  });
  if (!err.empty()) fail(GM_ENCCL, err);
  return api;
}

#define GM_NCCL(call)                                                                     \
  do {                                                                                    \
    const ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess)                                                                \
      ::gm::fail(GM_ENCCL, std::string(#call) + ": " + nccl_api().GetErrorString(r_));    \
  } while (0)

constexpr int kMaxShards = 64;
struct PtrTab {
  const uint64_t* p[kMaxShards];
};

__global__ void k_sum_peers(PtrTab in, int P, size_t count, uint64_t* out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x) {
    uint64_t s = 0;
    for (int q = 0; q < P; ++q) s += in.p[q][i];  // fixed shard order
    out[i] = s;
  }
}

struct PtrTabD {
  const double* p[kMaxShards];
};

__global__ void k_sum_peers_f64(PtrTabD in, int P, size_t count, double* out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += in.p[q][i];  // fixed shard order
    out[i] = s;
  }
}

}  // namespace

void Comm::set(int l) const { GM_CUDA(cudaSetDevice(dev[size_t(l)])); }

void comm_retain(Comm* c) { ++c->refs; }

void comm_release(Comm* c) {
  if (c && --c->refs == 0) delete c;
}

Comm::~Comm() {
  for (int l = 0; l < L; ++l) {
    cudaSetDevice(dev[size_t(l)]);
    cudaStreamSynchronize(st[size_t(l)]);
  }
  one.reset();
  if (use_nccl && nccl) nccl_api().CommDestroy(static_cast<ncclComm_t>(nccl));
  for (int l = 0; l < L; ++l) {
    cudaSetDevice(dev[size_t(l)]);
    if (size_t(l) < ev.size()) cudaEventDestroy(ev[size_t(l)]);
    cudaStreamDestroy(st[size_t(l)]);
  }
}

void Comm::barrier() {
  if (use_nccl) {
    set(0);
    GM_NCCL(nccl_api().AllReduce(one.get(), one.get(), 1, ncclUint64, ncclSum,
                                 static_cast<ncclComm_t>(nccl), st[0]));
    return;
  }
  if (L == 1) return;
  for (int l = 0; l < L; ++l) {
    set(l);
    GM_CUDA(cudaEventRecord(ev[size_t(l)], st[size_t(l)]));
  }
  for (int l = 0; l < L; ++l) {
    set(l);
    for (int q = 0; q < L; ++q)
      if (q != l) GM_CUDA(cudaStreamWaitEvent(st[size_t(l)], ev[size_t(q)], 0));
  }
}

void Comm::allreduce_u64(const std::vector<const uint64_t*>& in, const std::vector<uint64_t*>& out,
                         size_t count) {
  if (!count) return;
  if (use_nccl) {
    set(0);
    GM_NCCL(nccl_api().AllReduce(in[0], out[0], count, ncclUint64, ncclSum,
                                 static_cast<ncclComm_t>(nccl), st[0]));
    return;
  }
  barrier();
  PtrTab t{};
  for (int q = 0; q < P; ++q) t.p[q] = in[size_t(q)];
  for (int l = 0; l < L; ++l) {
    set(l);
    k_sum_peers<<<grid_for(count, 256, 148), 256, 0, st[size_t(l)]>>>(t, P, count, out[size_t(l)]);
    GM_LAUNCH_CHECK();
  }
  barrier();  // nobody rewrites an input another shard is still summing
}

void Comm::allreduce_f64(const std::vector<const double*>& in, const std::vector<double*>& out,
                         size_t count) {
  if (!count) return;
  if (use_nccl) {
    set(0);
    GM_NCCL(nccl_api().AllReduce(in[0], out[0], count, ncclFloat64, ncclSum,
                                 static_cast<ncclComm_t>(nccl), st[0]));
    return;
  }
  barrier();
  PtrTabD t{};
  for (int q = 0; q < P; ++q) t.p[q] = in[size_t(q)];
  for (int l = 0; l < L; ++l) {
    set(l);
    k_sum_peers_f64<<<grid_for(count, 256, 148), 256, 0, st[size_t(l)]>>>(t, P, count,
                                                                          out[size_t(l)]);
    GM_LAUNCH_CHECK();
  }
  barrier();
}

void Comm::allgather(const std::vector<const void*>& src, const std::vector<void*>& dst,
                     size_t bytes) {
  if (!bytes) return;
  if (use_nccl) {
    set(0);
    GM_NCCL(nccl_api().AllGather(src[0], dst[0], bytes, ncclUint8, static_cast<ncclComm_t>(nccl),
                                 st[0]));
    return;
  }
  barrier();
  for (int l = 0; l < L; ++l) {
    set(l);
    for (int q = 0; q < P; ++q)
      GM_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(dst[size_t(l)]) + size_t(q) * bytes,
                              src[size_t(q)], bytes, cudaMemcpyDefault, st[size_t(l)]));
  }
  barrier();
}

void Comm::alltoallv(const std::vector<const uint8_t*>& send,
                     const std::vector<std::vector<uint64_t>>& send_offs,
                     const std::vector<std::vector<uint64_t>>& send_counts,
                     const std::vector<uint8_t*>& recv,
                     const std::vector<std::vector<uint64_t>>& recv_offs) {
  if (use_nccl) {
    // recv counts: what every shard sends to this one
    std::vector<std::vector<uint64_t>> mine{send_counts[0]};
    const auto theirs = exchange_counts(mine);
    const NcclApi& A = nccl_api();
    const int me = first;
    set(0);
    GM_NCCL(A.GroupStart());
    for (int r = 0; r < P; ++r) {
      if (r == me) continue;
      if (send_counts[0][size_t(r)])
        GM_NCCL(A.Send(send[0] + send_offs[0][size_t(r)], send_counts[0][size_t(r)], ncclUint8, r,
                       static_cast<ncclComm_t>(nccl), st[0]));
      if (theirs[0][size_t(r)])
        GM_NCCL(A.Recv(recv[0] + recv_offs[0][size_t(r)], theirs[0][size_t(r)], ncclUint8, r,
                       static_cast<ncclComm_t>(nccl), st[0]));
    }
    GM_NCCL(A.GroupEnd());
    if (send_counts[0][size_t(me)])
      GM_CUDA(cudaMemcpyAsync(recv[0] + recv_offs[0][size_t(me)], send[0] + send_offs[0][size_t(me)],
                              send_counts[0][size_t(me)], cudaMemcpyDeviceToDevice, st[0]));
    return;
  }
  barrier();
  for (int r = 0; r < L; ++r) {
    set(r);
    for (int q = 0; q < P; ++q) {
      const uint64_t c = send_counts[size_t(q)][size_t(r)];
      if (c)
        GM_CUDA(cudaMemcpyAsync(recv[size_t(r)] + recv_offs[size_t(r)][size_t(q)],
                                send[size_t(q)] + send_offs[size_t(q)][size_t(r)], c,
                                cudaMemcpyDefault, st[size_t(r)]));
    }
  }
  barrier();
}

std::vector<std::vector<uint64_t>> Comm::exchange_counts(
    const std::vector<std::vector<uint64_t>>& mine) {
  std::vector<std::vector<uint64_t>> theirs(static_cast<size_t>(L), std::vector<uint64_t>(static_cast<size_t>(P)));
  if (!use_nccl) {
    for (int l = 0; l < L; ++l)
      for (int q = 0; q < P; ++q) theirs[size_t(l)][size_t(q)] = mine[size_t(q)][size_t(l)];
    return theirs;
  }
  set(0);
  DevBuf<uint64_t> a(size_t(P), st[0]), all(size_t(P) * P, st[0]);
  GM_CUDA(cudaMemcpyAsync(a.get(), mine[0].data(), size_t(P) * 8, cudaMemcpyHostToDevice, st[0]));
  GM_NCCL(nccl_api().AllGather(a.get(), all.get(), size_t(P), ncclUint64,
                               static_cast<ncclComm_t>(nccl), st[0]));
  std::vector<uint64_t> h(size_t(P) * P);
  GM_CUDA(cudaMemcpyAsync(h.data(), all.get(), h.size() * 8, cudaMemcpyDeviceToHost, st[0]));
  GM_CUDA(cudaStreamSynchronize(st[0]));
  for (int q = 0; q < P; ++q) theirs[0][size_t(q)] = h[size_t(q) * P + size_t(first)];
  return theirs;
}

uint64_t Comm::sum_host(const std::vector<uint64_t>& mine) {
  uint64_t s = 0;
  for (uint64_t v : mine) s += v;
  if (!use_nccl) return s;
  set(0);
  DevBuf<uint64_t> b(1, st[0]);
  GM_CUDA(cudaMemcpyAsync(b.get(), &s, 8, cudaMemcpyHostToDevice, st[0]));
  GM_NCCL(nccl_api().AllReduce(b.get(), b.get(), 1, ncclUint64, ncclSum,
                               static_cast<ncclComm_t>(nccl), st[0]));
  GM_CUDA(cudaMemcpyAsync(&s, b.get(), 8, cudaMemcpyDeviceToHost, st[0]));
  GM_CUDA(cudaStreamSynchronize(st[0]));
  return s;
}

void* Comm::peer_alloc(int l, size_t bytes) {
  set(l);
  void* p = nullptr;
  GM_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
  return p;
}

void Comm::peer_free(int l, void* p) {
  if (!p) return;
  set(l);
  cudaFree(p);
}

std::vector<std::vector<void*>> Comm::share(const std::vector<void*>& local) {
  std::vector<std::vector<void*>> t(static_cast<size_t>(L), std::vector<void*>(static_cast<size_t>(P), nullptr));
  if (!use_nccl) {
    for (int l = 0; l < L; ++l)
      for (int q = 0; q < P; ++q) t[size_t(l)][size_t(q)] = local[size_t(q)];
    return t;
  }
  set(0);
  cudaIpcMemHandle_t h;
  GM_CUDA(cudaIpcGetMemHandle(&h, local[0]));
  DevBuf<uint8_t> a(sizeof(h), st[0]), all(sizeof(h) * size_t(P), st[0]);
  GM_CUDA(cudaMemcpyAsync(a.get(), &h, sizeof(h), cudaMemcpyHostToDevice, st[0]));
  GM_NCCL(nccl_api().AllGather(a.get(), all.get(), sizeof(h), ncclUint8,
                               static_cast<ncclComm_t>(nccl), st[0]));
  std::vector<cudaIpcMemHandle_t> hs(static_cast<size_t>(P));
  GM_CUDA(cudaMemcpyAsync(hs.data(), all.get(), sizeof(h) * size_t(P), cudaMemcpyDeviceToHost, st[0]));
  GM_CUDA(cudaStreamSynchronize(st[0]));
  // open every peer's handle; agree on success so no rank proceeds alone
  std::string err;
  for (int q = 0; q < P; ++q) {
    if (q == first) {
      t[0][size_t(q)] = local[0];
      continue;
    }
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, hs[size_t(q)], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      if (err.empty()) err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
      continue;
    }
    t[0][size_t(q)] = p;
  }
  const uint64_t bad = sum_host({err.empty() ? 0ull : 1ull});
  if (bad) {
    unshare(t);
    fail(GM_ECUDA, err.empty() ? "a peer could not map this rank's buffer" : err);
  }
  return t;
}

void Comm::unshare(std::vector<std::vector<void*>>& t) {
  if (use_nccl) {
    set(0);
    for (int q = 0; q < P; ++q)
      if (q != first && t[0][size_t(q)]) cudaIpcCloseMemHandle(t[0][size_t(q)]);
  }
  for (auto& row : t)
    for (auto& p : row) p = nullptr;
}

Comm* comm_create_local(int ndev, const int* devices) {
  if (ndev < 1 || ndev > kMaxShards)
    fail(GM_EUSAGE, "comm: 1 to " + std::to_string(kMaxShards) + " shards");
  int count = 0;
  GM_CUDA(cudaGetDeviceCount(&count));
  std::unique_ptr<Comm> c(new Comm());
  c->P = c->L = ndev;
  c->first = 0;
  for (int l = 0; l < ndev; ++l) {
    const int d = devices ? devices[l] : 0;
    if (d < 0 || d >= count)
      fail(GM_EUSAGE, "comm: device " + std::to_string(d) + " does not exist");
    c->dev.push_back(d);
  }
  for (int l = 0; l < ndev; ++l) {
    c->set(l);
    cudaStream_t s;
    GM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    c->st.push_back(s);
    cudaEvent_t e;
    GM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ev.push_back(e);
  }
  // peer access between the distinct devices (NVLink loads/stores)
  for (int a = 0; a < ndev; ++a)
    for (int b = 0; b < ndev; ++b) {
      const int da = c->dev[size_t(a)], db = c->dev[size_t(b)];
      if (da == db) continue;
      int ok = 0;
      GM_CUDA(cudaDeviceCanAccessPeer(&ok, da, db));
      if (!ok)
        fail(GM_ECUDA, "comm: device " + std::to_string(da) + " cannot access device " +
                           std::to_string(db) + " (no peer access)");
      GM_CUDA(cudaSetDevice(da));
      const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GM_CUDA(e);
      (void)cudaGetLastError();
    }
  return c.release();
}

void comm_nccl_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  GM_NCCL(nccl_api().GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
}

Comm* comm_create_nccl(int nranks, int rank, int device, const void* id128) {
  if (nranks < 1 || nranks > kMaxShards || rank < 0 || rank >= nranks)
    fail(GM_EUSAGE, "comm: bad nranks / rank");
  std::unique_ptr<Comm> c(new Comm());
  c->use_nccl = true;
  c->P = nranks;
  c->L = 1;
  c->first = rank;
  c->dev.push_back(device);
  c->set(0);
  cudaStream_t s;
  GM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  c->st.push_back(s);
  cudaEvent_t e;
  GM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c->ev.push_back(e);
  c->one.alloc(1, s);
  c->one.zero(s);
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t nc = nullptr;
  GM_NCCL(nccl_api().CommInitRank(&nc, nranks, id, rank));
  c->nccl = nc;
  return c.release();
}

}  // namespace gm
