// common.cuh -- shared device/host plumbing for the B200 GraphMat backend.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>

#include "graphmat_b200.h"

namespace gm {

// Library-internal exception; translated to gm_status at the C ABI boundary
// (capi.cu).  InputError/EngineError of the reference (core.hpp:44-57) map to
// GM_EINPUT / GM_EENGINE.
struct Error {
  gm_status code;
  std::string msg;
};

[[noreturn]] inline void fail(gm_status code, std::string msg) { throw Error{code, std::move(msg)}; }

// A failed runtime call also leaves its (non-sticky) error in the runtime's
// last-error slot; it is cleared here so the next launch check of an
// unrelated call does not report it again.
#define GM_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      (void)cudaGetLastError();                                                          \
      ::gm::fail(GM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
    }                                                                                    \
  } while (0)

// Every kernel launch is followed by GM_LAUNCH_CHECK(), which also counts it
// (gm_kernel_launches(): the benchmark's launch evidence).
void count_launch();
uint64_t launches_so_far();
#define GM_LAUNCH_CHECK()      \
  do {                         \
    ::gm::count_launch();      \
    GM_CUDA(cudaGetLastError()); \
  } while (0)

// Device-side bounds checks of the hot kernels' indirect accesses, compiled in
// only for the checked build (libgraphmat_b200_checked.so, -DGM_DEVICE_CHECKS;
// tests/test_gpu_checked.py): a violated check prints its location and traps,
// which fails the call with GM_ECUDA.  The stand-in for compute-sanitizer's
// memcheck where the tool is unavailable.
#ifdef GM_DEVICE_CHECKS
#define GM_DCHECK(cond)                                                                   \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("GM_DCHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);              \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define GM_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

// RAII device buffer (stream-ordered allocation on the graph's stream).
template <typename T>
class DevBuf {
 public:
  using value_type = T;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { swap(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      swap(o);
    }
    return *this;
  }
  ~DevBuf() { reset(); }

  void alloc(size_t n, cudaStream_t s) {
    reset();
    n_ = n;
    s_ = s;
    if (n) GM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
  }
  void reset() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  void swap(DevBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(s_, o.s_);
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }
  explicit operator bool() const { return p_ != nullptr; }
  void zero(cudaStream_t s) {
    if (n_) GM_CUDA(cudaMemsetAsync(p_, 0, bytes(), s));
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

// Pinned host scratch for small per-superstep readbacks.
template <typename T>
class HostPinned {
 public:
  explicit HostPinned(size_t n = 1) {
    GM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p_), n * sizeof(T)));
    n_ = n;
  }
  ~HostPinned() {
    if (p_) cudaFreeHost(p_);
  }
  HostPinned(const HostPinned&) = delete;
  HostPinned& operator=(const HostPinned&) = delete;
  T* get() const { return p_; }
  T& operator[](size_t i) const { return p_[i]; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

inline unsigned bits_for(uint64_t n) {  // bits needed to hold values < n (>= 1)
  unsigned b = 1;
  while (b < 64 && (uint64_t(1) << b) < n) ++b;
  return b;
}

inline unsigned grid_for(uint64_t work, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (work + block - 1) / block;
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

inline size_t value_size(int t) {
  switch (t) {
    case GM_VAL_F64:
    case GM_VAL_I64:
      return 8;
    case GM_VAL_F32:
    case GM_VAL_U32:
      return 4;
    case GM_VAL_U8:
      return 1;
    default:
      return 0;
  }
}

inline const char* value_name(int t) {
  switch (t) {
    case GM_VAL_F64: return "f64";
    case GM_VAL_F32: return "f32";
    case GM_VAL_U8: return "u8";
    case GM_VAL_I64: return "i64";
    case GM_VAL_U32: return "u32";
    default: return "none";
  }
}

// ------------------------------------------------------------------ RNG
// Counter-based generators shared by ingest kernels (host + device).  The
// oracle restates the same definitions independently (oracle/graphmat_oracle.c).

__host__ __device__ inline void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    const uint64_t p0 = uint64_t(0xD2511F53u) * c0, p1 = uint64_t(0xCD9E8D57u) * c2;
    const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
    const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
#endif
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Seeded bijection on [0, 2^scale).
struct PermKeys {
  uint64_t add[4], mul[4], mask;
  unsigned shift;
};

inline PermKeys make_perm_keys(unsigned scale, uint64_t seed) {
  PermKeys pk{};
  uint64_t st = seed ^ 0x7E57AB1E5EEDull;
  auto next = [&st]() {
    st += 0x9E3779B97F4A7C15ull;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  for (int r = 0; r < 4; ++r) {
    pk.add[r] = next();
    pk.mul[r] = next() | 1ull;
  }
  pk.mask = scale >= 64 ? ~0ull : ((1ull << scale) - 1ull);
  pk.shift = scale / 2 + 1;
  return pk;
}

__host__ __device__ inline uint32_t perm_apply(const PermKeys& pk, uint32_t x) {
  uint64_t v = x;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    v = (v + pk.add[r]) & pk.mask;
    v = (v * pk.mul[r]) & pk.mask;
    v ^= v >> pk.shift;
  }
  return static_cast<uint32_t>(v);
}

__host__ __device__ inline uint8_t edge_weight(uint64_t seed_w, uint32_t src, uint32_t dst) {
  const uint64_t h = mix64(seed_w ^ ((uint64_t(src) << 32) | dst));
  return static_cast<uint8_t>(1u + uint32_t((h >> 32) % 255u));
}

__host__ __device__ inline uint8_t rating_of(uint64_t seed_r, uint32_t user, uint32_t item) {
  const uint32_t h = uint32_t(mix64(seed_r ^ ((uint64_t(user) << 32) | item)) >> 32);
  uint8_t r = 1;
  r += h >= 214748365u;
  r += h >= 644245094u;
  r += h >= 1889785610u;
  r += h >= 3350074491u;
  return r;
}

inline uint64_t prob_threshold(double p) {
  if (p >= 1.0) return 1ull << 32;
  if (p <= 0.0) return 0;
  return static_cast<uint64_t>(p * 4294967296.0);
}

// ------------------------------------------------------------ device utils
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ bool bit_test(const uint32_t* bm, uint32_t v) {
  return (bm[v >> 5] >> (v & 31u)) & 1u;
}

// Warp-aggregated atomic add on a 64-bit counter.
__device__ __forceinline__ void warp_add_u64(unsigned long long* ctr, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane_id() == 0 && v) atomicAdd(ctr, v);
}

}  // namespace gm
