// gather_bench.cu -- microbenchmarks for the PageRank pull SpMV's gather bound.
//
// Each test streams an index array of M u32 (the CSR(G^T) column stream) and
// gathers x[idx] (4 B) from a vector of S floats, summing per thread.  It tells
// the throughput of random 4-byte gathers served by L1 / L2 / shared memory on
// this GPU, which bounds k_pr_spmv.  Not product code.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return uint32_t((z ^ (z >> 31)) >> 16);
}

// mode 0: uniform [0, S); mode 1: hub fraction hf in [0, H), rest uniform in [H, S)
// mode 2: sorted within blocks of B entries (monotone), uniform [0,S)
__global__ void k_gen(uint32_t* idx, uint64_t m, uint32_t S, int mode, uint32_t H, float hf) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t r = mix(i * 2 + 1);
    if (mode == 0) idx[i] = r % S;
    else if (mode == 2) {  // monotone within chunks of H entries spread over [0, S)
      uint64_t c = i % H;
      idx[i] = uint32_t((c * S) / H);
    } else {
      uint32_t q = mix(i * 2 + 2);
      if ((q & 0xFFFF) < uint32_t(hf * 65536.f)) idx[i] = r % H;
      else idx[i] = H + r % (S - H);
    }
  }
}

__global__ void k_fill(float* x, uint32_t S) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) x[i] = 1e-7f * (i % 977);
}

template <int U>
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ idx, const float* __restrict__ x, uint64_t m, float* out) {
  float acc = 0.f;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t b = (blockIdx.x * uint64_t(blockDim.x)) * U + threadIdx.x; b < m; b += stride) {
    uint32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t k = b + u * blockDim.x; j[u] = k < m ? __ldg(&idx[k]) : 0; }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __ldg(&x[j[u]]);
  }
  if (acc == 123.f) out[0] = acc;
}

// idx stream only (no gather): the streaming floor
__global__ void __launch_bounds__(256) k_stream(const uint4* __restrict__ idx, uint64_t m4, float* out) {
  uint32_t acc = 0;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < m4; k += uint64_t(gridDim.x) * blockDim.x) {
    uint4 v = __ldg(&idx[k]);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 12345) out[0] = acc;
}

// persistent: hub prefix x[0,H) in smem, tail from global
__device__ __forceinline__ float ld_na(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
template <int U, int LD = 0>
__global__ void __launch_bounds__(1024, 1) k_gather_smem(const uint32_t* __restrict__ idx, const float* __restrict__ x, uint64_t m, uint32_t H, float* out) {
  extern __shared__ float sx[];
  for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) sx[i] = x[i];
  __syncthreads();
  float acc = 0.f;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t b = (blockIdx.x * uint64_t(blockDim.x)) * U + threadIdx.x; b < m; b += stride) {
    uint32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t k = b + u * blockDim.x; j[u] = k < m ? __ldg(&idx[k]) : 0; }
#pragma unroll
    for (int u = 0; u < U; ++u)
      acc += j[u] < H ? sx[j[u]] : (LD == 0 ? __ldg(&x[j[u]]) : LD == 1 ? __ldcg(&x[j[u]]) : ld_na(&x[j[u]]));
  }
  if (acc == 123.f) out[0] = acc;
}

// smem atomics throughput: per entry, atomicAdd into smem at a hashed slot
template <int KIND>
__global__ void __launch_bounds__(1024, 1) k_satom(const uint32_t* __restrict__ idx, uint64_t m, uint32_t R, float* out) {
  extern __shared__ unsigned long long sacc[];
  float* sf = reinterpret_cast<float*>(sacc);
  for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) sacc[i] = 0;
  __syncthreads();
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 4;
  for (uint64_t b = (blockIdx.x * uint64_t(blockDim.x)) * 4 + threadIdx.x; b < m; b += stride) {
    uint32_t j[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { uint64_t k = b + u * blockDim.x; j[u] = k < m ? __ldg(&idx[k]) : 0; }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t s = (j[u] * 2654435761u) % R;
      if (KIND == 0) atomicAdd(&sacc[s], (unsigned long long)j[u]);
      else if (KIND == 1) atomicAdd(&sf[s], 1e-7f);
      else sf[s] += 1e-7f;  // racy plain RMW: the no-atomic floor
    }
  }
  __syncthreads();
  if (sacc[threadIdx.x] == 12345) out[0] = 1;
}

int main() {
  const uint64_t M = 131165091ull;  // scale-23 nnz
  uint32_t* idx; float* x; float* out;
  CK(cudaMalloc(&idx, M * 4 + 64));
  CK(cudaMalloc(&x, (1u << 23) * 4));
  CK(cudaMalloc(&out, 64));
  int dev; CK(cudaGetDevice(&dev));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  k_fill<<<1024, 256>>>(x, 1u << 23);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    return best * 1000.f;
  };
  const uint32_t grid = nsm * 8;
  k_gen<<<4096, 256>>>(idx, M, 1u << 23, 0, 0, 0.f);
  CK(cudaDeviceSynchronize());
  float us = timeit([&] { k_stream<<<grid, 256>>>((const uint4*)idx, M / 4, out); });
  printf("stream idx only: %.1f us  %.0f GB/s\n", us, M * 4 / us / 1e3);
  const uint32_t sizes[] = {32768, 1u << 20, 3851872, 1u << 23};
  for (uint32_t S : sizes) {
    k_gen<<<4096, 256>>>(idx, M, S, 0, 0, 0.f);
    CK(cudaDeviceSynchronize());
    float u8 = timeit([&] { k_gather<8><<<grid, 256>>>(idx, x, M, out); });
    float u16 = timeit([&] { k_gather<16><<<grid, 256>>>(idx, x, M, out); });
    printf("uniform S=%u (%.1f MB): U8 %.1f us (%.1f Ggather/s)  U16 %.1f us\n", S, S * 4 / 1e6, u8, M / u8 / 1e3, u16);
  }
  // hub-skewed like R-MAT 23 relabeled: 51% in top 48K, rest over non-dangling
  for (float hf : {0.51f, 0.0f}) {
    const uint32_t H = 49152, S = 3851872;
    k_gen<<<4096, 256>>>(idx, M, S, 1, H, hf);
    CK(cudaDeviceSynchronize());
    float u8 = timeit([&] { k_gather<8><<<grid, 256>>>(idx, x, M, out); });
    CK(cudaFuncSetAttribute(k_gather_smem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, H * 4));
    float sm = timeit([&] { k_gather_smem<8><<<nsm, 1024, H * 4>>>(idx, x, M, H, out); });
    CK(cudaGetLastError());
    printf("skew hf=%.2f: global U8 %.1f us; smem-hub persistent %.1f us\n", hf, u8, sm);
    CK(cudaFuncSetAttribute(k_gather_smem<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, H * 4));
    CK(cudaFuncSetAttribute(k_gather_smem<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, H * 4));
    CK(cudaFuncSetAttribute(k_gather_smem<16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, H * 4));
    float s1 = timeit([&] { k_gather_smem<8, 1><<<nsm, 1024, H * 4>>>(idx, x, M, H, out); });
    float s2 = timeit([&] { k_gather_smem<8, 2><<<nsm, 1024, H * 4>>>(idx, x, M, H, out); });
    float s3 = timeit([&] { k_gather_smem<16, 0><<<nsm, 1024, H * 4>>>(idx, x, M, H, out); });
    printf("   smem-hub variants: ldcg %.1f us, nc.no_allocate %.1f us, U16 %.1f us\n", s1, s2, s3);
  }
  {
    k_gen<<<4096, 256>>>(idx, M, 3851872, 0, 0, 0.f);
    CK(cudaDeviceSynchronize());
    for (uint32_t g : {nsm * 8u, nsm * 4u, 74u * 8u, 37u * 8u}) {
      float u8 = timeit([&] { k_gather<8><<<g, 256>>>(idx, x, M, out); });
      printf("uniform 3.85M grid %u: %.1f us (%.1f Ggather/s)\n", g, u8, M / u8 / 1e3);
    }
  }
  for (uint32_t C : {392000u, 100000u}) {
    k_gen<<<4096, 256>>>(idx, M, 3851872, 2, C, 0.f);
    CK(cudaDeviceSynchronize());
    float u8 = timeit([&] { k_gather<8><<<grid, 256>>>(idx, x, M, out); });
    printf("monotone chunks of %u over 3.85M: U8 %.1f us\n", C, u8);
  }
  for (uint32_t R : {8192u, 24576u}) {
    k_gen<<<4096, 256>>>(idx, M, 1u << 23, 0, 0, 0.f);
    CK(cudaFuncSetAttribute(k_satom<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, R * 8));
    CK(cudaFuncSetAttribute(k_satom<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, R * 8));
    CK(cudaFuncSetAttribute(k_satom<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, R * 8));
    float a0 = timeit([&] { k_satom<0><<<nsm, 1024, R * 8>>>(idx, M, R, out); });
    float a1 = timeit([&] { k_satom<1><<<nsm, 1024, R * 8>>>(idx, M, R, out); });
    float a2 = timeit([&] { k_satom<2><<<nsm, 1024, R * 8>>>(idx, M, R, out); });
    CK(cudaGetLastError());
    printf("smem atomics R=%u: u64 add %.1f us, f32 add %.1f us, plain rmw %.1f us\n", R, a0, a1, a2);
  }
  return 0;
}
