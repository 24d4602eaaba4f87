// dsmem_bench.cu -- random 4-byte gathers served by distributed shared memory
// (cluster of C CTAs, each holding H floats of x), versus local smem and L2.
// Decides whether a cluster-wide hub window can replace L2 gathers in the
// PageRank pull SpMV.  Not product code.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return uint32_t((z ^ (z >> 31)) >> 16);
}
__global__ void k_gen(uint32_t* idx, uint64_t m, uint32_t S) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m; i += uint64_t(gridDim.x) * blockDim.x)
    idx[i] = mix(i * 2 + 1) % S;
}

// REMOTE: 0 = every load from the local CTA's smem; 1 = from CTA (j % C) of the cluster
template <int C, int REMOTE, int U>
__global__ void __launch_bounds__(1024, 1) k_dsmem(const uint32_t* __restrict__ idx, uint64_t m, uint32_t H, float* out) {
  extern __shared__ float sx[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) sx[i] = 1e-7f * i;
  cl.sync();
  float acc = 0.f;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t b = (blockIdx.x * uint64_t(blockDim.x)) * U + threadIdx.x; b < m; b += stride) {
    uint32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t k = b + u * blockDim.x; j[u] = k < m ? __ldg(&idx[k]) : 0; }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t rank = j[u] % C, off = (j[u] / C) % H;
      if (REMOTE) acc += cl.map_shared_rank(sx, rank)[off];
      else acc += sx[off];
    }
  }
  if (acc == 123.f) out[0] = acc;
  cl.sync();
}

template <int C, int REMOTE>
int run(const uint32_t* idx, uint64_t M, uint32_t H, float* out, int nsm) {
  auto kern = k_dsmem<C, REMOTE, 8>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, H * 4));
  if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = H * 4; cfg.attrs = at; cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int ncl = 0;
  CK(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
  cfg.gridDim = dim3(ncl * C);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaLaunchKernelEx(&cfg, kern, idx, M, H, out));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, kern, idx, M, H, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("cluster %d remote %d: %d clusters (%d CTAs) H=%u: %.1f us  %.1f Gload/s  %.2f loads/cyc/SM(1.965GHz)\n", C, REMOTE, ncl, ncl * C, H,
         best * 1e3, M / (best * 1e6), M / (best * 1e-3) / (ncl * C) / 1.965e9);
  return 0;
}

int main() {
  const uint64_t M = 131165091ull;
  uint32_t* idx; float* out;
  CK(cudaMalloc(&idx, M * 4)); CK(cudaMalloc(&out, 64));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  k_gen<<<4096, 256>>>(idx, M, 1u << 30);
  CK(cudaDeviceSynchronize());
  const uint32_t H = 50000;
  run<1, 0>(idx, M, H, out, nsm);
  run<2, 1>(idx, M, H, out, nsm);
  run<4, 1>(idx, M, H, out, nsm);
  run<8, 1>(idx, M, H, out, nsm);
  run<16, 1>(idx, M, H, out, nsm);
  return 0;
}
