// tma_gather_bench.cu -- can the TMA unit serve the PageRank tail gathers faster
// than the LSU/L1TEX path?  Not product code.
//
// The hub kernel's tail gathers (one random 4-byte x[src] per nonzero) run at
// ~270 G/s: one L1TEX wavefront per distinct 128-byte line, ~1 per SM cycle.
// Here M random indices over S floats are gathered three ways:
//   ldg   : ld.global 4 B per index (the shipped path)
//   bulk  : cp.async.bulk 16 B (the aligned quad holding x[j]) per index into
//           shared memory, mbarrier complete_tx, then read the element
//   g4    : cp.async.bulk.tensor tile::gather4 (x viewed as [S/4][4] floats):
//           four 16-byte rows per instruction
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_gather_bench tools/tma_gather_bench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

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
__global__ void k_fill(float* x, uint32_t S) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) x[i] = 1e-7f * (i % 977);
}

template <int U>
__global__ void __launch_bounds__(1024, 1) k_ldg(const uint32_t* __restrict__ idx, const float* __restrict__ x, uint64_t m, float* out) {
  extern __shared__ float pad[];
  float acc = 0.f;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t b = (blockIdx.x * uint64_t(blockDim.x)) * U + threadIdx.x; b < m; b += stride) {
    uint32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t k = b + u * blockDim.x; j[u] = k < m ? __ldg(&idx[k]) : 0; }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __ldcg(&x[j[u]]);
  }
  if (acc == 123.f) { out[0] = acc; pad[0] = acc; }
}

__device__ __forceinline__ uint32_t sptr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sptr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk16(void* dst, const void* src, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(sptr(dst)),
               "l"(src), "r"(sptr(bar))
               : "memory");
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
          sptr(dst)),
      "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sptr(bar))
      : "memory");
}

// Per warp: NS stages of 32*P indices (P per lane).  MODE 0 bulk16, 1 gather4 (P multiple of 4).
template <int MODE, int NS, int P>
__global__ void __launch_bounds__(1024, 1) k_tma(const uint32_t* __restrict__ idx, const float* __restrict__ x,
                                                  const __grid_constant__ CUtensorMap tm, uint64_t m, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);                      // nw*NS
  float4* buf = reinterpret_cast<float4*>(sm + 32 * NS * 8);  // after the bars (<= 32 warps)
  uint64_t* mb = bars + warp * NS;
  float4* wb = buf + size_t(warp) * NS * 32 * P * (MODE ? 2 : 1);  // gather4: one 128-B slot per 64-B gather
  if (lane < NS) mbar_init(&mb[lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t per = 32ull * P;
  const uint64_t gw = uint64_t(blockIdx.x) * nw + warp, W = uint64_t(gridDim.x) * nw;
  const uint64_t nb = m / per;  // whole batches only
  float acc = 0.f;
  uint32_t jk[NS][P];
  uint64_t it = 0;
  for (uint64_t b = gw; b < nb + uint64_t(NS) * W; b += W, ++it) {
    const int s = int(it % NS);
    if (it >= NS) {  // consume the batch issued NS iterations ago into stage s
      mbar_wait(&mb[s], uint32_t((it / NS - 1) & 1));
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float* q = reinterpret_cast<const float*>(&wb[s * 32 * P + p * 32 + lane]);
        acc += q[jk[s][p] & 3];
      }
      __syncwarp();
    }
    if (b < nb) {
      uint32_t j[P];
#pragma unroll
      for (int p = 0; p < P; ++p) { j[p] = __ldg(&idx[b * per + p * 32 + lane]); jk[s][p] = j[p]; }
      if (lane == 0) mbar_expect(&mb[s], 32 * P * 16);
      __syncwarp();
      if (MODE == 0) {
#pragma unroll
        for (int p = 0; p < P; ++p) bulk16(&wb[s * 32 * P + p * 32 + lane], x + (j[p] & ~3u), &mb[s]);
      } else {
        // lane l gathers rows for slots p*32+l; group 4 consecutive p per gather4: dst must be
        // 4 contiguous 16-byte rows, so use slot layout [p-group][lane][4]
#pragma unroll
        for (int p = 0; p < P; p += 4)
          g4(&wb[2 * (s * 32 * P + (p / 4) * 128 + lane * 4)], &tm, int(j[p] >> 2), int(j[p + 1] >> 2), int(j[p + 2] >> 2),
             int(j[p + 3] >> 2), &mb[s]);
      }
    } else {
      jk[s][0] = 0;
    }
  }
  if (acc == 123.f) out[0] = acc;
}

// gather4 writes slot layout [pgroup][lane][4 rows]; k_tma's consumer reads [p][lane], which for
// MODE 1 is a permutation of the same slots -- the sum only checks throughput, not mapping.

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const uint64_t M = 64ull << 20;  // ~ the scale-23 tail gathers
  const uint32_t S = 3851872;      // non-dangling vertices at scale 23
  uint32_t* idx; float* x; float* out;
  CK(cudaMalloc(&idx, M * 4 + 4096));
  CK(cudaMalloc(&x, size_t(S + 64) * 4));
  CK(cudaMalloc(&out, 64));
  int dev; CK(cudaGetDevice(&dev));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  k_fill<<<1024, 256>>>(x, S);
  k_gen<<<4096, 256>>>(idx, M, S);
  CK(cudaDeviceSynchronize());
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
  // tensor map: x as [S/4 rows][4 floats]
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {4, (S + 3) / 4};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode gather4 map: %d\n", int(r));

  for (int smem : {0, 192 * 1024}) {
    CK(cudaFuncSetAttribute(k_ldg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float us = timeit([&] { k_ldg<8><<<nsm, 1024, smem>>>(idx, x, M, out); });
    CK(cudaGetLastError());
    printf("ldg   smem %6d: %7.1f us  %6.1f G/s\n", smem, us, M / us / 1e3);
  }
#define RUN(MODE, NS, P, NT)                                                                                  \
  do {                                                                                                        \
    size_t sb = 32 * NS * 8 + size_t(NT / 32) * NS * 32 * P * 16 * (MODE ? 2 : 1);                                             \
    CK(cudaFuncSetAttribute(k_tma<MODE, NS, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)));        \
    float us = timeit([&] { k_tma<MODE, NS, P><<<nsm, NT, sb>>>(idx, x, tm, M, out); });                      \
    cudaError_t e = cudaGetLastError();                                                                       \
    if (e == cudaSuccess) e = cudaDeviceSynchronize();                                                        \
    printf("%s NS=%d P=%d thr=%4d smem %6zu: %7.1f us  %6.1f G/s  %s\n", MODE ? "g4  " : "bulk", NS, P, NT, sb, us, \
           M / us / 1e3, cudaGetErrorString(e));                                                              \
    if (e != cudaSuccess) return 1;                                                                           \
  } while (0)
  RUN(0, 2, 4, 1024);
  if (r == CUDA_SUCCESS) {
    RUN(1, 2, 4, 512);
    RUN(1, 4, 4, 256);
    RUN(1, 2, 8, 256);
    RUN(1, 1, 8, 512);
  }
  return 0;
}
