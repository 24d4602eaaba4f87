// The generic hub kernel's sequential consumer (32-entry chunks of fp64 from
// shared memory, one acquire-load of a ready flag per chunk) timed alone and
// beside 15 other warps that (0) exit, (1) sleep 1 us in a loop, (2) poll a
// shared flag, (3) issue dependent global loads.  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/consumer_bench tools/consumer_bench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(unsigned(__cvta_generic_to_shared(p))) : "memory");
  return v;
}
__global__ void k(int mode, int nch, double* out, long long* cyc, const uint32_t* g) {
  __shared__ double ring[64 * 32];
  __shared__ int ready[64];
  __shared__ volatile int done;
  __shared__ int cntv[32];
  __shared__ volatile int cons;
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) ring[i] = 1e-9 * i;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) ready[i] = 1;
  for (int i = threadIdx.x; i < 32; i += blockDim.x) cntv[i] = 64;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp > 0) {
    if ((mode & 3) == 0) return;
    uint32_t j = threadIdx.x;
    while (!done) {
      if ((mode & 3) == 1) __nanosleep(1000);
      else if ((mode & 3) == 2) (void)ld_acquire_cta(&ready[lane]);
      else j = g[(j * 2654435761u) & ((1u << 24) - 1)];
    }
    if (j == 12345) out[1] = j;
    return;
  }
  if (lane) return;
  double acc = 0.0;
  const long long t0 = clock64();
  for (int c = 0; c < nch; ++c) {
    const int slot = c & 63;
    if (mode < 8) {
      while (ld_acquire_cta(&ready[slot]) != 1) {
      }
    } else {
      while (((volatile int*)ready)[slot] != 1) {
      }
    }
    const double* rs = ring + (slot & 31) * 64;
    const int cnt = cntv[slot & 31];
    if (cnt == 64) {
      if (mode < 4) {
#pragma unroll
        for (int u = 0; u < 64; ++u) acc = acc + rs[u];
      } else {
        // explicit double buffer of 16 values
        double a[16], b[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = rs[u];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          if (h < 3) {
#pragma unroll
            for (int u = 0; u < 16; ++u) b[u] = rs[16 * (h + 1) + u];
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) acc = acc + a[u];
#pragma unroll
          for (int u = 0; u < 16; ++u) a[u] = b[u];
        }
      }
    }
    if ((c & 1) && mode < 12) cons = c + 1;
  }
  const long long t1 = clock64();
  done = 1;
  out[0] = acc;
  cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o;
  long long* c;
  uint32_t* g;
  cudaMalloc(&o, 16);
  cudaMallocManaged(&c, 8 * 296);
  cudaMalloc(&g, 4u << 24);
  cudaMemset(g, 0, 4u << 24);
  const int nch = 6000;
  for (int mode = 0; mode < 16; mode += 4)
    for (int grid : {1, 296}) {
      k<<<grid, 512>>>(mode, nch, o, c, g);
      cudaDeviceSynchronize();
      k<<<grid, 512>>>(mode, nch, o, c, g);
      cudaDeviceSynchronize();
      printf("mode %d grid %d: %.2f cycles per entry\n", mode, grid, double(c[0]) / (nch * 64.0));
    }
  return 0;
}
