// Grid-barrier latency on the B200: cooperative-groups grid.sync() against
// hand-written barriers (one arrival counter, thread 0 of each CTA arrives and
// spins), for the BFS kernel's shape (2 CTAs x 1024 threads per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gsync_bench tools/gsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned x) {
  unsigned v;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "r"(x) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned x) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}

// variant 1: counter + generation word; last arriver resets the counter and
// bumps the generation (release); others spin with acquire loads.
template <int kMode>
__device__ __forceinline__ void bar(unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* cnt = &g_count;
    unsigned* gen = const_cast<unsigned*>(&g_gen);
    if (kMode == 1) {
      const unsigned g0 = ld_relaxed(gen);
      if (atom_add_acqrel(cnt, 1) == nblocks - 1) {
        *cnt = 0;
        st_release(gen, g0 + 1);
      } else {
        while (ld_acquire(gen) == g0) {
        }
      }
    } else if (kMode == 2) {  // relaxed spin, one acquire fence after
      const unsigned g0 = ld_relaxed(gen);
      if (atom_add_acqrel(cnt, 1) == nblocks - 1) {
        *cnt = 0;
        st_release(gen, g0 + 1);
      } else {
        while (ld_relaxed(gen) == g0) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    } else {  // kMode 3: no ordering at all (floor)
      const unsigned g0 = g_gen;
      if (atomicAdd(cnt, 1) == nblocks - 1) {
        *cnt = 0;
        g_gen = g0 + 1;
      } else {
        while (g_gen == g0) {
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 2) k_cg(int iters, unsigned long long* out) {
  cg::grid_group grid = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

template <int kMode>
__global__ void __launch_bounds__(1024, 2) k_custom(int iters, unsigned long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar<kMode>(gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  for (int threads : {1024, 512, 256}) {
    for (int per_sm : {1, 2}) {
      const int blocks = sms * per_sm;
      void* fns[] = {(void*)k_cg, (void*)k_custom<1>, (void*)k_custom<2>, (void*)k_custom<3>};
      const char* names[] = {"cg::grid.sync", "acq_rel counter + acquire spin", "relaxed spin + fence", "volatile (no ordering)"};
      for (int f = 0; f < 4; ++f) {
        int it = iters;
        void* args[] = {&it, &d};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaLaunchCooperativeKernel(fns[f], dim3(blocks), dim3(threads), args, 0, 0);  // warm
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(fns[f], dim3(blocks), dim3(threads), args, 0, 0);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s blocks %4d x %4d threads: %s %.3f us per barrier\n", names[f], blocks, threads,
               e == cudaSuccess ? "" : cudaGetErrorString(e), ms * 1e3 / iters);
      }
    }
  }
  return 0;
}
