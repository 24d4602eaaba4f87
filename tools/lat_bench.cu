// Dependent-chain latencies on one thread (clock64): DADD, FADD, LDS.64 +
// DADD (the generic hub consumer's fold step).  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, int n, double a) {
  __shared__ double sh[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = 1e-9 * i;
  __syncthreads();
  if (threadIdx.x) return;
  double acc = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = acc + a;
  }
  long long t1 = clock64();
  float f = float(a);
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) f = f + float(a);
  }
  long long t2 = clock64();
  double acc2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* p = sh + ((i * 16) & 4095);
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = p[u];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc2 = acc2 + v[u];
  }
  long long t3 = clock64();
  out[0] = acc + f + acc2;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMallocManaged(&c, 24);
  const int n = 4096;
  k<<<1, 128>>>(o, c, n, 1.0000001);
  cudaDeviceSynchronize();
  k<<<1, 128>>>(o, c, n, 1.0000001);
  cudaDeviceSynchronize();
  printf("DADD chain %.2f cycles/op, FADD chain %.2f, LDS.64+DADD chain %.2f\n", double(c[0]) / (n * 16),
         double(c[1]) / (n * 16), double(c[2]) / (n * 16));
  return 0;
}
