// Probe: do CUB's DeviceRadixSort::SortKeys and in-place DeviceSelect::Flagged
// handle more than 2^32 items (int64 num_items)?  Prints sortedness / counts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/cub_big tools/cub_big.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>

__global__ void fill(uint64_t* k, int64_t m, uint8_t* f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t x = uint64_t(i) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 32;
    k[i] = x & ((1ull << 56) - 1);
    if (f) f[i] = (x >> 60) & 1;
  }
}

__global__ void check_sorted(const uint64_t* k, int64_t m, unsigned long long* bad, unsigned long long* sum) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    if (i > 0 && k[i - 1] > k[i]) atomicAdd(bad, 1ull);
    s += k[i] & 0xFFFF;
  }
  atomicAdd(sum, s);
}

__global__ void sum_keys(const uint64_t* k, int64_t m, unsigned long long* sum) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    s += k[i] & 0xFFFF;
  atomicAdd(sum, s);
}

__global__ void count_flags(const uint8_t* f, int64_t m, unsigned long long* c) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    s += f[i];
  atomicAdd(c, s);
}

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 5000000000ll;
  uint64_t *k, *k2;
  uint8_t* f;
  unsigned long long *bad, *sum, *sum0;
  int64_t* cnt;
  cudaMalloc(&k, m * 8);
  cudaMalloc(&k2, m * 8);
  cudaMalloc(&f, m);
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&sum, 8);
  cudaMallocManaged(&sum0, 8);
  cudaMallocManaged(&cnt, 8);
  *bad = 0; *sum = 0; *sum0 = 0;
  fill<<<148 * 16, 256>>>(k, m, nullptr);
  sum_keys<<<148 * 16, 256>>>(k, m, sum0);
  cub::DoubleBuffer<uint64_t> db(k, k2);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, m, 0, 56);
  void* t;
  cudaMalloc(&t, tmp);
  cudaError_t e = cub::DeviceRadixSort::SortKeys(t, tmp, db, m, 0, 56);
  cudaDeviceSynchronize();
  check_sorted<<<148 * 16, 256>>>(db.Current(), m, bad, sum);
  cudaDeviceSynchronize();
  printf("sort m=%lld err=%s tmp=%zu unsorted_pairs=%llu checksum %s\n", (long long)m,
         cudaGetErrorString(e), tmp, *bad, *sum == *sum0 ? "ok" : "MISMATCH");
  // in-place select
  fill<<<148 * 16, 256>>>(k, m, f);
  unsigned long long* want;
  cudaMallocManaged(&want, 8);
  *want = 0;
  cudaDeviceSynchronize();
  count_flags<<<148 * 16, 256>>>(f, m, want);
  cudaDeviceSynchronize();
  tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, k, f, cnt, m);
  cudaFree(t);
  cudaMalloc(&t, tmp);
  e = cub::DeviceSelect::Flagged(t, tmp, k, f, cnt, m);
  cudaDeviceSynchronize();
  printf("select m=%lld err=%s selected=%lld expected=%llu\n", (long long)m, cudaGetErrorString(e),
         (long long)*cnt, *want);
  printf("last error %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
