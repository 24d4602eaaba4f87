/* Host-side expansion of a packed level vector (u8 or u4 -> int32) with T
 * threads, on the GPU box's host cores: does a compressed D2H plus a host
 * expand beat copying 4 bytes per vertex over PCIe?  Not product code.
 * gcc -O3 -march=native -pthread -o tools/host_expand_bench tools/host_expand_bench.c */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static uint64_t N = 268435456ull;
static uint8_t* src8;
static int32_t* dst;
static int nib;
typedef struct { uint64_t lo, hi; } Range;

static void* work(void* p) {
  Range r = *(Range*)p;
  if (!nib) {
    for (uint64_t i = r.lo; i < r.hi; ++i) dst[i] = (int32_t)src8[i] - 1;
  } else {
    for (uint64_t i = r.lo; i < r.hi; i += 2) {
      const uint8_t b = src8[i >> 1];
      dst[i] = (int32_t)(b & 15) - 1;
      dst[i + 1] = (int32_t)(b >> 4) - 1;
    }
  }
  return NULL;
}

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

int main(void) {
  src8 = malloc(N);
  dst = malloc(N * 4);
  for (uint64_t i = 0; i < N; ++i) src8[i] = (uint8_t)(i * 2654435761u >> 28);
  memset(dst, 0, N * 4);
  printf("nproc %ld\n", sysconf(_SC_NPROCESSORS_ONLN));
  for (nib = 0; nib < 2; ++nib)
    for (int T = 1; T <= 64; T *= 2) {
      pthread_t th[64];
      Range rg[64];
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        const double t0 = now();
        for (int t = 0; t < T; ++t) {
          rg[t].lo = (N / T) * t & ~63ull;
          rg[t].hi = t == T - 1 ? N : ((N / T) * (t + 1) & ~63ull);
          pthread_create(&th[t], NULL, work, &rg[t]);
        }
        for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
        const double dt = now() - t0;
        if (dt < best) best = dt;
      }
      printf("%s T=%d: %.2f ms (%.1f GB/s written)\n", nib ? "u4" : "u8", T, best * 1e3, N * 4 / best / 1e9);
    }
  return 0;
}
