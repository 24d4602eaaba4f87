// ingest.cuh -- ingest building blocks shared by the single-GPU build
// (ingest.cu) and the sharded build (dist.cu).
#pragma once

#include "common.cuh"

namespace gm {

// Tuples [t0, t0 + count) of the seeded R-MAT stream (io::rmat_generate
// semantics, src/io.cpp:224-255; counter-based, so any range of tuples is
// generated independently -- each shard draws its own 1/P).
void rmat_range(unsigned scale, double a, double b, double c, uint64_t seed, int permute,
                uint64_t t0, uint64_t count, uint32_t* src, uint32_t* dst, cudaStream_t s);
// Ratings [part*T/parts, (part+1)*T/parts) of the seeded Zipf bipartite stream
// (T raw ratings in all, *total_out); src/dst sized by a first call with
// src = nullptr.  Returns the count.  users [0,U), items [U, U+I).
uint64_t bipartite_range(uint32_t users, uint32_t items, double c_num, uint32_t cap, uint64_t seed,
                         uint64_t part, uint64_t parts, uint32_t* src, uint32_t* dst,
                         uint64_t* total_out, cudaStream_t s);
// Stable LSD radix sort of 64-bit keys over bits [0, end_bit).
void sort_keys_u64(DevBuf<uint64_t>& keys, int64_t m, int end_bit, cudaStream_t s);
// Drop repeated keys of a sorted array in place; returns the new length.
int64_t unique_keys_u64(DevBuf<uint64_t>& keys, int64_t m, cudaStream_t s);
// ptr[0] = 0, ptr[i + 1] = counts[0] + ... + counts[i] (64-bit running sum).
void scan_counts_to_ptr(const uint32_t* counts, uint64_t* ptr, uint64_t n, cudaStream_t s);

}  // namespace gm
