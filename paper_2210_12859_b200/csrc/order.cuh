// order.cuh — Morton query ordering and tree-store helpers (order.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "fkd_b200.h"

namespace fkd {

struct MortonFrame {
    float lo[8];
    float scale[8];  // (2^bits - 1) / extent, 0 for a flat axis
    int bits;        // bits per dimension
};

int morton_bits_per_dim(int dim);
size_t morton_temp_bytes(int64_t m, int dim);
// Keys + counting or radix sort; ids_out receives the walk order.  The key
// pass also records the first non-finite query (id_base + i) in *bad.
// Returns launches or -1.
int morton_order(const float* d_queries, int64_t m, int dim, const MortonFrame& f,
                 uint32_t* keys_in, uint32_t* keys_out, uint32_t* ids_in, uint32_t* ids_out,
                 void* temp, size_t temp_bytes, unsigned long long* bad, int64_t id_base, cudaStream_t st);
// Morton keys only (frame resolution, f.bits per axis), first non-finite id -> *bad.
int morton_keys(const float* d_queries, int64_t m, int dim, const MortonFrame& f, uint32_t* keys,
                unsigned long long* bad, cudaStream_t st);
// First non-finite query (id_base + i) -> *bad, for batches walked without the key pass.
int scan_queries(const float* d_queries, int64_t m, int dim, unsigned long long* bad, int64_t id_base,
                 cudaStream_t st);

// *flag |= 1 if any of d_counts[0, m) differs from want.
int check_counts(const int32_t* d_counts, int64_t m, int32_t want, unsigned long long* flag, cudaStream_t st);

int pack_nodes(const float* d_src, int64_t n, int dim, int stride, float* d_dst, cudaStream_t st);
int tree_scan(const float* d_src, int64_t n, int dim, unsigned* d_lohi, unsigned long long* d_bad,
              cudaStream_t st);
float ordered_to_float(unsigned u);
int fill_empty(int32_t* d_counts, fkd_hit* d_hits, int64_t m, int k, cudaStream_t st);

}  // namespace fkd
