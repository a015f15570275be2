// build.cuh — GPU level-order builder (build.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fkd {

struct BuildStatus {
    cudaError_t err = cudaSuccess;
    const char* what = "";
    int launches = 0;
};

// d_out[n*dim] receives flatkd::build_tree's level-order array (round-robin
// split), byte for byte.  Points must be finite (checked by the caller).
BuildStatus build_tree_device(const float* d_pts, int64_t n, int dim, float* d_out, cudaStream_t st);

}  // namespace fkd
