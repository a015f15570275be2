// trace.cuh — literal-state-machine walks with event traces (trace.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fkd_b200.h"

namespace fkd {
int launch_trace(const float* nodes, int32_t n, int dim, int stride, const float* queries, int m,
                 float cap2, int k, int32_t* counts, fkd_hit* hits, fkd_query_stats* stats,
                 int32_t* events, int64_t cap, int64_t* lens, cudaStream_t st);
}
