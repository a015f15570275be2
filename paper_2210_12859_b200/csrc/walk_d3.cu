// walk_d3.cu — 3-D kernels: padded float4 store (S=4) and packed 12-byte store (S=3).
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d3(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    if (S == 3) return launch_fixed<3, 3>(a, KB, stats, unordered, phase, st);
    return launch_fixed<3, 4>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
