// walk_d8.cu — 8-D kernels over the S=8 store.
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d8(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed<8, 8>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
