// walk_d7.cu — 7-D kernels over the S=8 store.
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d7(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed<7, 8>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
