// walk_d1.cu — 1-D kernels over the S=1 store.
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d1(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed<1, 1>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
