// walk_d4.cu — 4-D kernels over the S=4 store.
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d4(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed<4, 4>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
