// walk_d2.cu — 2-D kernels over the S=2 store.
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d2(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed<2, 2>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
