// walk_d15.cu — 15-D kernels over the S=16 store (buckets 1/8/16/32/64).
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d15(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed_hd<15, 16>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
