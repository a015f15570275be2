// walk_d14.cu — 14-D kernels over the S=16 store (buckets 1/8/16/32/64).
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d14(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed_hd<14, 16>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
