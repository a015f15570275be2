// walk_d10.cu — 10-D kernels over the S=12 store (buckets 1/8/16/32/64).
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d10(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    (void)S;
    return launch_fixed_hd<10, 12>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
