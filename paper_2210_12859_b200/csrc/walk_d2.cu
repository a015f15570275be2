// walk_d2.cu — 2-D kernels: 16-byte store with the split plane in its last
// float (S=4, default) and the packed 8-byte store (S=2, FKD_LAYOUT=packed).
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_d2(const WalkArgs& a, int S, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    if (S == 4) return launch_fixed<2, 4>(a, KB, stats, unordered, phase, st);
    return launch_fixed<2, 2>(a, KB, stats, unordered, phase, st);
}
}  // namespace fkd
