// walk_heap.cu — large-k / runtime-dim kernels (list kept in the output slot).
#include "walk_inst.cuh"
namespace fkd {
int launch_walk_heap(const WalkArgs& a, int dim, bool stats, bool unordered, cudaStream_t st) {
    switch (dim) {
        case 1: return launch_heap<1>(a, stats, unordered, st);
        case 2: return launch_heap<2>(a, stats, unordered, st);
        case 3: return launch_heap<3>(a, stats, unordered, st);
        case 4: return launch_heap<4>(a, stats, unordered, st);
        default: return launch_heap<0>(a, stats, unordered, st);
    }
}
}  // namespace fkd
