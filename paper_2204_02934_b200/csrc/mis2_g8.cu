// mis2_g8.cu -- instantiations of the MIS-2 kernels (mis2_kernel.cuh) for
// lane-group width G = 8; one translation unit per G so the build runs in parallel.
#include "mis2_kernel.cuh"

namespace mis2h {
using namespace mis2k;

template <int G>
void* persistent_kernel(bool stats, bool push);
template <>
void* persistent_kernel<8>(bool stats, bool push) {
    if (stats) return push ? (void*)&mis2_persistent<8, true, true> : (void*)&mis2_persistent<8, true, false>;
    return push ? (void*)&mis2_persistent<8, false, true> : (void*)&mis2_persistent<8, false, false>;
}

template <int G>
void* dist_kernel();
template <>
void* dist_kernel<8>() {
    return (void*)&mis2_dist_persistent<8>;
}

}  // namespace mis2h
