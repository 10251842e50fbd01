// mis2_g32.cu -- instantiations of the MIS-2 kernels (mis2_kernel.cuh) for
// lane-group width G = 32; one translation unit per G so the build runs in parallel.
#include "mis2_kernel.cuh"

namespace mis2h {
using namespace mis2k;

template <int G>
void* persistent_kernel(bool stats, bool push);
template <>
void* persistent_kernel<32>(bool stats, bool push) {
    if (stats) return push ? (void*)&mis2_persistent<32, true, true> : (void*)&mis2_persistent<32, true, false>;
    return push ? (void*)&mis2_persistent<32, false, true> : (void*)&mis2_persistent<32, false, false>;
}

template <int G>
cudaError_t launch_part_phase(int ph, const MisParams& p, int it, int grid, int smem, int* cnts,
                              unsigned long long* wl1, cudaStream_t s);
template <>
cudaError_t launch_part_phase<32>(int ph, const MisParams& p, int it, int grid, int smem, int* cnts,
                                 unsigned long long* wl1, cudaStream_t s) {
    if (ph == 0) {
        cudaFuncSetAttribute((const void*)mis2_part_phase<32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        mis2_part_phase<32, 0><<<grid, kMB, smem, s>>>(p, it, cnts, wl1);
    } else {
        cudaFuncSetAttribute((const void*)mis2_part_phase<32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        mis2_part_phase<32, 1><<<grid, kMB, smem, s>>>(p, it, cnts, wl1);
    }
    return cudaGetLastError();
}

}  // namespace mis2h
