// mis2_g2s.cu -- a second copy of the MIS-2 kernels (mis2_kernel.cuh) for
// lane-group width G = 2 with smaller staging buffers (160-row tiles): on a
// skewed graph the shared memory they leave is L1, where the hubs' words stay
// (run_mis2).  Its own namespace (mis2k_s); MisParams has the same layout.
#define MIS2_TILE_ROWS 160
#define MIS2_GQ 1  // the skewed graphs' kernel: global queue of deferred rows
// rows for a whole block from 4K entries (balanced by the queue): C4, 1K /
// 2K / 4K / 8K / 32K: 28.8 / 28.8 / 27.4 / 27.5 / 28.3 ms
#define MIS2_HUGE_ROW 4096
#define mis2k mis2k_s
#include "mis2_kernel.cuh"
#undef mis2k

namespace mis2h {

template <int G>
void* persistent_kernel_small(bool stats, bool push);
template <>
void* persistent_kernel_small<2>(bool stats, bool push) {
    using namespace mis2k_s;
    if (stats) return push ? (void*)&mis2_persistent<2, true, true> : (void*)&mis2_persistent<2, true, false>;
    return push ? (void*)&mis2_persistent<2, false, true> : (void*)&mis2_persistent<2, false, false>;
}

}  // namespace mis2h
