// validate.cu -- device check of the input contract (mis2.h): rowptr
// monotone with rowptr[0] = 0 and rowptr[n] = nnz, colinds in range, rows
// strictly increasing (sorted, duplicate free), pattern symmetric.
#include "common.cuh"
#include "internal.h"

namespace mis2k {

enum { kBadRowptr = 1, kBadRange = 2, kBadOrder = 4, kBadSym = 8 };

// pass 1: rowptr[0] = 0, nondecreasing, rowptr[n] = nnz, within [0, nnz]
__global__ void k_validate_rowptr(int64_t n, int64_t nnz, const int64_t* __restrict__ rowptr, int* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const int64_t s = rowptr[v], e = rowptr[v + 1];
        if ((v == 0 && s != 0) || e < s || (v == n - 1 && e != nnz) || s < 0 || e > nnz) atomicOr(err, kBadRowptr);
    }
}
// pass 2 (skipped when pass 1 failed, so every row bound it reads is sound):
// colinds in range, rows strictly increasing, pattern symmetric
__global__ void k_validate(int64_t n, int64_t nnz, const int64_t* __restrict__ rowptr,
                           const int32_t* __restrict__ colinds, int* err) {
    if (*(volatile int*)err & kBadRowptr) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const int64_t s = rowptr[v], e = rowptr[v + 1];
        int32_t prev = -1;
        for (int64_t j = s; j < e; j++) {
            const int32_t w = colinds[j];
            if (w < 0 || w >= n) { atomicOr(err, kBadRange); break; }
            if (w <= prev) atomicOr(err, kBadOrder);
            prev = w;
            if (w == v) continue;
            // binary search v in row w
            int64_t lo = rowptr[w], hi = rowptr[w + 1];
            bool found = false;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                const int32_t x = colinds[mid];
                if (x == v) { found = true; break; }
                if (x < v) lo = mid + 1; else hi = mid;
            }
            if (!found) atomicOr(err, kBadSym);
        }
    }
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

int run_validate(const mis2_graph& g, void* ws, size_t ws_bytes, cudaStream_t s, size_t* bytes_needed) {
    Carve c(ws, ws_bytes);
    int* err = c.take<int>(4);
    if (bytes_needed) { *bytes_needed = c.off; return MIS2_OK; }
    if (!c.ok()) { set_error("workspace too small"); return MIS2_ENOMEM; }
    if (g.n == 0) return MIS2_OK;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    MIS2_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), s));
    int64_t blocks = (g.n + kBlock - 1) / kBlock;
    if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
    k_validate_rowptr<<<(unsigned)blocks, kBlock, 0, s>>>(g.n, g.nnz, g.rowptr, err);
    k_validate<<<(unsigned)blocks, kBlock, 0, s>>>(g.n, g.nnz, g.rowptr, g.colinds, err);
    count_launch(2);
    MIS2_CUDA_TRY(cudaGetLastError());
    int h = 0;
    MIS2_CUDA_TRY(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    if (h) {
        set_error("graph violates the input contract:%s%s%s%s", (h & kBadRowptr) ? " rowptr" : "",
                  (h & kBadRange) ? " colind-range" : "", (h & kBadOrder) ? " unsorted/duplicate" : "",
                  (h & kBadSym) ? " asymmetric" : "");
        return MIS2_EGRAPH;
    }
    return MIS2_OK;
}

}  // namespace mis2h
