// tools/mb_hash.cu -- measurement aid (not product code): cost of computing
// the iteration-0 status words word(0, w) on the fly for every entry of the
// 27-point 100^3 stencil (1M rows x 27) instead of gathering T[w].
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbhash tools/mb_hash.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t xs(uint64_t x) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; }
__device__ __forceinline__ uint64_t xss(uint64_t x) { return xs(x) * 0x2545F4914F6CDD1Dull; }
template <int MODE>
__global__ void __launch_bounds__(256) k(int64_t n, const uint64_t* __restrict__ T, uint32_t* __restrict__ M, uint64_t fi, uint64_t mask) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nth) {
        uint64_t m = ~0ull;
#pragma unroll
        for (int q = 0; q < 27; q++) {
            const int dz = q / 9 - 1, dy = (q / 3) % 3 - 1, dx = q % 3 - 1;
            int64_t w = v + dx + 100 * dy + 10000 * dz;
            w = w < 0 ? 0 : (w >= n ? n - 1 : w);
            uint64_t t;
            if (MODE == 0) t = T[w];
            else t = (xss(fi ^ xss((uint64_t)w)) & mask) | (uint64_t)(w + 1);
            m = t < m ? t : m;
        }
        M[v] = (uint32_t)m;
    }
}
int main() {
    const int64_t n = 1000000;
    uint64_t* T; uint32_t* M;
    cudaMalloc(&T, 8 * n); cudaMalloc(&M, 4 * n); cudaMemset(T, 1, 8 * n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; mode++)
        for (int per : {4, 8}) {
            float best = 1e9;
            for (int r = 0; r < 6; r++) {
                cudaEventRecord(a);
                if (mode == 0) k<0><<<sms * per, 256>>>(n, T, M, 123, ~0xfffffull);
                else k<1><<<sms * per, 256>>>(n, T, M, 123, ~0xfffffull);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
            }
            printf("%s grid %d: %.1f us\n", mode ? "hash on the fly" : "gather T     ", sms * per, best * 1e3);
        }
    return 0;
}
