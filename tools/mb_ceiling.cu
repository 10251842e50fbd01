// tools/mb_ceiling.cu -- measurement aid (not product code): ceilings for one
// MIS-2 call on the 27-point 100^3 graph.
//   1. streaming read bandwidth of a 106 MB / 1 GiB int32 array (cold L2)
//   2. a second pass over the same 106 MB right after the first (L2 reuse),
//      with and without an L2 access-policy window marking it persisting
//   3. cost of the grid barrier (cooperative launch, B blocks)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbc tools/mb_ceiling.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void __launch_bounds__(256) rd(const int4* __restrict__ a, int64_t n4, unsigned long long* sink, int passes) {
    unsigned acc = 0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; p++)
        for (int64_t i = tid; i < n4; i += U * nth) {
            int4 q[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t ii = i + u * nth;
                q[u] = ii < n4 ? __ldcs(a + ii) : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; u++) acc += q[u].x ^ q[u].y ^ q[u].z ^ q[u].w;
        }
    if (acc == 0x12345u) sink[0] = acc;
}
template <int U>
__global__ void __launch_bounds__(256) rdn(const int4* __restrict__ a, int64_t n4, unsigned long long* sink, int passes) {
    unsigned acc = 0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; p++)
        for (int64_t i = tid; i < n4; i += U * nth) {
            int4 q[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t ii = i + u * nth;
                q[u] = ii < n4 ? a[ii] : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; u++) acc += q[u].x ^ q[u].y ^ q[u].z ^ q[u].w;
        }
    if (acc == 0x12345u) sink[0] = acc;
}

__device__ __forceinline__ void gbar(unsigned int* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = (blockIdx.x == 0) ? (0x80000000u - (gridDim.x - 1)) : 1u;
        unsigned int old;
        asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
        unsigned int cur;
        for (;;) {
            asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
            if ((old ^ cur) & 0x80000000u) break;
            __nanosleep(32);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}
__device__ __forceinline__ void gbar_nosleep(unsigned int* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = (blockIdx.x == 0) ? (0x80000000u - (gridDim.x - 1)) : 1u;
        unsigned int old;
        asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
        unsigned int cur;
        for (;;) {
            asm volatile("ld.acquire.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
            if ((old ^ cur) & 0x80000000u) break;
        }
    }
    __syncthreads();
}
template <int MODE>
__global__ void __launch_bounds__(256) bars(unsigned int* bar, int iters) {
    for (int i = 0; i < iters; i++) {
        if (MODE == 0) gbar(bar);
        else if (MODE == 1) gbar_nosleep(bar);
        else cooperative_groups::this_grid().sync();
    }
}

int main(int argc, char** argv) {
    const int64_t big = 1ll << 30, c2 = 26463592ll * 4;
    char *buf, *flush;
    unsigned long long* sink;
    CK(cudaMalloc(&buf, big));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(buf, 1, big));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    auto timeit = [&](auto fn, bool fl) {
        float best = 1e9, tot = 0;
        for (int r = 0; r < 7; r++) {
            if (fl) CK(cudaMemsetAsync(flush, r, 512 << 20, s));
            CK(cudaEventRecord(a, s));
            fn();
            CK(cudaEventRecord(b, s));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r >= 2) { best = ms < best ? ms : best; tot += ms; }
        }
        return best;
    };
    for (int64_t bytes : {c2, big}) {
        for (int per : {2, 4, 8, 16}) {
            const int grid = sms * per;
            float t4 = timeit([&] { rd<4><<<grid, 256, 0, s>>>((const int4*)buf, bytes / 16, sink, 1); }, true);
            float t8 = timeit([&] { rd<8><<<grid, 256, 0, s>>>((const int4*)buf, bytes / 16, sink, 1); }, true);
            float n8 = timeit([&] { rdn<8><<<grid, 256, 0, s>>>((const int4*)buf, bytes / 16, sink, 1); }, true);
            float p2 = timeit([&] { rdn<8><<<grid, 256, 0, s>>>((const int4*)buf, bytes / 16, sink, 2); }, true);
            printf("read %6.1f MB grid %4d: U4 cs %.1f us %.0f GB/s | U8 cs %.1f us %.0f GB/s | U8 %.1f us %.0f GB/s | 2 passes %.1f us (2nd pass %.0f GB/s)\n",
                   bytes / 1e6, grid, t4 * 1e3, bytes / t4 / 1e6, t8 * 1e3, bytes / t8 / 1e6, n8 * 1e3, bytes / n8 / 1e6,
                   p2 * 1e3, bytes / (p2 - n8) / 1e6);
        }
    }
    // L2 persisting window on the C2-sized array
    {
        int maxp = 0;
        CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp));
        for (float frac : {0.5f, 0.7f, 1.0f}) {
            cudaStreamAttrValue v = {};
            v.accessPolicyWindow.base_ptr = buf;
            v.accessPolicyWindow.num_bytes = c2;
            v.accessPolicyWindow.hitRatio = frac * (float)maxp / (float)c2 > 1.f ? 1.f : frac * (float)maxp / (float)c2;
            v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
            const int grid = sms * 8;
            float one = timeit([&] { CK(cudaCtxResetPersistingL2Cache()); rdn<8><<<grid, 256, 0, s>>>((const int4*)buf, c2 / 16, sink, 1); }, true);
            float two = timeit([&] { CK(cudaCtxResetPersistingL2Cache()); rdn<8><<<grid, 256, 0, s>>>((const int4*)buf, c2 / 16, sink, 2); }, true);
            float four = timeit([&] { CK(cudaCtxResetPersistingL2Cache()); rdn<8><<<grid, 256, 0, s>>>((const int4*)buf, c2 / 16, sink, 4); }, true);
            printf("persist window hitRatio %.2f (max %d B): 1 pass %.1f us, 2 passes %.1f, 4 passes %.1f -> extra pass %.1f us\n",
                   v.accessPolicyWindow.hitRatio, maxp, one * 1e3, two * 1e3, four * 1e3, (four - one) / 3 * 1e3);
            // flush effectiveness: run 1 pass after a memset flush WITHOUT reset
            float warm = timeit([&] { rdn<8><<<grid, 256, 0, s>>>((const int4*)buf, c2 / 16, sink, 1); }, true);
            printf("   1 pass after memset flush without persisting reset: %.1f us\n", warm * 1e3);
        }
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.num_bytes = 0;
        CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
        CK(cudaCtxResetPersistingL2Cache());
    }
    // grid barrier cost
    unsigned int* bar;
    CK(cudaMalloc(&bar, 64));
    CK(cudaMemset(bar, 0, 64));
    for (int per : {1, 2, 4}) {
        const int grid = sms * per;
        int iters = 1000;
        void* args[] = {&bar, &iters};
        float t0 = timeit([&] { CK(cudaLaunchCooperativeKernel((void*)bars<0>, grid, 256, args, 0, s)); }, false);
        float t1 = timeit([&] { CK(cudaLaunchCooperativeKernel((void*)bars<1>, grid, 256, args, 0, s)); }, false);
        float t2 = timeit([&] { CK(cudaLaunchCooperativeKernel((void*)bars<2>, grid, 256, args, 0, s)); }, false);
        printf("grid barrier, %d blocks: sleep-poll %.2f us, acquire-poll %.2f us, cg grid.sync %.2f us\n", grid,
               t0 * 1e3 / iters, t1 * 1e3 / iters, t2 * 1e3 / iters);
    }
    return 0;
}
