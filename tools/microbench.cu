// tools/microbench.cu -- measurement aid (not product code): floors of the
// ingredients of one dense MIS-2 pass on the 27-point 100^3 graph.
//   mode 0: per-warp bulk-copy streaming of colinds tiles only
//   mode 1: mode 0 + thread-per-row T gathers + min + M write (the column pass)
//   mode 2: plain coalesced int4 streaming of colinds (no smem)
//   mode 3: thread-per-row gathers reading colinds straight from global
//   mode 4: mode 1 with 2 tiles processed per step (more gathers in flight)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kCap = 1024;
struct __align__(16) WS { int32_t buf[2][kCap + 8]; unsigned long long mbar[2]; };

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(b))); }
__device__ __forceinline__ void mb_tx(unsigned long long* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_wait(unsigned long long* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

// mode 5/6: cp.async.cg 16-byte staging (LDGSTS), double buffered per warp
__device__ __forceinline__ void cpa16(void* d, const void* s) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(d)), "l"(s) : "memory"); }
template <int MODE>
__global__ void __launch_bounds__(256) kb(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M, unsigned long long* sink) {
    extern __shared__ __align__(16) unsigned char raw[];
    WS& ws = reinterpret_cast<WS*>(raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int64_t W = (int64_t)gridDim.x * 8, gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int64_t lo = n * gw / W, hi = n * (gw + 1) / W;
    unsigned long long acc = 0;
    if (MODE == 8) {  // classic grid-stride int4 stream over the whole array, 4 loads in flight
        const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
        const int64_t n4 = nnz / 4;
        const int4* c4 = (const int4*)ci;
        for (int64_t i = tid; i < n4; i += 4 * nth) {
            int4 q[4];
#pragma unroll
            for (int u = 0; u < 4; u++) { const int64_t ii = i + u * nth; q[u] = ii < n4 ? c4[ii] : make_int4(0,0,0,0); }
#pragma unroll
            for (int u = 0; u < 4; u++) acc += q[u].x + q[u].y + q[u].z + q[u].w;
        }
        if (acc == 12345) sink[0] = acc;
        return;
    }
    if (MODE == 7) {  // unrolled int4 stream: 8 independent 16 B loads per lane
        const int64_t s = (rp[lo] + 3) & ~3ll, e = rp[hi] & ~3ll;
        for (int64_t j = s + 4 * lane; j < e; j += 128 * 8) {
            int4 q[8];
#pragma unroll
            for (int u = 0; u < 8; u++) { const int64_t jj = j + 128 * u; q[u] = jj < e ? *(const int4*)(ci + jj) : make_int4(0,0,0,0); }
#pragma unroll
            for (int u = 0; u < 8; u++) acc += q[u].x + q[u].y + q[u].z + q[u].w;
        }
        if (acc == 12345) sink[0] = acc;
        return;
    }
    const int ntiles = (int)((hi - lo + 31) / 32);
    auto issue = [&](int j, int b) {
        const int64_t r0 = lo + 32ll * j, r1 = r0 + 32 < hi ? r0 + 32 : hi;
        const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
        for (int64_t q = 4 * lane; q < e - s && q < kCap; q += 128) cpa16(ws.buf[b] + q, ci + s + q);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0, 0);
    for (int j = 0; j < ntiles; j++) {
        const int b = j & 1;
        __syncwarp();
        if (j + 1 < ntiles) issue(j + 1, b ^ 1);
        const int64_t v = lo + 32ll * j + lane;
        int64_t s = 0, e = 0;
        if (v < hi) { s = rp[v]; e = rp[v + 1]; }
        const int64_t sal = __shfl_sync(~0u, s, 0) & ~3ll;
        if (j + 1 < ntiles) asm volatile("cp.async.wait_group 1;" ::: "memory"); else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        if (MODE == 5) { if (v < hi) acc += ws.buf[b][s - sal]; continue; }
        if (v < hi) {
            const int32_t* x = ws.buf[b] + (s - sal);
            const int len = (int)(e - s);
            uint64_t m = T[v];
            for (int jj = 0; jj < len; jj += 16) {
                uint64_t tt[16];
#pragma unroll
                for (int q = 0; q < 16; q++) tt[q] = T[x[min(jj + q, len - 1)]];
#pragma unroll
                for (int q = 0; q < 16; q++) m = tt[q] < m ? tt[q] : m;
            }
            M[v] = (uint32_t)m;
        }
    }
    if (acc == 12345) sink[0] = acc;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                         const uint64_t* __restrict__ T, uint32_t* __restrict__ M, unsigned long long* sink) {
    extern __shared__ __align__(16) unsigned char raw[];
    WS& ws = reinterpret_cast<WS*>(raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int64_t W = (int64_t)gridDim.x * 8, gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int64_t lo = n * gw / W, hi = n * (gw + 1) / W;
    unsigned long long acc = 0;
    if (MODE == 2) {
        const int64_t s = rp[lo], e = rp[hi];
        const int64_t sa = (s + 3) & ~3ll, ea = e & ~3ll;
        for (int64_t j = sa + 4 * lane; j < ea; j += 128) { int4 q = *(const int4*)(ci + j); acc += q.x + q.y + q.z + q.w; }
        if (acc == 12345) sink[0] = acc;
        return;
    }
    if (MODE == 3) {
        for (int64_t r = lo + lane; r < hi + 31; r += 32) {
            uint64_t m = ~0ull;
            if (r < hi) { const int64_t s = rp[r], e = rp[r + 1]; for (int64_t j = s; j < e; j++) { uint64_t t = T[ci[j]]; m = t < m ? t : m; } M[r] = (uint32_t)m; }
        }
        return;
    }
    if (lane == 0) { mb_init(&ws.mbar[0]); mb_init(&ws.mbar[1]); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncwarp();
    const int ntiles = (int)((hi - lo + 31) / 32);
    auto issue = [&](int j, int b) {
        if (lane == 0) {
            const int64_t r0 = lo + 32ll * j, r1 = r0 + 32 < hi ? r0 + 32 : hi;
            const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
            const uint32_t by = (uint32_t)((e - s) * 4);
            asm volatile("fence.proxy.async.shared::cta;");
            mb_tx(&ws.mbar[b], by <= kCap * 4 ? by : 0);
            if (by <= kCap * 4 && by) bulk(ws.buf[b], ci + s, by, &ws.mbar[b]);
        }
    };
    uint32_t ph = 0;
    issue(0, 0);
    for (int j = 0; j < ntiles; j++) {
        const int b = j & 1;
        __syncwarp();
        if (j + 1 < ntiles) issue(j + 1, b ^ 1);
        const int64_t v = lo + 32ll * j + lane;
        int64_t s = 0, e = 0;
        if (v < hi) { s = rp[v]; e = rp[v + 1]; }
        const int64_t sal = __shfl_sync(~0u, s, 0) & ~3ll;
        mb_wait(&ws.mbar[b], (ph >> b) & 1);
        ph ^= 1u << b;
        if (MODE == 0) { if (v < hi) acc += ws.buf[b][s - sal]; continue; }
        if (v < hi) {
            const int32_t* x = ws.buf[b] + (s - sal);
            const int len = (int)(e - s);
            uint64_t m = T[v];
            for (int jj = 0; jj < len; jj += 16) {
                uint64_t tt[16];
#pragma unroll
                for (int q = 0; q < 16; q++) tt[q] = T[x[min(jj + q, len - 1)]];
#pragma unroll
                for (int q = 0; q < 16; q++) m = tt[q] < m ? tt[q] : m;
            }
            M[v] = (uint32_t)m;
        }
    }
    if (acc == 12345) sink[0] = acc;
}

int main(int argc, char** argv) {
    const int N = 100;
    const int64_t n = (int64_t)N * N * N;
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> ci;
    ci.reserve(27 * n);
    rp[0] = 0;
    for (int z = 0; z < N; z++) for (int y = 0; y < N; y++) for (int x = 0; x < N; x++) {
        for (int dz = -1; dz <= 1; dz++) for (int dy = -1; dy <= 1; dy++) for (int dx = -1; dx <= 1; dx++) {
            int a = x + dx, b = y + dy, c = z + dz;
            if (a < 0 || b < 0 || c < 0 || a >= N || b >= N || c >= N) continue;
            ci.push_back(a + N * (b + N * c));
        }
        rp[(x + N * (y + N * z)) + 1] = (int64_t)ci.size();
    }
    const int64_t nnz = ci.size();
    int64_t *d_rp; int32_t* d_ci; uint64_t* d_T; uint32_t* d_M; unsigned long long* d_s; char* flush;
    CK(cudaMalloc(&d_rp, 8 * (n + 1))); CK(cudaMalloc(&d_ci, 4 * nnz)); CK(cudaMalloc(&d_T, 8 * n)); CK(cudaMalloc(&d_M, 4 * n));
    CK(cudaMalloc(&d_s, 8)); CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemcpy(d_rp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_T, 0x11, 8 * n));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int smem = 8 * sizeof(WS);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name, int bps) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int grid = bps * sms;
        for (int cold = 0; cold < 2; cold++) {
            float best = 1e9;
            for (int rep = 0; rep < 5; rep++) {
                if (cold) CK(cudaMemset(flush, rep, 512 << 20));
                cudaEventRecord(a); kern<<<grid, 256, smem>>>(n, nnz, d_rp, d_ci, d_T, d_M, d_s); cudaEventRecord(b);
                CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            printf("%-40s blocks/SM=%d %s %8.2f us  colinds %.0f GB/s\n", name, bps, cold ? "cold" : "warm", best * 1e3, 4.0 * nnz / (best * 1e-3) / 1e9);
        }
    };
    for (int bps : {3, 4, 8}) run(kb<8>, "8 grid-stride int4 x4 stream", bps);
    // a 1 GiB read for calibration
    {
        int32_t* big; const int64_t nb = 256ll << 20;  // 1 GiB of int32
        CK(cudaMalloc(&big, 4 * nb)); CK(cudaMemset(big, 1, 4 * nb));
        for (int bps : {4, 8}) {
            float best = 1e9;
            for (int rep = 0; rep < 3; rep++) {
                cudaEventRecord(a); kb<8><<<bps * sms, 256, smem>>>(n, nb, d_rp, big, d_T, d_M, d_s); cudaEventRecord(b);
                CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            printf("1 GiB grid-stride read blocks/SM=%d %.1f us -> %.0f GB/s\n", bps, best * 1e3, 4.0 * nb / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
