// tools/mb_pool.cu -- measurement aid (not product code): does sharing the
// work of a dense Refresh Column pass between the blocks co-resident on one
// SM (a per-SM pool of 256-row tiles grabbed with an atomic, prefetched one
// tile ahead) beat the static assignment of tiles to blocks?  The youngest
// blocks of an SM finish a phase ~25% after the oldest (C2, measured), and
// then the SM runs with fewer warps.
//   S : static, block b takes tiles b, b + B, ...          (product layout)
//   P : pool,   SM k's blocks take tiles k, k + S, ... from a per-SM counter
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbpool tools/mb_pool.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_tx(unsigned long long* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_wait(unsigned long long* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}
constexpr uint64_t kOUT = ~0ull;
constexpr int ROWS = 256, CAP = ROWS * 27, B9 = 9;

__device__ void gbar(unsigned int* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = (blockIdx.x == 0) ? (0x80000000u - (gridDim.x - 1)) : 1u, old, cur;
        asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
        do { asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory"); } while (!((old ^ cur) & 0x80000000u));
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

struct Smem {
    int32_t buf[2][CAP + 8];
    unsigned long long bar[2];
    int64_t sal[2];
    int fits[2], tile[3];
    int pool, npools;
};

// ctr: [0] barrier, [1] pools registered, [64 + smid] blocks seen on smid, [1024 + smid] pool id + 1,
// [4096 + 32 * pool] next tile counter of the pool (pass p uses its own counter bank)
template <bool POOL>
__global__ void __launch_bounds__(256, 4) col(int64_t n, int64_t nnz, const int64_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci, const uint64_t* __restrict__ T,
                                              uint32_t* __restrict__ M, unsigned int* ctr, int passes) {
    extern __shared__ __align__(128) unsigned char raw[];
    Smem& s = *reinterpret_cast<Smem*>(raw);
    const int t = threadIdx.x;
    const int ntiles = (int)((n + ROWS - 1) / ROWS);
    if (t == 0) {
        mb_init(&s.bar[0], 1);
        mb_init(&s.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (POOL) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            if (atomicAdd(&ctr[64 + smid], 1u) == 0u) ctr[1024 + smid] = atomicAdd(&ctr[1], 1u) + 1u;
            s.pool = (int)smid;  // resolved to the pool id after the barrier
        }
    }
    gbar(&ctr[0]);
    if (POOL && t == 0) {
        s.pool = (int)(*(volatile unsigned int*)&ctr[1024 + s.pool]) - 1;
        s.npools = (int)*(volatile unsigned int*)&ctr[1];
    }
    __syncthreads();
    uint32_t ph = 0;
    for (int pass = 0; pass < passes; pass++) {
        unsigned int* pc = &ctr[4096 + 32 * (s.pool + 512 * (pass & 1))];
        auto tile_of = [&](int k) -> int {  // k-th tile of this block (static) / next pool tile (pool)
            if (!POOL) return (int)blockIdx.x + k * (int)gridDim.x;
            const unsigned i = atomicAdd(pc, 1u);
            return s.pool + (int)i * s.npools;
        };
        auto stage = [&](int slot, int tile) {
            if (tile >= ntiles) return;
            const int64_t r0 = (int64_t)ROWS * tile, r1 = min(r0 + ROWS, n);
            const int64_t a = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
            const bool f = (e - a) <= CAP && e <= (nnz & ~3ll);
            s.sal[slot] = a;
            s.fits[slot] = f;
            mb_tx(&s.bar[slot], f ? (uint32_t)((e - a) * 4) : 0u);
            if (f && e > a) bulk(s.buf[slot], ci + a, (uint32_t)((e - a) * 4), &s.bar[slot]);
        };
        if (t == 0) {
            s.tile[0] = tile_of(0);
            s.tile[1] = s.tile[0] < ntiles ? tile_of(1) : ntiles;
            stage(0, s.tile[0]);
        }
        __syncthreads();
        int64_t ns0 = 0, ne0 = 0;
        uint64_t ntv = kOUT;
        {
            const int64_t v0 = (int64_t)ROWS * s.tile[0] + t;
            if (s.tile[0] < ntiles && v0 < n) { ns0 = rp[v0]; ne0 = rp[v0 + 1]; ntv = T[v0]; }
        }
        for (int k = 0;; k++) {
            const int slot = k & 1;
            __syncthreads();
            const int tile = s.tile[k % 3], tnext = s.tile[(k + 1) % 3];
            if (tile >= ntiles) break;
            if (t == 0) {
                stage(slot ^ 1, tnext);
                s.tile[(k + 2) % 3] = tnext < ntiles ? tile_of(k + 2) : ntiles;
            }
            const int64_t v = (int64_t)ROWS * tile + t;
            const int64_t a = ns0, e = ne0;
            const uint64_t tv = ntv;
            if (tnext < ntiles) {
                const int64_t vn = (int64_t)ROWS * tnext + t;
                if (vn < n) { ns0 = rp[vn]; ne0 = rp[vn + 1]; ntv = T[vn]; }
            }
            mb_wait(&s.bar[slot], (ph >> slot) & 1u);
            ph ^= 1u << slot;
            if (v < n) {
                const int len = (int)(e - a);
                const int32_t* x = s.fits[slot] ? s.buf[slot] + (a - s.sal[slot]) : ci + a;
                uint64_t m = tv;
                const int last = len - 1;
                for (int j = 0; j < len; j += B9) {
                    uint64_t tt[B9];
#pragma unroll
                    for (int q = 0; q < B9; q++) tt[q] = T[x[min(j + q, last)]];
#pragma unroll
                    for (int q = 0; q < B9; q++) m = tt[q] < m ? tt[q] : m;
                }
                M[v] = (m == 0 || m == kOUT) ? 0xffffffffu : (uint32_t)m & 0xfffff;
            }
        }
        gbar(&ctr[0]);
        if (t == 0 && POOL) *(volatile unsigned int*)&ctr[4096 + 32 * (s.pool + 512 * ((pass + 1) & 1))] = 0u;
        gbar(&ctr[0]);
    }
}

int main() {
    const int N = 100;
    const int64_t n = (int64_t)N * N * N;
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> ci;
    ci.reserve(27 * n);
    for (int z = 0; z < N; z++) for (int y = 0; y < N; y++) for (int x = 0; x < N; x++) {
        for (int dz = -1; dz <= 1; dz++) for (int dy = -1; dy <= 1; dy++) for (int dx = -1; dx <= 1; dx++) {
            int a = x + dx, b = y + dy, c = z + dz;
            if (a < 0 || b < 0 || c < 0 || a >= N || b >= N || c >= N) continue;
            ci.push_back(a + N * (b + N * c));
        }
        rp[(x + N * (y + N * z)) + 1] = (int64_t)ci.size();
    }
    const int64_t nnz = ci.size();
    std::vector<uint64_t> T(n);
    uint64_t st = 88172645463325252ull;
    for (int64_t v = 0; v < n; v++) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; T[v] = (st & ~0xfffffull) | (uint64_t)(v + 1); }
    int64_t* d_rp; int32_t* d_ci; uint64_t* d_T; uint32_t* d_M; unsigned int* d_ctr;
    CK(cudaMalloc(&d_rp, 8 * (n + 1))); CK(cudaMalloc(&d_ci, 4 * nnz)); CK(cudaMalloc(&d_T, 8 * n)); CK(cudaMalloc(&d_M, 4 * n));
    CK(cudaMalloc(&d_ctr, 4 << 20));
    CK(cudaMemcpy(d_rp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_T, T.data(), 8 * n, cudaMemcpyHostToDevice));
    std::vector<uint32_t> Mh(n), Md(n);
    for (int64_t v = 0; v < n; v++) {
        uint64_t m = T[v];
        for (int64_t j = rp[v]; j < rp[v + 1]; j++) m = T[ci[j]] < m ? T[ci[j]] : m;
        Mh[v] = (uint32_t)m & 0xfffff;
    }
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name, int passes) {
        const int smem = (int)sizeof(Smem);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
        const int grid = occ * sms;
        float best = 1e9;
        for (int rep = 0; rep < 6; rep++) {
            CK(cudaMemset(d_ctr, 0, 4 << 20));
            CK(cudaMemset(d_M, 0, 4 * n));
            int p = passes;
            void* args[] = {(void*)&n, (void*)&nnz, &d_rp, &d_ci, &d_T, &d_M, &d_ctr, &p};
            cudaEventRecord(a);
            CK(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(256), args, smem, 0));
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
        }
        CK(cudaMemcpy(Md.data(), d_M, 4 * n, cudaMemcpyDeviceToHost));
        printf("%-10s grid %d (occ %d/SM) %d passes: %.1f us per pass  %s\n", name, grid, occ, passes, best * 1e3 / passes,
               Md == Mh ? "ok" : "WRONG");
    };
    for (int passes : {1, 10}) {
        run(col<false>, "static", passes);
        run(col<true>, "SM pool", passes);
    }
    return 0;
}
