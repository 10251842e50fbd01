// tools/mb_window.cu -- measurement aid (not product code): is the dense
// Refresh Column pass on the 27-point 100^3 graph bound by the T gathers
// through L1/L2, and how fast is it when the gathered words come from
// shared memory instead?
//   P   : pure stencil gathers from global (offsets computed, no colinds)
//   W1  : per 256-row step, the 9 (dy,dz) windows of T (258 words each) are
//         bulk-copied into shared memory one step ahead; the 27 gathers per
//         row are shared-memory loads (offsets computed, no colinds)
//   W2  : W1 + the step's colinds bulk-copied too; each entry is located in
//         its window by a per-step chunk table built from the colinds
//         (generic: 64-word chunks of T referenced by the step)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbwin tools/mb_window.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
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
constexpr int N = 100;

__global__ void __launch_bounds__(256) pg(int64_t n, const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nth) {
        const int x = v % N, y = (v / N) % N, z = v / (N * N);
        uint64_t m = kOUT;
        uint64_t tt[27];
#pragma unroll
        for (int q = 0; q < 27; q++) {
            const int dz = q / 9 - 1, dy = (q / 3) % 3 - 1, dx = q % 3 - 1;
            const bool in = x + dx >= 0 && x + dx < N && y + dy >= 0 && y + dy < N && z + dz >= 0 && z + dz < N;
            tt[q] = in ? T[v + dx + N * dy + N * N * dz] : kOUT;
        }
#pragma unroll
        for (int q = 0; q < 27; q++) m = tt[q] < m ? tt[q] : m;
        M[v] = (uint32_t)m & 0xfffff;
    }
}

// W1: block range of consecutive rows in 256-row steps; windows one step ahead
constexpr int kWin = 264;  // words per window slot (258 used + alignment)
struct W1Smem {
    uint64_t w[2][9][kWin];
    int64_t base[2][9];
    unsigned long long bar[2];
};
__device__ __forceinline__ void w1_issue(W1Smem& s, int slot, int64_t r0, int64_t n, const uint64_t* T) {
    uint32_t bytes = 0;
    int64_t bs[9], be[9];
    for (int k = 0; k < 9; k++) {
        const int dy = k % 3 - 1, dz = k / 3 - 1;
        int64_t a = r0 + N * dy + N * N * dz - 1, e = r0 + 256 + N * dy + N * N * dz + 1;
        a = a < 0 ? 0 : a;
        e = e > n ? n : e;
        a &= ~(int64_t)1;  // 16-byte aligned
        if (e <= a) e = a;
        e = (e + 1) & ~(int64_t)1;
        if (e > n) e = n & ~(int64_t)1;  // keep in bounds; the tail word is read from global below
        bs[k] = a;
        be[k] = e;
        bytes += (uint32_t)(e > a ? (e - a) * 8 : 0);
    }
    mb_tx(&s.bar[slot], bytes);
    for (int k = 0; k < 9; k++) {
        s.base[slot][k] = bs[k];
        if (be[k] > bs[k]) bulk(s.w[slot][k], T + bs[k], (uint32_t)((be[k] - bs[k]) * 8), &s.bar[slot]);
    }
}
__global__ void __launch_bounds__(256) w1(int64_t n, const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    extern __shared__ __align__(128) unsigned char raw[];
    W1Smem& s = *reinterpret_cast<W1Smem*>(raw);
    const int t = threadIdx.x;
    const int64_t B = gridDim.x;
    const int64_t blo = n * blockIdx.x / B, bhi = n * (blockIdx.x + 1) / B;
    const int64_t nsteps = (bhi - blo + 255) / 256;
    if (t == 0) {
        mb_init(&s.bar[0], 1);
        mb_init(&s.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nsteps > 0) w1_issue(s, 0, blo, n, T);
    }
    __syncthreads();
    uint32_t ph = 0;
    for (int64_t k = 0; k < nsteps; k++) {
        const int slot = (int)(k & 1);
        __syncthreads();
        if (t == 0 && k + 1 < nsteps) w1_issue(s, slot ^ 1, blo + (k + 1) * 256, n, T);
        const int64_t v = blo + k * 256 + t;
        mb_wait(&s.bar[slot], (ph >> slot) & 1u);
        ph ^= 1u << slot;
        if (v < bhi) {
            const int x = v % N, y = (v / N) % N, z = v / (N * N);
            uint64_t m = kOUT;
#pragma unroll
            for (int q = 0; q < 27; q++) {
                const int dz = q / 9 - 1, dy = (q / 3) % 3 - 1, dx = q % 3 - 1;
                const bool in = x + dx >= 0 && x + dx < N && y + dy >= 0 && y + dy < N && z + dz >= 0 && z + dz < N;
                if (in) {
                    const int64_t w = v + dx + N * dy + N * N * dz;
                    const int kk = (dz + 1) * 3 + (dy + 1);
                    const int64_t o = w - s.base[slot][kk];
                    const uint64_t tw = (o < kWin && w < (n & ~(int64_t)1)) ? s.w[slot][kk][o] : T[w];
                    m = tw < m ? tw : m;
                }
            }
            M[v] = (uint32_t)m & 0xfffff;
        }
    }
}

// W2: generic.  Per step the colinds span is bulk-copied (tile k+2), the
// distinct 64-word chunks of T it references are collected into a slot
// table (tile k+1, after its colinds arrived) and bulk-copied, and tile k is
// reduced from shared memory.  Chunk table: a per-step direct map from
// (chunk - cbase) to a slot over a span of kSpan chunks; a chunk outside the
// span or beyond the slot capacity is read from global.
constexpr int kRows = 256, kCiCap = kRows * 27 + 8, kChunk = 64, kSlots = 48, kSpan = 512;
struct W2Smem {
    int32_t ci[3][kCiCap];
    uint64_t tw[2][kSlots][kChunk];
    int16_t map[2][kSpan];
    int64_t cbase[2];
    int64_t sal[3];
    int32_t nslot[2];
    unsigned long long bci[3], btw[2];
};
__global__ void __launch_bounds__(256) w2(int64_t n, int64_t nnz, const int64_t* __restrict__ rp,
                                          const int32_t* __restrict__ ci, const uint64_t* __restrict__ T,
                                          uint32_t* __restrict__ M) {
    extern __shared__ __align__(128) unsigned char raw[];
    W2Smem& s = *reinterpret_cast<W2Smem*>(raw);
    const int t = threadIdx.x;
    const int64_t B = gridDim.x;
    const int64_t blo = n * blockIdx.x / B, bhi = n * (blockIdx.x + 1) / B;
    const int64_t nsteps = (bhi - blo + kRows - 1) / kRows;
    auto issue_ci = [&](int slot, int64_t k) {
        const int64_t r0 = blo + k * kRows, r1 = min(r0 + kRows, bhi);
        const int64_t a = rp[r0] & ~(int64_t)3, e = (rp[r1] + 3) & ~(int64_t)3;
        const int64_t ee = e > (nnz & ~(int64_t)3) ? (nnz & ~(int64_t)3) : e;
        s.sal[slot] = a;
        mb_tx(&s.bci[slot], (uint32_t)((ee - a) * 4));
        bulk(s.ci[slot], ci + a, (uint32_t)((ee - a) * 4), &s.bci[slot]);
    };
    if (t == 0) {
        for (int i = 0; i < 3; i++) mb_init(&s.bci[i], 1);
        for (int i = 0; i < 2; i++) mb_init(&s.btw[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // build the chunk table of step k (its colinds are in ci[k % 3]) and issue its T chunk copies
    auto build = [&](int64_t k) {
        const int cs = (int)(k % 3), ts = (int)(k & 1);
        const int64_t r0 = blo + k * kRows, r1 = min(r0 + kRows, bhi);
        const int64_t s0 = rp[r0], s1 = rp[r1];
        for (int i = t; i < kSpan; i += 256) s.map[ts][i] = -1;
        if (t == 0) {
            s.cbase[ts] = (r0 - N * N - 1) / kChunk;  // first chunk of the step's lowest neighbour (stencil hint)
            if (s.cbase[ts] < 0) s.cbase[ts] = 0;
            s.nslot[ts] = 0;
        }
        __syncthreads();
        const int64_t cb = s.cbase[ts];
        for (int64_t j = s0 + t; j < s1; j += 256) {
            const int64_t c = s.ci[cs][j - s.sal[cs]] / kChunk - cb;
            if (c >= 0 && c < kSpan && s.map[ts][c] < 0) s.map[ts][c] = 0x7fff;  // benign race: all write the flag
        }
        __syncthreads();
        if (t < 32) {  // warp 0 numbers the referenced chunks (ballot scan over the span)
            int base = 0;
            for (int i0 = 0; i0 < kSpan; i0 += 32) {
                const bool used = s.map[ts][i0 + t] == 0x7fff;
                const unsigned bal = __ballot_sync(0xffffffffu, used);
                const int idx = base + __popc(bal & ((1u << t) - 1));
                if (used) s.map[ts][i0 + t] = idx < kSlots ? (int16_t)idx : (int16_t)-1;
                base += __popc(bal);
            }
            if (t == 0) s.nslot[ts] = base < kSlots ? base : kSlots;
        }
        __syncthreads();
        if (t == 0) {
            uint32_t bytes = 0;
            for (int i = 0; i < kSpan; i++) {
                const int sl = s.map[ts][i];
                if (sl < 0) continue;
                int64_t a = (cb + i) * kChunk, e = a + kChunk;
                if (e > n) e = n & ~(int64_t)1;
                if (e > a) bytes += (uint32_t)((e - a) * 8);
            }
            mb_tx(&s.btw[ts], bytes);
            for (int i = 0; i < kSpan; i++) {
                const int sl = s.map[ts][i];
                if (sl < 0) continue;
                int64_t a = (cb + i) * kChunk, e = a + kChunk;
                if (e > n) e = n & ~(int64_t)1;
                if (e > a) bulk(s.tw[ts][sl], T + a, (uint32_t)((e - a) * 8), &s.btw[ts]);
            }
        }
    };
    uint32_t phc = 0, pht = 0;
    if (t == 0) {
        if (nsteps > 0) issue_ci(0, 0);
        if (nsteps > 1) issue_ci(1, 1);
    }
    if (nsteps > 0) {
        mb_wait(&s.bci[0], 0);
        phc ^= 1;
        build(0);
    }
    for (int64_t k = 0; k < nsteps; k++) {
        const int cs = (int)(k % 3), ts = (int)(k & 1);
        __syncthreads();
        if (t == 0 && k + 2 < nsteps) issue_ci((int)((k + 2) % 3), k + 2);
        if (k + 1 < nsteps) {  // next step's table while this step's T chunks land
            const int ns = (int)((k + 1) % 3);
            mb_wait(&s.bci[ns], (phc >> ns) & 1u);
            phc ^= 1u << ns;
            build(k + 1);
        }
        mb_wait(&s.btw[ts], (pht >> ts) & 1u);
        pht ^= 1u << ts;
        const int64_t v = blo + k * kRows + t;
        if (v < bhi) {
            const int64_t a = rp[v], e = rp[v + 1];
            const int64_t cb = s.cbase[ts];
            uint64_t m = kOUT;
            for (int64_t j = a; j < e; j++) {
                const int32_t w = s.ci[cs][j - s.sal[cs]];
                const int64_t c = w / kChunk - cb;
                const int sl = (c >= 0 && c < kSpan) ? s.map[ts][c] : -1;
                const uint64_t tw = (sl >= 0 && w < (n & ~(int64_t)1)) ? s.tw[ts][sl][w % kChunk] : T[w];
                m = tw < m ? tw : m;
            }
            M[v] = (uint32_t)m & 0xfffff;
        }
    }
}

int main() {
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
    int64_t* d_rp; int32_t* d_ci; uint64_t* d_T; uint32_t* d_M; char* flush;
    CK(cudaMalloc(&d_rp, 8 * (n + 1))); CK(cudaMalloc(&d_ci, 4 * nnz)); CK(cudaMalloc(&d_T, 8 * n)); CK(cudaMalloc(&d_M, 4 * n));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemcpy(d_rp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_T, T.data(), 8 * n, cudaMemcpyHostToDevice));
    std::vector<uint32_t> Mh(n), Md(n);
    for (int64_t v = 0; v < n; v++) {
        uint64_t m = kOUT;
        for (int64_t j = rp[v]; j < rp[v + 1]; j++) m = T[ci[j]] < m ? T[ci[j]] : m;
        Mh[v] = (uint32_t)m & 0xfffff;
    }
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name, int grid, int smem, auto launch) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem < 48 * 1024 ? 48 * 1024 : smem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
        float bw = 1e9, bc = 1e9;
        for (int cold = 0; cold < 2; cold++)
            for (int rep = 0; rep < 8; rep++) {
                if (cold) CK(cudaMemset(flush, rep, 512 << 20));
                CK(cudaMemset(d_M, 0, 4 * n));
                cudaEventRecord(a); launch(grid, smem); cudaEventRecord(b);
                CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) { if (cold) bc = ms < bc ? ms : bc; else bw = ms < bw ? ms : bw; }
            }
        CK(cudaMemcpy(Md.data(), d_M, 4 * n, cudaMemcpyDeviceToHost));
        int64_t bad = 0;
        for (int64_t v = 0; v < n; v++) bad += Md[v] != Mh[v];
        printf("%-24s grid %5d occ %d/SM smem %6d: warm %6.1f us cold %6.1f us  %s\n", name, grid, occ, smem, bw * 1e3, bc * 1e3,
               bad ? "WRONG" : "ok");
    };
    for (int per : {4, 8})
        run(pg, "P stencil u64", sms * per, 0, [&](int g, int sm) { pg<<<g, 256, sm>>>(n, d_T, d_M); });
    for (int per : {2, 4, 6})
        run(w1, "W1 smem windows", sms * per, (int)sizeof(W1Smem), [&](int g, int sm) { w1<<<g, 256, sm>>>(n, d_T, d_M); });
    for (int per : {1, 2, 3})
        run(w2, "W2 generic chunks", sms * per, (int)sizeof(W2Smem),
            [&](int g, int sm) { w2<<<g, 256, sm>>>(n, nnz, d_rp, d_ci, d_T, d_M); });
    return 0;
}
