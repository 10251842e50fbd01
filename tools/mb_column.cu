// tools/mb_column.cu -- measurement aid (not product code): one dense
// Refresh Column pass (M_v = id field of min T over N[v]) on the 27-point
// 100^3 graph, in several kernel organisations, to find what bounds it.
//   V1 direct   : thread per row, colinds and T straight from global (no smem)
//   V2 warpring : per-warp ring of S slots, each slot = colinds of 32 rows,
//                 filled by the bulk-copy engine (lane 0, mbarrier), S-1 ahead
//   V3 blockbuf : current product organisation (block tile of 256 rows,
//                 bulk copy one tile ahead, __syncthreads per step)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbcol tools/mb_column.cu
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
__device__ __forceinline__ uint32_t mfield(uint64_t m) { return (m == 0 || m == kOUT) ? 0xffffffffu : (uint32_t)m & 0xfffff; }

template <int B>
__device__ __forceinline__ uint64_t rowmin(const uint64_t* __restrict__ T, const int32_t* x, int len, uint64_t m) {
    const int last = len - 1;
    for (int j = 0; j < len; j += B) {
        uint64_t tt[B];
#pragma unroll
        for (int q = 0; q < B; q++) tt[q] = T[x[min(j + q, last)]];
#pragma unroll
        for (int q = 0; q < B; q++) m = tt[q] < m ? tt[q] : m;
    }
    return m;
}

template <int B, int G>
__device__ __forceinline__ uint64_t rowmin_g(const uint64_t* __restrict__ T, const int32_t* x, int len, int sub, uint64_t m) {
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint64_t tt[B];
#pragma unroll
        for (int q = 0; q < B; q++) tt[q] = T[x[min(j + q * G, last)]];
#pragma unroll
        for (int q = 0; q < B; q++) m = tt[q] < m ? tt[q] : m;
    }
    return m;
}

// V1: thread per row, grid-stride over rows in warp-contiguous chunks
template <int B>
__global__ void __launch_bounds__(256) v1(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nth) {
        const int64_t s = rp[v], e = rp[v + 1];
        const uint64_t m = rowmin<B>(T, ci + s, (int)(e - s), T[v]);
        M[v] = mfield(m);
    }
}

// V2: per-warp ring of S slots of 32 rows
constexpr int kSlotCap = 32 * 27 + 8;
template <int S, int B>
__global__ void __launch_bounds__(256) v2(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    extern __shared__ __align__(16) unsigned char raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    int32_t* buf = reinterpret_cast<int32_t*>(raw) + (size_t)warp * S * kSlotCap;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(reinterpret_cast<int32_t*>(raw) + (size_t)nw * S * kSlotCap) + warp * S;
    const int64_t W = (int64_t)gridDim.x * nw, gw = (int64_t)blockIdx.x * nw + warp;
    const int64_t lo = n * gw / W, hi = n * (gw + 1) / W;
    const int ntiles = (int)((hi - lo + 31) / 32);
    if (lane == 0) {
        for (int i = 0; i < S; i++) mb_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // lane r holds rp[lo + 32 j + r] for the tile being issued; lane 0 issues
    auto issue = [&](int j) {
        const int slot = j % S;
        const int64_t r0 = lo + 32ll * j, r1 = min(r0 + 32, hi);
        const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
        if (lane == 0) {
            uint32_t by = (uint32_t)((e - s) * 4);
            if (by > kSlotCap * 4 || e > (nnz & ~3ll)) by = 0;
            mb_tx(&bar[slot], by);
            if (by) bulk(buf + slot * kSlotCap, ci + s, by, &bar[slot]);
        }
    };
    for (int j = 0; j < S - 1 && j < ntiles; j++) issue(j);
    for (int j = 0; j < ntiles; j++) {
        const int slot = j % S;
        const int64_t v = lo + 32ll * j + lane;
        int64_t s = 0, e = 0;
        uint64_t tv = kOUT;
        if (v < hi) { s = rp[v]; e = rp[v + 1]; tv = T[v]; }
        const int64_t s0 = __shfl_sync(~0u, s, 0);
        const int64_t sal = s0 & ~3ll;
        const int64_t e31 = __shfl_sync(~0u, e, 31);
        const bool fits = (((e31 + 3) & ~3ll) - sal) <= kSlotCap && ((e31 + 3) & ~3ll) <= (nnz & ~3ll);
        mb_wait(&bar[slot], (j / S) & 1);
        if (v < hi) {
            const int32_t* x = fits ? buf + slot * kSlotCap + (s - sal) : ci + s;
            M[v] = mfield(rowmin<B>(T, x, (int)(e - s), tv));
        }
        __syncwarp();
        if (j + S - 1 < ntiles) issue(j + S - 1);
    }
}

// V3: the product's organisation (block tile of ROWS rows, bulk copy one
// tile ahead, __syncthreads per step), G = 256 / ROWS lanes per row
template <int G>
__device__ __forceinline__ uint64_t gmin(uint64_t x) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) { uint64_t y = __shfl_xor_sync(~0u, x, o); x = y < x ? y : x; }
    return x;
}
template <int ROWS, int B>
__global__ void __launch_bounds__(256) v3(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    constexpr int G = 256 / ROWS, CAP = ROWS * 27;
    extern __shared__ __align__(16) unsigned char raw[];
    int32_t (*buf)[CAP + 8] = reinterpret_cast<int32_t (*)[CAP + 8]>(raw);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 2 * (CAP + 8) * 4);
    int64_t* sal_s = reinterpret_cast<int64_t*>(bar + 2);
    int* fits_s = reinterpret_cast<int*>(sal_s + 2);
    const int t = threadIdx.x, g = t / G, sub = t % G;
    const int64_t Bn = gridDim.x, blo = n * blockIdx.x / Bn, bhi = n * (blockIdx.x + 1) / Bn;
    const int64_t nsteps = (bhi - blo + ROWS - 1) / ROWS;
    if (t == 0) { mb_init(&bar[0], 1); mb_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    auto stage = [&](int slot, int64_t k) {
        const int64_t r0 = blo + ROWS * k, r1 = min(r0 + ROWS, bhi);
        const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
        const bool f = (e - s) <= CAP && e <= (nnz & ~3ll);
        sal_s[slot] = s; fits_s[slot] = f;
        mb_tx(&bar[slot], f ? (uint32_t)((e - s) * 4) : 0u);
        if (f && e > s) bulk(buf[slot], ci + s, (uint32_t)((e - s) * 4), &bar[slot]);
    };
    if (t == 0 && nsteps > 0) stage(0, 0);
    uint32_t ph = 0;
    for (int64_t k = 0; k < nsteps; k++) {
        const int slot = (int)(k & 1);
        __syncthreads();
        if (t == 0 && k + 1 < nsteps) stage(slot ^ 1, k + 1);
        const int64_t v = blo + ROWS * k + g;
        int64_t s = 0, e = 0; uint64_t tv = kOUT;
        if (v < bhi) { s = rp[v]; e = rp[v + 1]; if (sub == 0) tv = T[v]; }
        mb_wait(&bar[slot], (ph >> slot) & 1); ph ^= 1u << slot;
        uint64_t m = tv;
        if (v < bhi) {
            const int len = (int)(e - s);
            if (fits_s[slot]) m = rowmin_g<B, G>(T, buf[slot] + (s - sal_s[slot]), len, sub, m);
            else m = rowmin_g<B, G>(T, ci + s, len, sub, m);
        }
        m = gmin<G>(m);
        if (v < bhi && sub == 0) M[v] = mfield(m);
    }
}

// V4: warp-specialised pipeline.  Warp 8 (producer, lane 0) stages per tile
// the rowptr slice, the T slice of the tile's own rows and the colinds span
// into a ring of S stages (bulk copies, one full mbarrier per stage); the 8
// consumer warps read everything but the neighbour gathers from shared
// memory and release the stage on an empty mbarrier (one arrival per warp).
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
template <int ROWS, int S, int B>
struct V4Cfg {
    static constexpr int G = 256 / ROWS;
    static constexpr int CAP = ROWS * 27 + 8;                   // int32 colinds per stage
    static constexpr int RPW = ROWS + 4;                        // int64 rowptr per stage
    static constexpr int STAGE = CAP * 4 + RPW * 8 + (ROWS + 2) * 8;  // bytes
    static constexpr int SMEM = S * STAGE + 2 * S * 8 + 64;
};
template <int ROWS, int S, int B>
__global__ void __launch_bounds__(288) v4(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    using C = V4Cfg<ROWS, S, B>;
    constexpr int G = C::G;
    extern __shared__ __align__(128) unsigned char raw[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(raw + S * C::STAGE);
    unsigned long long* empty = full + S;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int64_t Bn = gridDim.x, blo = n * blockIdx.x / Bn, bhi = n * (blockIdx.x + 1) / Bn;
    const int nsteps = (int)((bhi - blo + ROWS - 1) / ROWS);
    if (t == 0) {
        for (int i = 0; i < S; i++) { mb_init(&full[i], 1); mb_init(&empty[i], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto stage_ptr = [&](int st) { return raw + st * C::STAGE; };
    if (warp == 8) {
        if (lane != 0) return;
        for (int k = 0; k < nsteps; k++) {
            const int st = k % S;
            if (k >= S) mb_wait(&empty[st], ((k / S) - 1) & 1);
            const int64_t r0 = blo + (int64_t)ROWS * k, r1 = min(r0 + ROWS, bhi);
            unsigned char* p = stage_ptr(st);
            int32_t* cbuf = reinterpret_cast<int32_t*>(p);
            int64_t* rbuf = reinterpret_cast<int64_t*>(p + C::CAP * 4);
            uint64_t* tbuf = reinterpret_cast<uint64_t*>(p + C::CAP * 4 + C::RPW * 8);
            const int64_t cs = rp[r0], ce = rp[r1];
            const int64_t sal = cs & ~3ll, eal = (ce + 3) & ~3ll;
            const bool fits = (eal - sal) <= C::CAP && eal <= (nnz & ~3ll);
            const int64_t ra = r0 & ~1ll, rb = (r1 + 1 + 1) & ~1ll;   // rowptr[r0 .. r1] (16 B hull)
            const int64_t ta = r0 & ~1ll, tb = (r1 + 1) & ~1ll;       // T[r0 .. r1)
            uint32_t bytes = (uint32_t)((rb - ra) * 8 + (tb - ta) * 8) + (fits ? (uint32_t)((eal - sal) * 4) : 0u);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(bytes) : "memory");
            bulk(rbuf, rp + ra, (uint32_t)((rb - ra) * 8), &full[st]);
            bulk(tbuf, T + ta, (uint32_t)((tb - ta) * 8), &full[st]);
            if (fits && eal > sal) bulk(cbuf, ci + sal, (uint32_t)((eal - sal) * 4), &full[st]);
        }
        return;
    }
    const int g = t / G, sub = t % G;
    for (int k = 0; k < nsteps; k++) {
        const int st = k % S;
        const int64_t r0 = blo + (int64_t)ROWS * k;
        mb_wait(&full[st], (k / S) & 1);
        const unsigned char* p = stage_ptr(st);
        const int32_t* cbuf = reinterpret_cast<const int32_t*>(p);
        const int64_t* rbuf = reinterpret_cast<const int64_t*>(p + C::CAP * 4);
        const uint64_t* tbuf = reinterpret_cast<const uint64_t*>(p + C::CAP * 4 + C::RPW * 8);
        const int64_t v = r0 + g;
        const int64_t ra = r0 & ~1ll;
        uint64_t m = kOUT;
        int64_t s = 0, e = 0;
        if (v < bhi) {
            s = rbuf[v - ra];
            e = rbuf[v - ra + 1];
            if (sub == 0) m = tbuf[v - ra];
        }
        const int64_t cs = rbuf[r0 - ra];
        const int64_t rend = min(r0 + ROWS, bhi);
        const int64_t ce = rbuf[rend - ra];
        const int64_t sal = cs & ~3ll, eal = (ce + 3) & ~3ll;
        const bool fits = (eal - sal) <= C::CAP && eal <= (nnz & ~3ll);
        if (v < bhi) {
            const int len = (int)(e - s);
            if (fits) m = rowmin_g<B, G>(T, cbuf + (s - sal), len, sub, m);
            else m = rowmin_g<B, G>(T, ci + s, len, sub, m);
        }
        m = gmin<G>(m);
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[st]);
        if (v < bhi && sub == 0) M[v] = mfield(m);
    }
}

// P: pure gathers without colinds: 27 stencil offsets computed arithmetically
template <typename W, int MODE>
__global__ void __launch_bounds__(256) pg(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T8, uint32_t* __restrict__ M) {
    const W* T = reinterpret_cast<const W*>(T8);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nth) {
        W m = T[v];
        W tt[27];
#pragma unroll
        for (int q = 0; q < 27; q++) {
            const int dz = q / 9 - 1, dy = (q / 3) % 3 - 1, dx = q % 3 - 1;
            int64_t w = MODE == 0 ? v + dx + 100 * dy + 10000 * dz
                      : MODE == 1 ? v + dx
                      : MODE == 2 ? v + dx + 100 * dy + 100 * dz          // all within the block
                      : MODE == 3 ? v + 4099 * (q - 13)                   // 27 distinct far lines
                      : (v * 27 + q * 40961) % n;                         // scattered
            w = w < 0 ? 0 : (w >= n ? n - 1 : w);
            tt[q] = T[w];
        }
#pragma unroll
        for (int q = 0; q < 27; q++) m = tt[q] < m ? tt[q] : m;
        M[v] = (uint32_t)m;
    }
}

// V5: V3 (256 rows, G = 1) + the push-form Decide work.  OUT rows = rows
// whose min T is below a threshold (about frac of them).  MODE bit 1: count
// for the argmin with plain RED; bit 2: count with match_any aggregation;
// bit 4: push OUT rows thread-per-row (27 byte stores per thread); bit 8:
// warp-cooperative push; bit 16: 4-byte keys instead of 8-byte T gathers.
__device__ uint8_t* g_oflag;
__device__ uint32_t* g_cnt;
__device__ uint32_t* g_K;
__device__ uint64_t g_thresh;
template <int MODE>
__global__ void __launch_bounds__(256) v5(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    constexpr int ROWS = 256, CAP = ROWS * 27;
    extern __shared__ __align__(16) unsigned char raw[];
    int32_t (*buf)[CAP + 8] = reinterpret_cast<int32_t (*)[CAP + 8]>(raw);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 2 * (CAP + 8) * 4);
    int64_t* sal_s = reinterpret_cast<int64_t*>(bar + 2);
    int* fits_s = reinterpret_cast<int*>(sal_s + 2);
    uint8_t* oflag = g_oflag;
    uint32_t* cnt = g_cnt;
    const uint32_t* K = g_K;
    const uint64_t thr = g_thresh;
    const int t = threadIdx.x, lane = t & 31;
    const int64_t Bn = gridDim.x, blo = n * blockIdx.x / Bn, bhi = n * (blockIdx.x + 1) / Bn;
    const int64_t nsteps = (bhi - blo + ROWS - 1) / ROWS;
    if (t == 0) { mb_init(&bar[0], 1); mb_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    auto stage = [&](int slot, int64_t k) {
        const int64_t r0 = blo + ROWS * k, r1 = min(r0 + ROWS, bhi);
        const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
        const bool f = (e - s) <= CAP && e <= (nnz & ~3ll);
        sal_s[slot] = s; fits_s[slot] = f;
        mb_tx(&bar[slot], f ? (uint32_t)((e - s) * 4) : 0u);
        if (f && e > s) bulk(buf[slot], ci + s, (uint32_t)((e - s) * 4), &bar[slot]);
    };
    if (t == 0 && nsteps > 0) stage(0, 0);
    uint32_t ph = 0;
    for (int64_t k = 0; k < nsteps; k++) {
        const int slot = (int)(k & 1);
        __syncthreads();
        if (t == 0 && k + 1 < nsteps) stage(slot ^ 1, k + 1);
        const int64_t v = blo + ROWS * k + t;
        int64_t s = 0, e = 0; uint64_t tv = kOUT;
        if (v < bhi) { s = rp[v]; e = rp[v + 1]; tv = T[v]; }
        mb_wait(&bar[slot], (ph >> slot) & 1); ph ^= 1u << slot;
        uint64_t m = tv;
        uint32_t kmin = (uint32_t)(tv >> 32), wmin = (uint32_t)v;
        const int32_t* x = buf[slot] + (s - sal_s[slot]);
        const int len = (int)(e - s);
        if (v < bhi && fits_s[slot]) {
            if (MODE & 16) {
                const int last = len - 1;
                for (int j = 0; j < len; j += 16) {
                    uint32_t kk[16]; int ww[16];
#pragma unroll
                    for (int q = 0; q < 16; q++) { ww[q] = x[min(j + q, last)]; kk[q] = K[ww[q]]; }
#pragma unroll
                    for (int q = 0; q < 16; q++) {
                        const bool lt = kk[q] < kmin || (kk[q] == kmin && (uint32_t)ww[q] < wmin);
                        kmin = lt ? kk[q] : kmin; wmin = lt ? ww[q] : wmin;
                    }
                }
                m = ((uint64_t)kmin << 32) | (wmin + 1);
            } else {
                m = rowmin_g<16, 1>(T, x, len, 0, m);
            }
        }
        const bool act = v < bhi && fits_s[slot];
        const bool out = act && m < thr;
        const uint32_t a = (uint32_t)m & 0xfffff;
        if (MODE & 2) {
            const bool c = act && !out;
            const uint32_t key = c ? a : (0x80000000u | lane);
            const unsigned grp = __match_any_sync(~0u, key);
            if (c && lane == __ffs(grp) - 1) atomicAdd(&cnt[a & 0xfffff], (uint32_t)__popc(grp));
        } else if (MODE & 1) {
            if (act && !out) atomicAdd(&cnt[a & 0xfffff], 1u);
        }
        if (MODE & 4) {
            if (out) for (int j = 0; j < len; j++) oflag[x[j]] = 1;
        } else if (MODE & 8) {
            unsigned bal = __ballot_sync(~0u, out);
            while (bal) {
                const int l = __ffs(bal) - 1; bal &= bal - 1;
                const int32_t* xr = reinterpret_cast<const int32_t*>(__shfl_sync(~0u, reinterpret_cast<unsigned long long>(x), l));
                const int lr = __shfl_sync(~0u, len, l);
                if (lane < lr) oflag[xr[lane]] = 1;
            }
        }
        if (v < bhi) M[v] = mfield(m);
    }
}

// V6: sparse column pass over a sorted worklist (random subset of rows),
// G lanes per row, colinds straight from global, B gathers in flight per lane
__device__ const int32_t* g_wl;
__device__ int64_t g_nwl;
template <int G, int B>
__global__ void __launch_bounds__(256) v6(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    const int32_t* wl = g_wl;
    const int64_t nwl = g_nwl;
    const int sub = threadIdx.x % G;
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G, ng = (int64_t)gridDim.x * blockDim.x / G;
    // contiguous chunk of the worklist per group-slot: rows i*ng + gid (interleaved)
    const int64_t iters = (nwl + ng - 1) / ng;
    for (int64_t it = 0; it < iters; it++) {
        const int64_t idx = it * ng + gid;
        uint64_t m = kOUT;
        int64_t v = -1;
        if (idx < nwl) {
            v = wl[idx];
            const int64_t s = rp[v], e = rp[v + 1];
            if (sub == 0) m = T[v];
            m = rowmin_g<B, G>(T, ci + s, (int)(e - s), sub, m);
        }
        m = gmin<G>(m);
        if (v >= 0 && sub == 0) M[v] = mfield(m);
    }
}

// V7: V3 (256-row tiles, G = 1, bulk copy one tile ahead) with tiles
// grabbed dynamically from a global counter instead of static block ranges
__device__ unsigned int* g_ctr;
template <int B>
__global__ void __launch_bounds__(256) v7(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    constexpr int ROWS = 256, CAP = ROWS * 27;
    extern __shared__ __align__(16) unsigned char raw[];
    int32_t (*buf)[CAP + 8] = reinterpret_cast<int32_t (*)[CAP + 8]>(raw);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 2 * (CAP + 8) * 4);
    int64_t* sal_s = reinterpret_cast<int64_t*>(bar + 2);
    int* fits_s = reinterpret_cast<int*>(sal_s + 2);
    int* tile_s = reinterpret_cast<int*>(fits_s + 2);
    unsigned int* ctr = g_ctr;
    const int t = threadIdx.x;
    const int ntiles = (int)((n + ROWS - 1) / ROWS);
    if (t == 0) { mb_init(&bar[0], 1); mb_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    auto stage = [&](int slot, int tile) {
        tile_s[slot] = tile;
        if (tile >= ntiles) return;
        const int64_t r0 = (int64_t)ROWS * tile, r1 = min(r0 + ROWS, n);
        const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
        const bool f = (e - s) <= CAP && e <= (nnz & ~3ll);
        sal_s[slot] = s; fits_s[slot] = f;
        mb_tx(&bar[slot], f ? (uint32_t)((e - s) * 4) : 0u);
        if (f && e > s) bulk(buf[slot], ci + s, (uint32_t)((e - s) * 4), &bar[slot]);
    };
    int next = 0;
    if (t == 0) { stage(0, (int)atomicAdd(ctr, 1u)); next = (int)atomicAdd(ctr, 1u); }
    __syncthreads();
    uint32_t ph = 0;
    for (int k = 0;; k++) {
        const int slot = k & 1;
        const int tile = tile_s[slot];
        if (tile >= ntiles) break;
        __syncthreads();
        if (t == 0) { stage(slot ^ 1, next); if (next < ntiles) next = (int)atomicAdd(ctr, 1u); }
        const int64_t v = (int64_t)ROWS * tile + t;
        int64_t s = 0, e = 0; uint64_t tv = kOUT;
        if (v < n) { s = rp[v]; e = rp[v + 1]; tv = T[v]; }
        mb_wait(&bar[slot], (ph >> slot) & 1); ph ^= 1u << slot;
        uint64_t m = tv;
        if (v < n) {
            const int len = (int)(e - s);
            if (fits_s[slot]) m = rowmin_g<B, 1>(T, buf[slot] + (s - sal_s[slot]), len, 0, m);
            else m = rowmin_g<B, 1>(T, ci + s, len, 0, m);
            M[v] = mfield(m);
        }
        __syncthreads();
    }
}

// V8: V3 (256 rows, G = 1) gathering 4-byte keys K_w (top 32 bits of T_w)
// with B gathers in flight; min over (K_w, w) and a tie flag
template <int B>
__global__ void __launch_bounds__(256) v8(int64_t n, int64_t nnz, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const uint64_t* __restrict__ T, uint32_t* __restrict__ M) {
    constexpr int ROWS = 256, CAP = ROWS * 27;
    extern __shared__ __align__(16) unsigned char raw[];
    int32_t (*buf)[CAP + 8] = reinterpret_cast<int32_t (*)[CAP + 8]>(raw);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 2 * (CAP + 8) * 4);
    int64_t* sal_s = reinterpret_cast<int64_t*>(bar + 2);
    int* fits_s = reinterpret_cast<int*>(sal_s + 2);
    const uint32_t* __restrict__ K = g_K;
    const int t = threadIdx.x;
    const int64_t Bn = gridDim.x, blo = n * blockIdx.x / Bn, bhi = n * (blockIdx.x + 1) / Bn;
    const int64_t nsteps = (bhi - blo + ROWS - 1) / ROWS;
    if (t == 0) { mb_init(&bar[0], 1); mb_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    auto stage = [&](int slot, int64_t k) {
        const int64_t r0 = blo + ROWS * k, r1 = min(r0 + ROWS, bhi);
        const int64_t s = rp[r0] & ~3ll, e = (rp[r1] + 3) & ~3ll;
        const bool f = (e - s) <= CAP && e <= (nnz & ~3ll);
        sal_s[slot] = s; fits_s[slot] = f;
        mb_tx(&bar[slot], f ? (uint32_t)((e - s) * 4) : 0u);
        if (f && e > s) bulk(buf[slot], ci + s, (uint32_t)((e - s) * 4), &bar[slot]);
    };
    if (t == 0 && nsteps > 0) stage(0, 0);
    uint32_t ph = 0;
    for (int64_t k = 0; k < nsteps; k++) {
        const int slot = (int)(k & 1);
        __syncthreads();
        if (t == 0 && k + 1 < nsteps) stage(slot ^ 1, k + 1);
        const int64_t v = blo + ROWS * k + t;
        int64_t s = 0, e = 0; uint32_t kv = 0xffffffffu;
        if (v < bhi) { s = rp[v]; e = rp[v + 1]; kv = K[v]; }
        mb_wait(&bar[slot], (ph >> slot) & 1); ph ^= 1u << slot;
        if (v < bhi && fits_s[slot]) {
            const int32_t* x = buf[slot] + (s - sal_s[slot]);
            const int len = (int)(e - s), last = len - 1;
            uint32_t kmin = kv, wmin = (uint32_t)v;
            bool tie = false;
            for (int j = 0; j < len; j += B) {
                uint32_t kk[B];
#pragma unroll
                for (int q = 0; q < B; q++) kk[q] = K[x[min(j + q, last)]];
#pragma unroll
                for (int q = 0; q < B; q++) {
                    const uint32_t w = (uint32_t)x[min(j + q, last)];
                    const bool lt = kk[q] < kmin;
                    tie = lt ? false : (tie | (kk[q] == kmin && w != wmin));
                    kmin = lt ? kk[q] : kmin;
                    wmin = lt ? w : wmin;
                }
            }
            M[v] = tie ? 0xfffffffeu : ((kmin == 0u || kmin == 0xffffffffu) ? 0xffffffffu : ((wmin + 1) & 0xfffff));
        }
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
    int64_t* d_rp; int32_t* d_ci; uint64_t* d_T; uint32_t* d_M; char* flush;
    CK(cudaMalloc(&d_rp, 8 * (n + 1))); CK(cudaMalloc(&d_ci, 4 * nnz)); CK(cudaMalloc(&d_T, 8 * n)); CK(cudaMalloc(&d_M, 4 * n));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemcpy(d_rp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_T, T.data(), 8 * n, cudaMemcpyHostToDevice));
    // expected M on the host
    std::vector<uint32_t> Mh(n), Md(n);
    for (int64_t v = 0; v < n; v++) {
        uint64_t m = T[v];
        for (int64_t j = rp[v]; j < rp[v + 1]; j++) m = T[ci[j]] < m ? T[ci[j]] : m;
        Mh[v] = (uint32_t)m & 0xfffff;
    }
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const double alg = 4.0 * nnz + 8.0 * n * 2 + 4.0 * n + 8.0 * n;  // colinds + rowptr + M + T (once)
    auto run = [&](auto kern, const char* name, int grid, int block, int smem) {
        if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        {   // smallest carveout that holds grid/SM blocks (the rest is L1)
            const int per = (grid + sms - 1) / sms;
            int pct = (int)((double)(per * (smem + 1024)) * 100.0 / (228.0 * 1024) + 0.999);
            if (pct > 100) pct = 100;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        }
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
        float bc = 1e9, bw = 1e9;
        for (int cold = 0; cold < 2; cold++)
            for (int rep = 0; rep < 6; rep++) {
                if (cold) CK(cudaMemset(flush, rep, 512 << 20));
                CK(cudaMemset(d_M, 0, 4 * n));
                cudaEventRecord(a); kern<<<grid, block, smem>>>(n, nnz, d_rp, d_ci, d_T, d_M); cudaEventRecord(b);
                CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) { if (cold) bc = ms < bc ? ms : bc; else bw = ms < bw ? ms : bw; }
            }
        CK(cudaMemcpy(Md.data(), d_M, 4 * n, cudaMemcpyDeviceToHost));
        bool ok = Md == Mh || name[0] == 'P' || name[1] == '6' || name[1] == '8';
        printf("%-28s grid %5d occ %d/SM: warm %6.1f us  cold %6.1f us  (alg %.0f GB/s cold) %s\n", name, grid, occ, bw * 1e3, bc * 1e3,
               alg / (bc * 1e-3) / 1e9, ok ? "ok" : "WRONG");
    };
    for (int per : {4, 8}) {
        run(pg<uint64_t, 0>, "P stencil gathers u64", sms * per, 256, 0);
        run(pg<uint32_t, 0>, "P stencil gathers u32", sms * per, 256, 0);
        run(pg<uint64_t, 1>, "P same-line gathers u64", sms * per, 256, 0);
        run(pg<uint64_t, 2>, "P in-block gathers u64", sms * per, 256, 0);
        run(pg<uint64_t, 3>, "P far-line gathers u64", sms * per, 256, 0);
        run(pg<uint32_t, 3>, "P far-line gathers u32", sms * per, 256, 0);
        run(pg<uint64_t, 4>, "P scattered gathers u64", sms * per, 256, 0);
    }
    for (int per : {4, 8}) run(v1<16>, "V1 direct B16", sms * per, 256, 0);
    run(v1<8>, "V1 direct B8", sms * 8, 256, 0);
    run(v1<27>, "V1 direct B27", sms * 4, 256, 0);
    for (int per : {2, 4}) {
        run(v2<2, 16>, "V2 warpring S2 B16", sms * per, 256, 8 * (2 * kSlotCap * 4 + 16 * 2));
        run(v2<3, 16>, "V2 warpring S3 B16", sms * per, 256, 8 * (3 * kSlotCap * 4 + 16 * 3));
        run(v2<4, 16>, "V2 warpring S4 B16", sms * per, 256, 8 * (4 * kSlotCap * 4 + 16 * 4));
    }
    run(v2<3, 27>, "V2 warpring S3 B27", sms * 2, 256, 8 * (3 * kSlotCap * 4 + 16 * 3));
    auto v3s = [](int rows) { return 2 * (rows * 27 + 8) * 4 + 64; };
    for (int per : {3, 4}) run(v3<256, 16>, "V3 256 rows B16", sms * per, 256, v3s(256));
    for (int per : {4, 6, 8}) run(v3<128, 16>, "V3 128 rows B16 (G2)", sms * per, 256, v3s(128));
    for (int per : {4, 6, 8}) run(v3<128, 8>, "V3 128 rows B8 (G2)", sms * per, 256, v3s(128));
    for (int per : {4, 8}) run(v3<64, 8>, "V3 64 rows B8 (G4)", sms * per, 256, v3s(64));
    for (int per : {4, 8}) run(v3<64, 4>, "V3 64 rows B4 (G4)", sms * per, 256, v3s(64));
    run(v4<256, 2, 16>, "V4 256 S2 B16", sms * 2, 288, V4Cfg<256, 2, 16>::SMEM);
    run(v4<256, 3, 16>, "V4 256 S3 B16", sms * 2, 288, V4Cfg<256, 3, 16>::SMEM);
    run(v4<128, 3, 16>, "V4 128 S3 B16", sms * 3, 288, V4Cfg<128, 3, 16>::SMEM);
    run(v4<128, 4, 16>, "V4 128 S4 B16", sms * 3, 288, V4Cfg<128, 4, 16>::SMEM);
    run(v4<128, 3, 16>, "V4 128 S3 B16 4/SM", sms * 4, 288, V4Cfg<128, 3, 16>::SMEM);
    run(v4<128, 2, 16>, "V4 128 S2 B16 4/SM", sms * 4, 288, V4Cfg<128, 2, 16>::SMEM);
    run(v4<64, 4, 8>, "V4 64 S4 B8", sms * 6, 288, V4Cfg<64, 4, 8>::SMEM);
    run(v4<64, 3, 8>, "V4 64 S3 B8", sms * 7, 288, V4Cfg<64, 3, 8>::SMEM);
    {
        uint8_t* of; uint32_t* cn; uint32_t* Kd;
        CK(cudaMalloc(&of, n)); CK(cudaMalloc(&cn, 4 * n)); CK(cudaMalloc(&Kd, 4 * n));
        CK(cudaMemset(of, 0, n)); CK(cudaMemset(cn, 0, 4 * n));
        std::vector<uint32_t> Kh(n);
        for (int64_t v = 0; v < n; v++) Kh[v] = (uint32_t)(T[v] >> 32);
        CK(cudaMemcpy(Kd, Kh.data(), 4 * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpyToSymbol(g_oflag, &of, sizeof(of))); CK(cudaMemcpyToSymbol(g_cnt, &cn, sizeof(cn)));
        CK(cudaMemcpyToSymbol(g_K, &Kd, sizeof(Kd)));
        const int V5S = 2 * (256 * 27 + 8) * 4 + 64;
        for (double frac : {0.0, 0.2}) {
            // threshold so that about frac of the row minima fall below it
            std::vector<uint64_t> mins(n);
            for (int64_t v = 0; v < n; v++) { uint64_t m = T[v]; for (int64_t j = rp[v]; j < rp[v + 1]; j++) m = std::min(m, T[ci[j]]); mins[v] = m; }
            std::sort(mins.begin(), mins.end());
            uint64_t thr = frac > 0 ? mins[(size_t)(frac * n)] : 0;
            CK(cudaMemcpyToSymbol(g_thresh, &thr, sizeof(thr)));
            printf("-- OUT fraction %.2f\n", frac);
            run(v5<0>, "V5 base", sms * 4, 256, V5S);
            run(v5<1>, "V5 +RED count", sms * 4, 256, V5S);
            run(v5<2>, "V5 +match count", sms * 4, 256, V5S);
            run(v5<4>, "V5 +push thread", sms * 4, 256, V5S);
            run(v5<8>, "V5 +push warp", sms * 4, 256, V5S);
            run(v5<5>, "V5 +RED +push thread", sms * 4, 256, V5S);
            run(v5<16>, "V5 4B keys", sms * 4, 256, V5S);
            run(v5<21>, "V5 4B keys +RED +push thread", sms * 4, 256, V5S);
        }
    }
    for (double frac : {0.27, 0.05}) {
        std::vector<int32_t> wl;
        uint64_t r = 12345;
        for (int64_t v = 0; v < n; v++) { r ^= r << 13; r ^= r >> 7; r ^= r << 17; if ((r % 10000) < frac * 10000) wl.push_back((int32_t)v); }
        int32_t* dwl; CK(cudaMalloc(&dwl, 4 * wl.size())); CK(cudaMemcpy(dwl, wl.data(), 4 * wl.size(), cudaMemcpyHostToDevice));
        int64_t nwl = wl.size();
        CK(cudaMemcpyToSymbol(g_wl, &dwl, sizeof(dwl))); CK(cudaMemcpyToSymbol(g_nwl, &nwl, sizeof(nwl)));
        printf("-- sparse worklist fraction %.2f (%lld rows): M only checked on the list\n", frac, (long long)nwl);
        run(v6<1, 16>, "V6 G1 B16", sms * 8, 256, 0);
        run(v6<2, 16>, "V6 G2 B16", sms * 8, 256, 0);
        run(v6<4, 8>, "V6 G4 B8", sms * 8, 256, 0);
        run(v6<8, 4>, "V6 G8 B4", sms * 8, 256, 0);
        run(v6<16, 2>, "V6 G16 B2", sms * 8, 256, 0);
        run(v6<32, 1>, "V6 G32 B1", sms * 8, 256, 0);
        run(v6<4, 8>, "V6 G4 B8 grid 4/SM", sms * 4, 256, 0);
    }
    {
        unsigned int* c; CK(cudaMalloc(&c, 64)); CK(cudaMemcpyToSymbol(g_ctr, &c, sizeof(c)));
        const int V7S = 2 * (256 * 27 + 8) * 4 + 64;
        for (int per : {2, 3, 4}) {
            // the counter is reset inside run() through the M memset hook below
            auto k7 = v7<16>;
            CK(cudaFuncSetAttribute(k7, cudaFuncAttributeMaxDynamicSharedMemorySize, V7S));
            float best = 1e9;
            for (int rep = 0; rep < 6; rep++) {
                CK(cudaMemset(flush, rep, 512 << 20)); CK(cudaMemset(c, 0, 64)); CK(cudaMemset(d_M, 0, 4 * n));
                cudaEventRecord(a); k7<<<sms * per, 256, V7S>>>(n, nnz, d_rp, d_ci, d_T, d_M); cudaEventRecord(b);
                CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (rep && ms < best) best = ms;
            }
            CK(cudaMemcpy(Md.data(), d_M, 4 * n, cudaMemcpyDeviceToHost));
            float bw = 1e9;
            for (int rep = 0; rep < 6; rep++) {
                CK(cudaMemset(c, 0, 64));
                cudaEventRecord(a); k7<<<sms * per, 256, V7S>>>(n, nnz, d_rp, d_ci, d_T, d_M); cudaEventRecord(b);
                CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (rep && ms < bw) bw = ms;
            }
            printf("V7 dynamic tiles %d/SM: warm %.1f us cold %.1f us %s\n", per, bw * 1e3, best * 1e3, Md == Mh ? "ok" : "WRONG");
        }
        run(v3<256, 16>, "V3 256 rows B16 (static)", sms * 4, 256, 2 * (256 * 27 + 8) * 4 + 64);
    }
    {
        const int V8S = 2 * (256 * 27 + 8) * 4 + 64;
        run(v8<16>, "V8 4B keys B16", sms * 4, 256, V8S);
        run(v8<32>, "V8 4B keys B32", sms * 4, 256, V8S);
        run(v8<28>, "V8 4B keys B28", sms * 4, 256, V8S);
        run(v3<256, 16>, "V3 256 rows B16 (8B)", sms * 4, 256, 2 * (256 * 27 + 8) * 4 + 64);
    }
    return 0;
}
