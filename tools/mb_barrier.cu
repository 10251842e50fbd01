// tools/mb_barrier.cu -- measurement aid (not product code): cost of one
// grid-wide barrier of a cooperative grid (the persistent MIS-2 kernel's
// phase separator) for several grid shapes and barrier variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbbar tools/mb_barrier.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// MODE 0: product barrier (atom.add.release, relaxed poll + nanosleep, acq_rel fence)
// MODE 1: same without nanosleep
// MODE 2: red.release arrival (no return) on a per-barrier counter, poll for count
// MODE 3: two-level: per-group (16 blocks) counter, group leader arrives globally
template <int MODE>
__global__ void bar_kernel(unsigned int* ctr, int iters, int stores, unsigned int* junk) {
    for (int i = 0; i < iters; i++) {
        for (int s = threadIdx.x; s < stores; s += blockDim.x) junk[(blockIdx.x * stores + s) & 0xffffff] = i;
        __syncthreads();
        if (threadIdx.x == 0) {
            if (MODE <= 1) {
                unsigned int nb = (blockIdx.x == 0) ? (0x80000000u - (gridDim.x - 1)) : 1u;
                unsigned int old, cur;
                asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(ctr), "r"(nb) : "memory");
                for (;;) {
                    asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(ctr) : "memory");
                    if ((old ^ cur) & 0x80000000u) break;
                    if (MODE == 0) __nanosleep(32);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (MODE == 2) {
                unsigned int* c = ctr + 32 * (i & 3);
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
                unsigned int cur;
                for (;;) {
                    asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(c) : "memory");
                    if (cur >= (unsigned)gridDim.x * (unsigned)(i / 4 + 1)) break;
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (MODE == 6 || MODE == 7) {
                // one arrival counter; the last arriver publishes the epoch to 8
                // release lines (256 B apart); block b polls line b & 7
                unsigned int old, cur;
                asm volatile("atom.add.acq_rel.gpu.u32 %0,[%1],1;" : "=r"(old) : "l"(ctr) : "memory");
                if (old == (unsigned)gridDim.x * (unsigned)(i + 1) - 1)
                    for (int q = 0; q < 8; q++) asm volatile("st.relaxed.gpu.u32 [%0], %1;" ::"l"(ctr + 64 * (q + 1)), "r"(i + 1) : "memory");
                unsigned int* rl = ctr + 64 * ((blockIdx.x & 7) + 1);
                for (;;) {
                    asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(rl) : "memory");
                    if (cur >= (unsigned)(i + 1)) break;
                    if (MODE == 6) __nanosleep(32);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (MODE == 4 || MODE == 5) {
                // arrivals spread over 32 counters 256 B apart (different L2 slices);
                // the poll sums them (warp 0 polls, lane j reads counter j)
                unsigned int* c = ctr + 64 * (blockIdx.x & 31);
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
            } else {
                const int grp = blockIdx.x / 16, ng = (gridDim.x + 15) / 16;
                const int gsz = min(16, (int)gridDim.x - grp * 16);
                unsigned int* gc = ctr + 256 + 32 * grp;
                unsigned int* top = ctr + 128;
                unsigned int* rel = ctr + 160;
                unsigned int old, cur;
                asm volatile("atom.add.acq_rel.gpu.u32 %0,[%1],1;" : "=r"(old) : "l"(gc) : "memory");
                if (old == (unsigned)gsz * (i + 1) - 1) {  // last of the group
                    asm volatile("atom.add.acq_rel.gpu.u32 %0,[%1],1;" : "=r"(old) : "l"(top) : "memory");
                    if (old == (unsigned)ng * (i + 1) - 1) asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(rel), "r"(i + 1) : "memory");
                }
                for (;;) {
                    asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(rel) : "memory");
                    if (cur >= (unsigned)(i + 1)) break;
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        if (MODE == 4 || MODE == 5) {
            if (threadIdx.x < 32) {
                const unsigned int target = (unsigned)gridDim.x * (unsigned)(i + 1);
                for (;;) {
                    unsigned int cur;
                    asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(ctr + 64 * threadIdx.x) : "memory");
                    cur = __reduce_add_sync(0xffffffffu, cur);
                    if (cur >= target) break;
                    if (MODE == 5) __nanosleep(20);
                }
                if (threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
}

int main() {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned int *ctr, *junk;
    CK(cudaMalloc(&ctr, 1 << 20)); CK(cudaMalloc(&junk, 64 << 20));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto k, const char* name, int grid, int block, int stores) {
        const int iters = 200;
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            CK(cudaMemset(ctr, 0, 1 << 20));
            void* args[] = {&ctr, (void*)&iters, &stores, &junk};
            int it2 = iters;
            args[1] = &it2;
            cudaEventRecord(a);
            CK(cudaLaunchCooperativeKernel((void*)k, dim3(grid), dim3(block), args, 0, 0));
            cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); if (rep && ms < best) best = ms;
        }
        printf("%-22s grid %5d x %4d stores/blk %5d: %.2f us per barrier\n", name, grid, block, stores, best * 1e3 / iters);
    };
    for (int stores : {0, 1024}) {
        for (int per : {1, 4}) {
            const int blk = per == 1 ? 1024 : 256;
            run(bar_kernel<0>, "atom+poll+sleep", sms * per, blk, stores);
            run(bar_kernel<1>, "atom+poll", sms * per, blk, stores);
            run(bar_kernel<2>, "red+count poll", sms * per, blk, stores);
            run(bar_kernel<3>, "two-level 16", sms * per, blk, stores);
            run(bar_kernel<4>, "spread32 red, warp poll", sms * per, blk, stores);
            run(bar_kernel<5>, "spread32 + sleep", sms * per, blk, stores);
            run(bar_kernel<6>, "last->8 lines +sleep", sms * per, blk, stores);
            run(bar_kernel<7>, "last->8 lines", sms * per, blk, stores);
        }
    }
    return 0;
}
