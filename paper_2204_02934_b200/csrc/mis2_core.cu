// mis2_core.cu -- Alg. 1 (MIS-2, §III-A) as ONE persistent,
// cooperatively launched sm_100a kernel.
//
// Design:
//  * Every warp owns a fixed contiguous slice [lo, hi) of the vertex range.
//    worklist_1 / worklist_2 (§V-B) are stored IN PLACE
//    inside the owning warp's slice of two int32[n] arrays and compacted with
//    __ballot_sync/__popc -- no global scan, no atomics, ascending order kept.
//  * Each CSR row is processed by a group of G lanes (G = 1..32) -- §V-D
//    "SIMD parallelism ... only if the average vertex degree is at least 16"
//     generalised to a tunable group width; min / exists / forall
//    are reduced with shuffles.
//  * Phases are separated by a grid-wide barrier instead of kernel launches;
//    the loop condition |worklist_1| == 0 is evaluated on the device, so one
//    MIS-2 call is 1 memset + 1 kernel launch.
//  * Refresh Row for iteration i+1 is fused into Decide of
//    iteration i; iteration 0's refresh is the init phase.
//  * Status words are 64-bit (Eq. 1, reading Q6), so every min is
//    one integer compare.
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace mis2k {

struct MisParams {
    int64_t n;
    const int64_t* __restrict__ rowptr;
    const int32_t* __restrict__ colinds;
    const int32_t* __restrict__ labels;  // phase-2 mask (active iff labels[v] < 0) or null
    uint64_t* T;                         // row status T_v
    uint64_t* M;                         // column status M_v
    int32_t* L1;                         // worklist_1, per-warp in-place segments
    int32_t* L2;                         // worklist_2
    int32_t* c1;                         // per-warp |segment of worklist_1|
    int32_t* c2;
    unsigned long long* ctrl;
    unsigned int* mark;    // stats only
    long long* dstats;     // stats only
    Prio prio;
    int max_iters;
    uint8_t* in_set;
    int64_t* d_count;
    int32_t* d_iters;
    int32_t* d_status;
};

// ---------------------------------------------------------------- phases
// Refresh Column: for v in worklist_2: M_v = min(T_w : w in N[v]);
// IN -> OUT.  Inactive vertices (phase 2) carry T = OUT, neutral for min.
// Survivors (M_v != OUT) are compacted in place into the warp's L2 segment.
template <int G, bool STATS>
__device__ __forceinline__ void column_phase(const MisParams& p, int it, int64_t lo, int64_t hi,
                                             int gw, int lane) {
    constexpr int RPW = 32 / G;
    const int grp = lane / G, sub = lane % G;
    const bool dense = (it == 0);
    const int64_t total = dense ? (hi - lo) : (int64_t)p.c2[gw];
    int32_t k = 0;
    long long r_acc = 0, e_acc = 0, d_acc = 0;
    const unsigned tag = 2u * (unsigned)it + 1u;  // column runs before decide
    for (int64_t base = 0; base < total; base += RPW) {
        const int64_t idx = base + grp;
        const bool valid = idx < total;
        int64_t v = 0;
        bool act = false;
        if (valid) {
            v = dense ? lo + idx : (int64_t)p.L2[lo + idx];
            act = dense && p.labels ? (p.labels[v] < 0) : true;
        }
        uint64_t m = kOUT;
        if (act) {
            const int64_t s = p.rowptr[v], e = p.rowptr[v + 1];
            if (sub == 0) m = p.T[v];
            int64_t j = s + sub;
            // 4 independent gathers in flight per lane
            for (; j + 3 * G < e; j += 4 * G) {
                const int32_t w0 = p.colinds[j], w1 = p.colinds[j + G], w2 = p.colinds[j + 2 * G],
                              w3 = p.colinds[j + 3 * G];
                const uint64_t t0 = p.T[w0], t1 = p.T[w1], t2 = p.T[w2], t3 = p.T[w3];
                const uint64_t a = t0 < t1 ? t0 : t1, b = t2 < t3 ? t2 : t3;
                const uint64_t c = a < b ? a : b;
                m = c < m ? c : m;
            }
            for (; j < e; j += G) {
                const uint64_t t = p.T[p.colinds[j]];
                m = t < m ? t : m;
            }
            if (STATS) {
                if (sub == 0) {
                    r_acc++;
                    e_acc += e - s;
                    if (atomicMax(&p.mark[v], tag) < tag) d_acc++;
                }
                for (int64_t jj = s + sub; jj < e; jj += G)
                    if (atomicMax(&p.mark[p.colinds[jj]], tag) < tag) d_acc++;
            }
        }
        m = group_min<G>(m);
        bool keep = false;
        if (act && sub == 0) {
            if (m == kIN) m = kOUT;
            p.M[v] = m;
            keep = (m != kOUT);
        }
        const unsigned ball = __ballot_sync(kFull, keep);
        if (keep) p.L2[lo + k + __popc(ball & lanemask_lt())] = (int32_t)v;
        k += __popc(ball);
    }
    if (lane == 0) p.c2[gw] = k;
    if (STATS) {
        long long r_tot = warp_sum_ll(r_acc), e_tot = warp_sum_ll(e_acc), d_tot = warp_sum_ll(d_acc);
        if (lane == 0) {
            long long* st = p.dstats + 6 * it;
            atomicAdd((unsigned long long*)&st[1], (unsigned long long)r_tot);
            atomicAdd((unsigned long long*)&st[3], (unsigned long long)e_tot);
            atomicAdd((unsigned long long*)&st[5], (unsigned long long)d_tot);
        }
    }
}

// Decide on the pre-update T_v (reading Q2):
//   exists w in N[v]: M_w = OUT  -> OUT
//   else forall w in N[v]: M_w = T_v -> IN
//   else undecided: fused Refresh Row of iteration it+1.
// M_w = 0 marks an inactive (phase-2) vertex and is ignored (reading Q15).
template <int G, bool STATS>
__device__ __forceinline__ int32_t decide_phase(const MisParams& p, int it, int64_t lo, int64_t hi,
                                                int gw, int lane, uint64_t fi_next) {
    constexpr int RPW = 32 / G;
    const int grp = lane / G, sub = lane % G;
    const bool dense = (it == 0);
    const int64_t total = dense ? (hi - lo) : (int64_t)p.c1[gw];
    int32_t k = 0;
    long long r_acc = 0, e_acc = 0, d_acc = 0;
    const unsigned tag = 2u * (unsigned)it + 2u;
    for (int64_t base = 0; base < total; base += RPW) {
        const int64_t idx = base + grp;
        const bool valid = idx < total;
        int64_t v = 0;
        uint64_t tv = kOUT;
        bool act = false;
        if (valid) {
            v = dense ? lo + idx : (int64_t)p.L1[lo + idx];
            tv = p.T[v];
            act = (tv != kIN && tv != kOUT);
        }
        int any_out = 0, all_eq = 1;
        if (act) {
            const int64_t s = p.rowptr[v], e = p.rowptr[v + 1];
            if (sub == 0) {
                const uint64_t m = p.M[v];
                any_out = (m == kOUT);
                all_eq = (m == tv);
            }
            int64_t j = s + sub;
            for (; j + 3 * G < e; j += 4 * G) {
                const int32_t w0 = p.colinds[j], w1 = p.colinds[j + G], w2 = p.colinds[j + 2 * G],
                              w3 = p.colinds[j + 3 * G];
                const uint64_t m0 = p.M[w0], m1 = p.M[w1], m2 = p.M[w2], m3 = p.M[w3];
                any_out |= (m0 == kOUT) | (m1 == kOUT) | (m2 == kOUT) | (m3 == kOUT);
                all_eq &= (m0 == tv || m0 == 0) & (m1 == tv || m1 == 0) & (m2 == tv || m2 == 0) &
                          (m3 == tv || m3 == 0);
            }
            for (; j < e; j += G) {
                const uint64_t m = p.M[p.colinds[j]];
                any_out |= (m == kOUT);
                all_eq &= (m == tv || m == 0);
            }
            if (STATS) {
                if (sub == 0) {
                    r_acc++;
                    e_acc += e - s;
                    if (atomicMax(&p.mark[v], tag) < tag) d_acc++;
                }
                for (int64_t jj = s + sub; jj < e; jj += G)
                    if (atomicMax(&p.mark[p.colinds[jj]], tag) < tag) d_acc++;
            }
        }
        any_out = group_or<G>(any_out);
        all_eq = group_and<G>(all_eq);
        bool keep = false;
        if (act && sub == 0) {
            if (any_out) p.T[v] = kOUT;
            else if (all_eq) p.T[v] = kIN;
            else {
                p.T[v] = p.prio.word(it + 1, fi_next, v);
                keep = true;
            }
        }
        const unsigned ball = __ballot_sync(kFull, keep);
        if (keep) p.L1[lo + k + __popc(ball & lanemask_lt())] = (int32_t)v;
        k += __popc(ball);
    }
    if (lane == 0) p.c1[gw] = k;
    if (STATS) {
        long long r_tot = warp_sum_ll(r_acc), e_tot = warp_sum_ll(e_acc), d_tot = warp_sum_ll(d_acc);
        if (lane == 0) {
            long long* st = p.dstats + 6 * it;
            atomicAdd((unsigned long long*)&st[0], (unsigned long long)r_tot);
            atomicAdd((unsigned long long*)&st[2], (unsigned long long)e_tot);
            atomicAdd((unsigned long long*)&st[4], (unsigned long long)d_tot);
        }
    }
    return k;
}

template <int G, bool STATS>
__global__ void __launch_bounds__(kBlock) mis2_persistent(MisParams p) {
    __shared__ long long s_tmp[kWarpsPerBlock];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = gridDim.x * kWarpsPerBlock;
    const int gw = blockIdx.x * kWarpsPerBlock + warp;
    const int64_t lo = p.n * gw / W, hi = p.n * (gw + 1) / W;
    unsigned int* bar = (unsigned int*)&p.ctrl[0];
    unsigned long long* ring = &p.ctrl[1];

    // worklists <- 0..|V| and Refresh Row of iteration 0
    {
        const uint64_t fi0 = p.prio.iter_term(0);
        for (int64_t v = lo + lane; v < hi; v += 32) {
            const bool act = p.labels ? (p.labels[v] < 0) : true;
            p.T[v] = act ? p.prio.word(0, fi0, v) : kOUT;
            if (!act) p.M[v] = 0;  // inactive sentinel (reading Q15)
        }
    }
    grid_barrier(bar);

    int it = 0;
    int status = MIS2_OK;
    for (;;) {
        column_phase<G, STATS>(p, it, lo, hi, gw, lane);
        grid_barrier(bar);
        const uint64_t fi_next = p.prio.iter_term(it + 1);
        const int32_t k = decide_phase<G, STATS>(p, it, lo, hi, gw, lane, fi_next);
        const long long bsum = block_sum_warps(lane == 0 ? k : 0, s_tmp);
        if (threadIdx.x == 0) {
            if (bsum) atomicAdd(&ring[it & 3], (unsigned long long)bsum);
            if (blockIdx.x == 0) ring[(it + 2) & 3] = 0;  // slot read two barriers ago
        }
        grid_barrier(bar);
        const unsigned long long remaining = ld_acquire_u64(&ring[it & 3]);
        it++;
        if (remaining == 0) break;        // worklist_1 empty
        if (it >= p.max_iters) {          // reading Q12
            status = MIS2_ENOTCONVERGED;
            break;
        }
    }

    // return {v : T_v = IN}
    long long cnt = 0;
    for (int64_t v = lo + lane; v < hi; v += 32) {
        const uint8_t in = (p.T[v] == kIN);
        p.in_set[v] = in;
        cnt += in;
    }
    cnt = warp_sum_ll(cnt);
    const long long bcnt = block_sum_warps(lane == 0 ? cnt : 0, s_tmp);
    if (threadIdx.x == 0) {
        atomicAdd(&p.ctrl[5], (unsigned long long)bcnt);
        __threadfence();
        const unsigned long long ticket = atomicAdd(&p.ctrl[6], 1ull);
        if (ticket == gridDim.x - 1) {  // last block publishes the scalars
            __threadfence();
            *p.d_count = (int64_t)ld_acquire_u64(&p.ctrl[5]);
            *p.d_iters = it;
            *p.d_status = status;
        }
    }
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

int bits_for(int64_t n) {
    int b = 0;
    while (b < 63 && ((int64_t)1 << b) < n + 2) b++;
    return b;
}

int max_iters_for(int64_t n, int requested) { return requested > 0 ? requested : 10 * bits_for(n) + 20; }

int choose_group(int64_t n, int64_t nnz, int requested) {
    if (requested > 0) return requested;
    const double avg = n > 0 ? (double)nnz / (double)n : 0.0;
    // about 4 entries per lane; a warp per row only for long rows
    int g = 1;
    while (g < 32 && g * 4 < avg) g *= 2;
    return g;
}

template <int G, bool S>
static void* kernel_ptr() {
    return (void*)&mis2_persistent<G, S>;
}

static void* pick_kernel(int G, bool stats) {
    switch (G) {
        case 1: return stats ? kernel_ptr<1, true>() : kernel_ptr<1, false>();
        case 2: return stats ? kernel_ptr<2, true>() : kernel_ptr<2, false>();
        case 4: return stats ? kernel_ptr<4, true>() : kernel_ptr<4, false>();
        case 8: return stats ? kernel_ptr<8, true>() : kernel_ptr<8, false>();
        case 16: return stats ? kernel_ptr<16, true>() : kernel_ptr<16, false>();
        case 32: return stats ? kernel_ptr<32, true>() : kernel_ptr<32, false>();
    }
    return nullptr;
}

int max_coop_warps(const DeviceInfo& d) {
    // upper bound used for workspace sizing: 64 resident warps per SM
    return d.sms * 64;
}

void carve_mis2(Carve& c, int64_t n, int max_warps, Mis2Ws* w) {
    w->ctrl = c.take<unsigned long long>(16);
    w->T = c.take<uint64_t>((size_t)n + 1);
    w->M = c.take<uint64_t>((size_t)n + 1);
    w->L1 = c.take<int32_t>((size_t)n + 1);
    w->L2 = c.take<int32_t>((size_t)n + 1);
    w->c1 = c.take<int32_t>((size_t)max_warps);
    w->c2 = c.take<int32_t>((size_t)max_warps);
    w->mark = c.take<unsigned int>((size_t)n + 1);
    w->dstats = c.take<long long>((size_t)kStatsMaxIters * 6);
    w->scal = c.take<long long>(8);
}

int run_mis2(const mis2_graph& g, const mis2_opts& o, const int32_t* labels, uint8_t* in_set,
             int64_t* d_count, int32_t* d_iters, int32_t* d_status, int64_t* stats_host,
             const Mis2Ws& w, cudaStream_t s) {
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    const int G = choose_group(g.n, g.nnz, o.group);
    const bool stats = stats_host != nullptr;
    const int max_iters = max_iters_for(g.n, o.max_iters);
    if (stats && max_iters > kStatsMaxIters) {
        set_error("stats mode supports max_iters <= %d", kStatsMaxIters);
        return MIS2_EINVAL;
    }
    void* fn = pick_kernel(G, stats);
    if (!fn) {
        set_error("group must be one of 1,2,4,8,16,32 (got %d)", G);
        return MIS2_EINVAL;
    }
    int per_sm = 0;
    MIS2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, 0));
    if (per_sm < 1) {
        set_error("persistent kernel does not fit on an SM");
        return MIS2_EINTERNAL;
    }
    const int64_t max_grid = (int64_t)per_sm * di.sms;
    int64_t want = (g.n + kBlock - 1) / kBlock;
    const int grid = (int)(want < 1 ? 1 : (want > max_grid ? max_grid : want));

    MIS2_CUDA_TRY(cudaMemsetAsync(w.ctrl, 0, 16 * sizeof(unsigned long long), s));
    count_launch();
    if (stats) {
        MIS2_CUDA_TRY(cudaMemsetAsync(w.mark, 0, sizeof(unsigned int) * ((size_t)g.n + 1), s));
        MIS2_CUDA_TRY(cudaMemsetAsync(w.dstats, 0, sizeof(long long) * kStatsMaxIters * 6, s));
        count_launch(2);
    }
    MisParams p;
    p.n = g.n;
    p.rowptr = g.rowptr;
    p.colinds = g.colinds;
    p.labels = labels;
    p.T = w.T;
    p.M = w.M;
    p.L1 = w.L1;
    p.L2 = w.L2;
    p.c1 = w.c1;
    p.c2 = w.c2;
    p.ctrl = w.ctrl;
    p.mark = w.mark;
    p.dstats = w.dstats;
    p.prio.scheme = o.scheme;
    p.prio.b = bits_for(g.n);
    p.prio.seed = o.seed;
    p.prio.hi_mask = ~((1ull << p.prio.b) - 1ull);
    p.prio.n = g.n;
    p.prio.override_ = o.prio_override;
    p.prio.override_iters = o.prio_override ? o.prio_iters : 0;
    p.max_iters = max_iters;
    p.in_set = in_set;
    p.d_count = d_count;
    p.d_iters = d_iters;
    p.d_status = d_status;
    void* args[] = {&p};
    MIS2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args, 0, s));
    count_launch();
    if (stats) {
        MIS2_CUDA_TRY(cudaMemcpyAsync(stats_host, w.dstats, sizeof(long long) * 6 * (size_t)max_iters,
                                      cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    }
    return MIS2_OK;
}

}  // namespace mis2h
