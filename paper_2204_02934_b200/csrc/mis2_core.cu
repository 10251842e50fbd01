// mis2_core.cu -- host side of the persistent MIS-2 kernel (mis2_kernel.cuh):
// launch configuration, workspace carving, the partitioned driver's phase
// launches.  The kernel templates are instantiated per G in mis2_g<G>.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mis2_kernel.cuh"

namespace mis2k {

__global__ void __launch_bounds__(kMB) mis2_part_init(MisParams p, int* cnts, unsigned long long* n_active) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
    const int64_t B = gridDim.x;
    const int64_t blo = p.n * blockIdx.x / B, bhi = p.n * (blockIdx.x + 1) / B;
    const uint64_t fi0 = p.prio.iter_term(0);
    int act_cnt = 0;
    for (int64_t v = blo + threadIdx.x; v < bhi; v += kMB) {
        const bool act = p.labels ? (p.labels[v] < 0) : true;
        p.T[v] = act ? p.prio.word(0, fi0, p.gbase + v) : kOUT;
        p.M[v] = act ? kPending : 0u;
        act_cnt += act;
    }
    const long long s = block_sum_int(sm, act_cnt);
    if (threadIdx.x == 0) {
        cnts[blockIdx.x] = (int)(bhi - blo);
        cnts[B + blockIdx.x] = (int)(bhi - blo);
        if (s) atomicAdd(n_active, (unsigned long long)s);
    }
}


__global__ void mis2_part_final(MisParams p, unsigned long long* count) {
    {
        const int64_t B = gridDim.x;
        l2_release(p, make_rows(p.n, B, blockIdx.x, kMB, false));
    }
    int c = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < p.n; v += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t in = (p.T[v] == kIN);
        p.in_set[v] = in;
        c += in;
    }
    c = group_sum<32>(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

int bits_for(int64_t n) {
    int b = 0;
    while (b < 63 && ((int64_t)1 << b) < n + 2) b++;
    return b;
}

// fraction of the colinds stream marked evict_last (l2_policy): an L2 budget
// (default 30% of L2, measured best on C2; MIS2_L2_KEEP_MB overrides, 0 disables) over its size
float l2_keep_for(int64_t nnz) {
    static int l2_bytes = -1;
    if (l2_bytes < 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, dev) != cudaSuccess)
            l2_bytes = 0;
    }
    double budget = 0.3 * (double)l2_bytes;
    if (const char* e = getenv("MIS2_L2_KEEP_MB")) budget = atof(e) * 1048576.0;
    const double bytes = (double)nnz * 4.0;
    if (budget <= 0.0 || bytes <= 0.0) return 0.f;
    return budget >= bytes ? 1.f : (float)(budget / bytes);
}

int max_iters_for(int64_t n, int requested) { return requested > 0 ? requested : 10 * bits_for(n) + 20; }

int choose_group(int64_t n, int64_t nnz, int requested) {
    if (requested > 0) return requested;
    const double avg = n > 0 ? (double)nnz / (double)n : 0.0;
    // a step of kMB / G rows should fit one staging buffer
    int g = 1;
    while (g < 32 && (double)(kMB / g) * avg > (double)kTileCap) g *= 2;
    return g;
}

// per-G entry points (mis2_g<G>.cu): the persistent kernel of a lane-group
// width, and one phase launch of the partitioned driver
template <int G>
void* persistent_kernel(bool stats, bool push);
template <int G>
cudaError_t launch_part_phase(int ph, const MisParams& p, int it, int grid, int smem, int* cnts,
                              unsigned long long* wl1, cudaStream_t s);
#define MIS2_DECLARE_G(G)                                                                            \
    template <>                                                                                      \
    void* persistent_kernel<G>(bool, bool);                                                          \
    template <>                                                                                      \
    cudaError_t launch_part_phase<G>(int, const MisParams&, int, int, int, int*, unsigned long long*, \
                                     cudaStream_t);
MIS2_DECLARE_G(1)
MIS2_DECLARE_G(2)
MIS2_DECLARE_G(4)
MIS2_DECLARE_G(8)
MIS2_DECLARE_G(16)
MIS2_DECLARE_G(32)
#undef MIS2_DECLARE_G

static void* pick_kernel(int G, bool stats, bool push) {
    switch (G) {
        case 1: return persistent_kernel<1>(stats, push);
        case 2: return persistent_kernel<2>(stats, push);
        case 4: return persistent_kernel<4>(stats, push);
        case 8: return persistent_kernel<8>(stats, push);
        case 16: return persistent_kernel<16>(stats, push);
        case 32: return persistent_kernel<32>(stats, push);
    }
    return nullptr;
}

int max_coop_warps(const DeviceInfo& d) { return d.sms * 64; }

void carve_mis2(Carve& c, int64_t n, int64_t nnz, int max_warps, Mis2Ws* w) {
    (void)max_warps;
    w->ctrl = c.take<unsigned long long>(16);
    w->T = c.take<uint64_t>((size_t)n + 1);
    w->M = c.take<uint32_t>((size_t)n + 1);
    for (int i = 0; i < 2; i++) {
        w->L1[i] = c.take<int32_t>((size_t)n + 1);
        w->L2[i] = c.take<int32_t>((size_t)n + 1);
    }
    w->heavy = c.take<int32_t>((size_t)n + 1);
    w->mark = c.take<unsigned int>((size_t)n + 1);
    w->oflag = c.take<uint8_t>((size_t)n + 1);
    w->cnt = c.take<uint32_t>((size_t)n + 1);
    w->degc = c.take<uint32_t>((size_t)n + 1);
    w->K = c.take<uint32_t>((size_t)n + 1);
    w->dstats = c.take<long long>((size_t)kStatsMaxIters * 6);
    w->scal = c.take<long long>(8);
}

static MisParams part_params(const PartDev& d) {
    MisParams p;
    memset(&p, 0, sizeof(p));
    p.n = d.n_own;
    p.gbase = d.gbase;
    p.nnz = d.nnz;
    p.rowptr = d.rowptr;
    p.colinds = d.colinds;
    p.labels = d.labels;
    p.T = d.T;
    p.M = d.M;
    for (int i = 0; i < 2; i++) {
        p.L1[i] = d.L1[i];
        p.L2[i] = d.L2[i];
    }
    p.prio.scheme = d.scheme;
    p.prio.hshift = d.hshift;
    p.prio.b = bits_for(d.n_global);
    p.prio.seed = d.seed;
    p.prio.hi_mask = ~((1ull << p.prio.b) - 1ull);
    p.id_mask = (uint32_t)((1ull << p.prio.b) - 1ull);
    p.prio.n = d.n_global;
    p.l2_keep = l2_keep_for(d.nnz);
    p.in_set = d.in_set;
    p.heavy = d.heavy;
    return p;
}

int part_step(const PartDev& d, int op, int it, cudaStream_t s) {
    const MisParams p = part_params(d);
    const int smem = (int)sizeof(TileSmem);
    const int grid = d.grid;
    if (op == kPartInit) {
        cudaFuncSetAttribute((const void*)mis2_part_init, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        mis2_part_init<<<grid, kMB, smem, s>>>(p, d.cnts, d.ctr + 0);
        count_launch();
        MIS2_CUDA_TRY(cudaGetLastError());
        return MIS2_OK;
    }
    if (op == kPartFinal) {
        mis2_part_final<<<grid, kMB, 0, s>>>(p, d.ctr + 2);
        count_launch();
        MIS2_CUDA_TRY(cudaGetLastError());
        return MIS2_OK;
    }
    const int ph = op == kPartColumn ? 0 : 1;
    cudaError_t e;
    switch (d.G) {
        case 1: e = launch_part_phase<1>(ph, p, it, grid, smem, d.cnts, d.ctr + 1, s); break;
        case 2: e = launch_part_phase<2>(ph, p, it, grid, smem, d.cnts, d.ctr + 1, s); break;
        case 4: e = launch_part_phase<4>(ph, p, it, grid, smem, d.cnts, d.ctr + 1, s); break;
        case 8: e = launch_part_phase<8>(ph, p, it, grid, smem, d.cnts, d.ctr + 1, s); break;
        case 16: e = launch_part_phase<16>(ph, p, it, grid, smem, d.cnts, d.ctr + 1, s); break;
        default: e = launch_part_phase<32>(ph, p, it, grid, smem, d.cnts, d.ctr + 1, s); break;
    }
    count_launch();
    if (e != cudaSuccess) {
        set_error("part phase launch: %s", cudaGetErrorString(e));
        return MIS2_ECUDA;
    }
    return MIS2_OK;
}

int debug_read(void* ws, size_t ws_bytes, int64_t n, long long* out, int64_t count) {
    Carve c(ws, ws_bytes);
    Mis2Ws w;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    carve_mis2(c, n, 0, max_coop_warps(di), &w);  // mark precedes the nnz-sized pieces
    const int64_t cap = ((int64_t)n + 1) / 2;
    if (count > cap) count = cap;
    MIS2_CUDA_TRY(cudaMemcpy(out, w.mark, sizeof(long long) * count, cudaMemcpyDeviceToHost));
    return MIS2_OK;
}

int part_grid(int64_t n_own, int G) {
    DeviceInfo di;
    if (device_info(&di) != MIS2_OK) return 1;
    const int64_t rpb = kMB / G;
    int64_t want = (n_own + 2 * rpb - 1) / (2 * rpb);
    const int64_t cap = (int64_t)kMinBlocksPerSM * di.sms;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (int)want;
}

int run_mis2(const mis2_graph& g, const mis2_opts& o, const int32_t* labels, uint8_t* in_set, int64_t* d_count,
             int32_t* d_iters, int32_t* d_status, int64_t* stats_host, const Mis2Ws& w, cudaStream_t s) {
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    if (g.n == 0) {  // empty set, 0 iterations (P5); no kernel touches rowptr (may be NULL)
        MIS2_CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
        MIS2_CUDA_TRY(cudaMemsetAsync(d_iters, 0, sizeof(int32_t), s));
        MIS2_CUDA_TRY(cudaMemsetAsync(d_status, 0, sizeof(int32_t), s));
        if (stats_host) {
            const size_t cnt = (o.flags & MIS2_FLAG_TIMELINE) ? 2 * (size_t)max_iters_for(0, o.max_iters) + 2
                                                              : 6 * (size_t)max_iters_for(0, o.max_iters);
            memset(stats_host, 0, sizeof(long long) * cnt);
        }
        return MIS2_OK;
    }
    const int G = choose_group(g.n, g.nnz, o.group);
    const bool timeline = stats_host != nullptr && (o.flags & MIS2_FLAG_TIMELINE);
    const bool stats = stats_host != nullptr && !timeline;
    const int max_iters = max_iters_for(g.n, o.max_iters);
    if ((stats && max_iters > kStatsMaxIters) || (timeline && 2 * max_iters + 2 > kStatsMaxIters * 6)) {
        set_error("stats/timeline mode supports max_iters <= %d", kStatsMaxIters);
        return MIS2_EINVAL;
    }
    // Decide form per iteration: push (its per-row push / count overhead
    // amortised over long rows) for every iteration of a dense graph; for a
    // medium one in iterations 0 and 1: in iteration 0 no M is OUT yet
    // (nothing to push) and the pull form's full second sweep over all rows
    // is replaced by one count per row; in iteration 1 ~99% of the rows are
    // still undecided, so the pull Decide is again a full sweep (C2 push
    // iterations 1 / 2 / 3: 376.8 / 374.8 / 374.9 us).  Pull otherwise.
    // Measured on C5 (avg degree 80), C2 (26.5), C3 (7).
    // MIS2_FLAG_PUSH_DECIDE / PULL_DECIDE force a form (MIS2_PUSH_ITERS:
    // measurement knob).
    const double avg_deg = g.n > 0 ? (double)g.nnz / (double)g.n : 0.0;
    int push_iters = avg_deg >= 32.0 ? max_iters : (avg_deg >= 16.0 ? 2 : 0);
    if (o.flags & MIS2_FLAG_PUSH_DECIDE) push_iters = max_iters;
    if (o.flags & MIS2_FLAG_PULL_DECIDE) push_iters = 0;
    if (const char* e = getenv("MIS2_PUSH_ITERS")) push_iters = atoi(e);
    void* fn = pick_kernel(G, stats, push_iters > 0);
    if (!fn) {
        set_error("group must be one of 1,2,4,8,16,32 (got %d)", G);
        return MIS2_EINVAL;
    }
    const int smem = (int)sizeof(TileSmem);
    MIS2_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    MIS2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kMB, smem));
    if (per_sm < 1) {
        set_error("persistent kernel does not fit on an SM");
        return MIS2_EINTERNAL;
    }
    if (const char* env = getenv("MIS2_BLOCKS_PER_SM")) {  // tuning knob (measurement only)
        const int want_per_sm = atoi(env);
        if (want_per_sm >= 1 && want_per_sm < per_sm) per_sm = want_per_sm;
    }
    const int64_t max_grid = (int64_t)per_sm * di.sms;
    // small graphs: about two steps of rows per block
    const int64_t rpb = kMB / G;
    const int64_t want = (g.n + 2 * rpb - 1) / (2 * rpb);
    const int grid = (int)(want < 1 ? 1 : (want > max_grid ? max_grid : want));

    MIS2_CUDA_TRY(cudaMemsetAsync(w.ctrl, 0, 16 * sizeof(unsigned long long), s));
    if (stats) {
        MIS2_CUDA_TRY(cudaMemsetAsync(w.mark, 0, sizeof(unsigned int) * ((size_t)g.n + 1), s));
        MIS2_CUDA_TRY(cudaMemsetAsync(w.dstats, 0, sizeof(long long) * kStatsMaxIters * 6, s));
    }
    MisParams p;
    memset(&p, 0, sizeof(p));
    p.n = g.n;
    p.gbase = 0;
    p.nnz = g.nnz;
    p.rowptr = g.rowptr;
    p.colinds = g.colinds;
    p.labels = labels;
    p.T = w.T;
    p.M = w.M;
    // 32-bit column keys: the two 64-bit minima per entry cost more ALU than
    // the halved gather bytes save on the stencil configs (C2 387 -> 451 us,
    // C3 5.6 -> 6.5 ms, C5 8.2 -> 10.1 ms); they help random-access graphs
    // whose T does not fit L2 (C4 92 -> 77 ms).  Automatic: candidates are
    // graphs with 8n > 64 MB; the kernel then uses the keys iff the largest
    // degree exceeds 16x the average (skewed, random access).
    // MIS2_FLAG_KEYS / MIS2_FLAG_NO_KEYS force (results identical).
    int keys = (double)g.n * 8.0 > 64.0 * 1048576.0 ? 2 : 0;  // 2 = decide on the device
    if (o.flags & MIS2_FLAG_KEYS) keys = 1;
    if (o.flags & MIS2_FLAG_NO_KEYS) keys = 0;
    if (const char* e = getenv("MIS2_KEYS")) keys = atoi(e);  // measurement knob
    if (o.flags & MIS2_FLAG_WORD32) keys = 0;  // the keys are the words' high halves
    p.K = keys ? w.K : nullptr;
    p.keys_mode = keys == 1 ? 1 : 0;
    for (int i = 0; i < 2; i++) {
        p.L1[i] = w.L1[i];
        p.L2[i] = w.L2[i];
    }
    p.ctrl = w.ctrl;
    p.heavy = w.heavy;
    p.mark = w.mark;
    p.oflag = w.oflag;
    p.cnt = w.cnt;
    p.degc = w.degc;
    p.dstats = w.dstats;
    p.timeline = timeline ? w.dstats : nullptr;
    p.dbg_it = -1;
    p.dbg_ph = 0;
    if (timeline) {
        if (const char* e = getenv("MIS2_DBG_IT")) p.dbg_it = atoi(e);
        if (const char* e = getenv("MIS2_DBG_PH")) p.dbg_ph = atoi(e);
        // per-block debug records (64 int64 each) live in `mark` (4(n+1) bytes):
        // only when every block's record fits
        if ((size_t)grid * 64 * sizeof(long long) > sizeof(unsigned int) * ((size_t)g.n + 1)) p.dbg_it = -1;
        if (p.dbg_it >= 0) MIS2_CUDA_TRY(cudaMemsetAsync(w.mark, 0, sizeof(long long) * 64 * (size_t)grid, s));
    }
    p.prio.scheme = o.scheme;
    p.prio.hshift = (o.flags & MIS2_FLAG_WORD32) ? 32 : 0;
    p.prio.b = bits_for(g.n);
    p.prio.seed = o.seed;
    p.prio.hi_mask = ~((1ull << p.prio.b) - 1ull);
    p.id_mask = (uint32_t)((1ull << p.prio.b) - 1ull);
    p.prio.n = g.n;
    p.l2_keep = l2_keep_for(g.nnz);
    // cyclic row ownership (mis2_kernel.cuh Rows); MIS2_CYCLIC=0: contiguous
    // ranges (measurement knob, results identical)
    p.cyclic = 1;
    if (const char* e = getenv("MIS2_CYCLIC")) p.cyclic = atoi(e) != 0;
    p.push_iters = push_iters;
    p.prio.override_ = o.prio_override;
    p.prio.override_iters = o.prio_override ? o.prio_iters : 0;
    p.max_iters = max_iters;
    p.in_set = in_set;
    p.d_count = d_count;
    p.d_iters = d_iters;
    p.d_status = d_status;
    void* args[] = {&p};
    MIS2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kMB), args, smem, s));
    count_launch();
    if (stats || timeline) {
        const size_t cnt = stats ? 6 * (size_t)max_iters : 2 * (size_t)max_iters + 2;
        MIS2_CUDA_TRY(cudaMemcpyAsync(stats_host, w.dstats, sizeof(long long) * cnt, cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    }
    return MIS2_OK;
}

}  // namespace mis2h
