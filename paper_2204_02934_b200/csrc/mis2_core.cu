// mis2_core.cu -- host side of the persistent MIS-2 kernel (mis2_kernel.cuh):
// launch configuration, workspace carving, the partitioned driver's phase
// launches.  The kernel templates are instantiated per G in mis2_g<G>.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mis2_kernel.cuh"

namespace mis2k {

// largest row length (skew test of run_mis2)
__global__ void k_max_degree(int64_t n, const int64_t* __restrict__ rowptr, unsigned long long* out) {
    int64_t m = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        m = max(m, rowptr[v + 1] - rowptr[v]);
    m = ~group_min<32>(~(uint64_t)m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, (unsigned long long)m);
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
void* dist_kernel();
#define MIS2_DECLARE_G(G)                   \
    template <>                             \
    void* persistent_kernel<G>(bool, bool); \
    template <>                             \
    void* dist_kernel<G>();
MIS2_DECLARE_G(1)
MIS2_DECLARE_G(2)
MIS2_DECLARE_G(4)
MIS2_DECLARE_G(8)
MIS2_DECLARE_G(16)
MIS2_DECLARE_G(32)
#undef MIS2_DECLARE_G

// the small-tile copies (mis2_g<G>s.cu), for skewed graphs
template <int G>
void* persistent_kernel_small(bool stats, bool push);
template <>
void* persistent_kernel_small<1>(bool, bool);
template <>
void* persistent_kernel_small<2>(bool, bool);
template <>
void* persistent_kernel_small<4>(bool, bool);
int tile_smem_small();
int tile_cap_small();
static void* pick_kernel_small(int G, bool stats, bool push) {
    switch (G) {
        case 1: return persistent_kernel_small<1>(stats, push);
        case 2: return persistent_kernel_small<2>(stats, push);
        case 4: return persistent_kernel_small<4>(stats, push);
    }
    return nullptr;
}

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
    w->ctrl = c.take<unsigned long long>(80);
    w->maxdeg = c.take<unsigned long long>(1);
    w->T = c.take<uint64_t>((size_t)n + 1);
    w->M = c.take<uint32_t>((size_t)n + 1);
    for (int i = 0; i < 2; i++) {
        w->L1[i] = c.take<int32_t>((size_t)n + 1);
        w->L2[i] = c.take<int32_t>((size_t)n + 1);
    }
    w->heavy = c.take<int32_t>((size_t)n + 1);
    w->mark = c.take<unsigned int>((size_t)n + 1);
    w->gq = c.take<int32_t>((size_t)n + 1);
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

static void* pick_dist_kernel(int G) {
    switch (G) {
        case 1: return dist_kernel<1>();
        case 2: return dist_kernel<2>();
        case 4: return dist_kernel<4>();
        case 8: return dist_kernel<8>();
        case 16: return dist_kernel<16>();
        case 32: return dist_kernel<32>();
    }
    return nullptr;
}

size_t dist_scratch_bytes(int nlocal) { return sizeof(PartK) * (size_t)(nlocal > 0 ? nlocal : 1) + 256; }

int dist_mis2_launch(const std::vector<PartDev>& parts, const std::vector<uint64_t*>& peer_T,
                     const std::vector<uint32_t*>& peer_M, const std::vector<unsigned long long*>& peer_box,
                     bool sys_scope, int G, int max_iters, unsigned int* epoch, void* dev_scratch, int64_t* count,
                     int32_t* iters, cudaStream_t s) {
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    const int nl = (int)parts.size();
    const int P = (int)peer_T.size();
    if (P > kMaxParts || nl < 1) {
        set_error("partitions: %d local of %d (at most %d)", nl, P, kMaxParts);
        return MIS2_EINVAL;
    }
    void* fn = pick_dist_kernel(G);
    if (!fn) {
        set_error("group must be one of 1,2,4,8,16,32 (got %d)", G);
        return MIS2_EINVAL;
    }
    const int smem = (int)sizeof(TileSmem);
    static thread_local void* cached_fn = nullptr;  // attribute + occupancy per kernel, once per thread
    static thread_local int cached_per_sm = 0;
    if (cached_fn != fn) {
        MIS2_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        MIS2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached_per_sm, fn, kMB, smem));
        cached_fn = fn;
    }
    const int per_sm = cached_per_sm;
    if (per_sm < 1) {
        set_error("partitioned kernel does not fit on an SM");
        return MIS2_EINTERNAL;
    }
    // blocks per local partition: the co-resident maximum split by owned
    // rows, about two dense steps per block at most, at least one each
    const int64_t max_grid = (int64_t)per_sm * di.sms;
    const int64_t rpb = kMB / G;
    int64_t tot_rows = 0;
    for (const PartDev& d : parts) tot_rows += d.n_own;
    std::vector<int> nblk(nl);
    int64_t grid = 0;
    for (int i = 0; i < nl; i++) {
        int64_t want = (parts[i].n_own + 2 * rpb - 1) / (2 * rpb);
        const int64_t share = tot_rows > 0 ? (max_grid - nl) * parts[i].n_own / tot_rows + 1 : 1;
        if (want > share) want = share;
        if (want < 1) want = 1;
        nblk[i] = (int)want;
        grid += want;
    }
    std::vector<PartK> hk(nl);
    int blk0 = 0;
    for (int i = 0; i < nl; i++) {
        const PartDev& d = parts[i];
        PartK& k = hk[i];
        memset(&k, 0, sizeof(k));
        k.mp = part_params(d);
        k.blk0 = blk0;
        k.nblk = nblk[i];
        blk0 += nblk[i];
        k.gpart = d.gpart;
        k.nsend = d.nsend;
        k.send_csp = d.send_csp;
        k.send_src = d.send_src;
        k.send_peer = d.send_peer;
        k.send_dst = d.send_dst;
        k.bar = d.bar;
        k.acc = d.acc;
        k.box = d.box;
        k.rel = d.rel;
    }
    PeerTab peers;
    memset(&peers, 0, sizeof(peers));
    peers.P = P;
    peers.sys = sys_scope ? 1 : 0;
    for (int q = 0; q < P; q++) {
        peers.T[q] = peer_T[q];
        peers.M[q] = peer_M[q];
        peers.box[q] = peer_box[q];
    }
    PartK* dk = (PartK*)dev_scratch;
    unsigned long long* dout = (unsigned long long*)((char*)dev_scratch + sizeof(PartK) * nl);
    dout = (unsigned long long*)(((uintptr_t)dout + 15) & ~(uintptr_t)15);
    // the parameter block changes only with the per-call options (seed,
    // masks, outputs): upload it when it differs from the last call's
    static thread_local std::vector<char> last;
    static thread_local void* last_dst = nullptr;
    const size_t kb = sizeof(PartK) * nl;
    if (last_dst != (void*)dk || last.size() != kb || memcmp(last.data(), hk.data(), kb) != 0) {
        MIS2_CUDA_TRY(cudaMemcpyAsync(dk, hk.data(), kb, cudaMemcpyHostToDevice, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));  // hk is a host stack vector
        last.assign((const char*)hk.data(), (const char*)hk.data() + kb);
        last_dst = (void*)dk;
    }
    unsigned int e0 = *epoch;
    MIS2_CUDA_TRY(cudaMemsetAsync(dout + 3, 0, sizeof(unsigned long long), s));  // peer-wait timeout flag
    void* args[] = {&dk, (void*)&nl, &peers, &e0, &max_iters, &dout};
    int nlv = nl;
    args[1] = &nlv;
    MIS2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(kMB), args, smem, s));
    count_launch();
    unsigned long long h[3];
    MIS2_CUDA_TRY(cudaMemcpyAsync(h, dout, sizeof(h), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    *count = (int64_t)h[0];
    *iters = (int32_t)(h[1] & 0xffffffffull);
    *epoch = (unsigned int)h[2];
    const int st = (int)(int32_t)(h[1] >> 32);
    if (st == MIS2_EINTERNAL) set_error("partition barrier: a peer GPU did not post within 10 s");
    else if (st != MIS2_OK) set_error("MIS-2 did not converge within max_iters");
    return st;
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

int run_mis2(const mis2_graph& g, const mis2_opts& o, const int32_t* labels, uint8_t* in_set, int64_t* d_count,
             int32_t* d_iters, int32_t* d_status, int64_t* stats_host, const Mis2Ws& w, cudaStream_t s,
             const SubGraph* sub) {
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
    const int max_iters = max_iters_for(sub ? sub->n_full : g.n, o.max_iters);
    if ((stats && max_iters > kStatsMaxIters) || (timeline && 2 * max_iters + 2 > kStatsMaxIters * 6)) {
        set_error("stats/timeline mode supports max_iters <= %d", kStatsMaxIters);
        return MIS2_EINVAL;
    }
    // Decide form per iteration: push for the first iterations, where
    // nearly every row of worklist_2 is still undecided and the pull form's
    // second sweep would re-read almost every row the column pass read; pull
    // once worklist_1 is a small part of worklist_2 (the push form's OUT
    // pushes then cost more than the pull form's early-exit reads).  Short
    // rows (average degree < 16): iteration 0 only (there is no OUT to push
    // yet).  Measured (us / ms per call, push iterations 1 / 2 / 3 / 4 / all):
    // C2 (avg 26.5) - / 348 / 342 / - / 395; C3 (7) 4.68 / 4.84 (0: 4.84) ms;
    // C4 (31) 40.9 / 38.2 / 37.5 ms; C5 (80) 8.03 / 7.52 / 7.26 / 7.24 / 7.67 ms.
    const double avg_deg = g.n > 0 ? (double)g.nnz / (double)g.n : 0.0;
    int push_iters = avg_deg >= 16.0 ? 3 : 1;
    if (o.flags & MIS2_FLAG_PUSH_DECIDE) push_iters = max_iters;
    if (o.flags & MIS2_FLAG_PULL_DECIDE) push_iters = 0;
    if (const char* e = getenv("MIS2_PUSH_ITERS")) push_iters = atoi(e);
    void* fn = pick_kernel(G, stats, push_iters > 0);
    if (!fn) {
        set_error("group must be one of 1,2,4,8,16,32 (got %d)", G);
        return MIS2_EINVAL;
    }
    // Skewed degree distributions (largest degree > 16x the average, on
    // graphs with 8n > 64 MB): neighbour ids are random, the gathers hit
    // L2 sector by sector and the hubs' words are the only reuse -- which
    // only the L1 can serve.  One reduction over rowptr (and a 24-byte
    // read) decides, before the launch: the 32-bit column keys (half the
    // gather bytes) and 3 blocks per SM instead of 4, the carve-out giving
    // the freed shared memory to L1 (C4: 72.9 -> 46.4 ms; 3 blocks on the
    // stencils: C2 358 -> 375 us, C3 5.41 -> 5.57 ms, C5 7.71 -> 8.59 ms).
    bool skewed = false, tested = false;
    unsigned long long md = 0;
    if ((double)g.n * 8.0 > 64.0 * 1048576.0) {
        tested = true;
        MIS2_CUDA_TRY(cudaMemsetAsync(w.maxdeg, 0, sizeof(unsigned long long), s));
        k_max_degree<<<(unsigned)(di.sms * 4), 256, 0, s>>>(g.n, g.rowptr, w.maxdeg);
        count_launch();
        MIS2_CUDA_TRY(cudaMemcpyAsync(&md, w.maxdeg, sizeof(md), cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
        skewed = (double)md > 16.0 * (double)g.nnz / (double)g.n;
    }
    // The small-tile kernels (160-row staging buffers, 35 KB per block
    // instead of 55) whenever a dense step of the chosen G fits them: every
    // step of a tested graph (G rows at the largest degree: C3), or the
    // average step of a skewed one (its hub rows are deferred anyway: C4)
    // -- the shared memory saved is L1 (C4 46.4 -> 37.9 ms, C3 5.29 -> 4.83
    // ms).  MIS2_SMALL_TILES=0/2: never / whenever the average step fits
    // (measurement knob).
    int smem = (int)sizeof(TileSmem);
    {
        int mode = 1;
        if (const char* e = getenv("MIS2_SMALL_TILES")) mode = atoi(e);
        const double step_avg = g.n > 0 ? (double)(kMB / G) * (double)g.nnz / (double)g.n : 0.0;
        const double step_max = (double)(kMB / G) * (double)md;
        const double cap = (double)tile_cap_small();
        const bool small = mode == 2 ? step_avg <= cap
                                     : mode == 1 && tested && (skewed ? step_avg <= cap : step_max + 8.0 <= cap);
        void* fs = small ? pick_kernel_small(G, stats, push_iters > 0) : nullptr;
        if (fs) {
            fn = fs;
            smem = tile_smem_small();
        }
    }
    MIS2_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    MIS2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kMB, smem));
    int skew_blocks = 3;  // MIS2_SKEW_BLOCKS: measurement knob
    if (const char* e = getenv("MIS2_SKEW_BLOCKS")) skew_blocks = atoi(e);
    if (skewed && per_sm > skew_blocks) per_sm = skew_blocks;
    if (per_sm < 1) {
        set_error("persistent kernel does not fit on an SM");
        return MIS2_EINTERNAL;
    }
    if (const char* env = getenv("MIS2_BLOCKS_PER_SM")) {  // tuning knob (measurement only)
        const int want_per_sm = atoi(env);
        if (want_per_sm >= 1 && want_per_sm < per_sm) per_sm = want_per_sm;
    }
    {
        // shared-memory carve-out: just what per_sm blocks need, the rest of
        // the 256 KB is L1 (MIS2_CARVEOUT=percent: measurement knob)
        int pct = (int)(((double)per_sm * (smem + 1024) * 100.0) / (228.0 * 1024.0) + 0.999);
        if (pct > 100) pct = 100;
        if (const char* e = getenv("MIS2_CARVEOUT")) pct = atoi(e);
        MIS2_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    }
    const int64_t max_grid = (int64_t)per_sm * di.sms;
    // small graphs: about two steps of rows per block
    const int64_t rpb = kMB / G;
    const int64_t want = (g.n + 2 * rpb - 1) / (2 * rpb);
    const int grid = (int)(want < 1 ? 1 : (want > max_grid ? max_grid : want));

    MIS2_CUDA_TRY(cudaMemsetAsync(w.ctrl, 0, 80 * sizeof(unsigned long long), s));
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
    // whose T does not fit L2 (C4 92 -> 77 ms).  Automatic: the skewed
    // graphs (above).
    // MIS2_FLAG_KEYS / MIS2_FLAG_NO_KEYS force (results identical).
    int keys = skewed ? 1 : 0;
    if (o.flags & MIS2_FLAG_KEYS) keys = 1;
    if (o.flags & MIS2_FLAG_NO_KEYS) keys = 0;
    if (const char* e = getenv("MIS2_KEYS")) keys = atoi(e);  // measurement knob
    if (o.flags & MIS2_FLAG_WORD32) keys = 0;  // the keys are the words' high halves
    if (sub) keys = 0;                          // key ties resolve to rows, M holds original ids
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
    const int64_t n_ids = sub ? sub->n_full : g.n;  // b of the whole graph (reading Q15)
    p.prio.b = bits_for(n_ids);
    p.prio.seed = o.seed;
    p.prio.hi_mask = ~((1ull << p.prio.b) - 1ull);
    p.id_mask = (uint32_t)((1ull << p.prio.b) - 1ull);
    p.prio.n = n_ids;
    p.gid = sub ? sub->gid : nullptr;
    p.inv = sub ? sub->inv : nullptr;
    p.l2_keep = l2_keep_for(g.nnz);
    // cyclic row ownership (mis2_kernel.cuh Rows); MIS2_CYCLIC=0: contiguous
    // ranges (measurement knob, results identical)
    p.cyclic = 1;
    if (const char* e = getenv("MIS2_CYCLIC")) p.cyclic = atoi(e) != 0;
    p.push_iters = push_iters;
    // Skewed graphs defer rows beyond one gather batch of their lane group
    // (G = 2 on C4: 32 entries) to the block's warps, whose coalesced row
    // loops beat the lane groups' on long rows (C4, batches 1 / 2 / 3 / 4 /
    // 8 / 16 / 32: 30.9-31.2 / 31.1-31.4 / 32.1 / 31.6 / 37.5 / 37.9 / 55.4
    // ms); the others keep 8 (C2's 27-entry rows at G = 1 need > 3; C5
    // unchanged).
    p.heavy_batches = skewed ? 1 : 0;
    p.gather_keep = skewed ? 1 : 0;
    // global queue of deferred rows (compiled into the G = 2 small-tile
    // kernels only: mis2_g2s.cu); MIS2_GQ_RT=0: off (measurement knob)
    p.gq = skewed ? w.gq : nullptr;
    if (const char* e = getenv("MIS2_GQ_RT")) p.gq = atoi(e) ? w.gq : nullptr;
    if (const char* e = getenv("MIS2_GATHER_KEEP")) p.gather_keep = atoi(e);  // measurement knob
    if (const char* e = getenv("MIS2_HEAVY_BATCHES_RT")) p.heavy_batches = atoi(e);  // measurement knob
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
