// cgs.cu -- Alg. 4 "Cluster Multicolor Gauss-Seidel" (§III-C):
// the colouring of the coarse graph (setup), the cluster / colour-set
// structure and the symmetric sweeps.
//
// Colouring (reading Q30): Jones-Plassmann rounds with the MIS-2 status
// words of iteration 0 as priorities -- in round r every uncoloured vertex
// whose word is below the words of all its neighbours uncoloured at the
// start of the round takes the smallest colour no earlier-coloured neighbour
// has.  Candidates of one round are never adjacent, so a round is one
// race-free pass (a vertex coloured in round r records r, and "uncoloured at
// the start of round r" = "coloured in round >= r").
//
// Sweeps: one launch per colour and direction; a warp per cluster of the
// colour walks the cluster's rows in order (ascending forward, descending
// backward); a row's residual r = b_i - A_i x is summed by the lanes
// (fixed order: lane-strided partial sums, then a tree), and lane 0 applies
// x_i += r / A_ii (reading Q31: the standard update; P:349's literal
// "x_i <- r/A_ii" double counts the diagonal).  Clusters of one colour share
// no edge, so they run concurrently without touching each other's x.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace mis2k {

// All rounds of the colouring in one cooperative launch (grid barrier
// between rounds): round 0 visits every vertex, later rounds the vertices
// left uncoloured (a worklist compacted with one atomic per warp, counts in a
// ring of three).  G lanes per row with batched gathers; the decision is the
// Jones-Plassmann rule of reading Q30: a vertex coloured in round r records r,
// so "uncoloured at the start of round r" is cround >= r and the round is
// race-free; the free colour comes from a 64-bit mask of the neighbours'
// colours, with a scan beyond 64.
struct ColorState {
    uint64_t* W;
    int32_t* cround;
    int32_t* color;
    int32_t* wl[2];
    unsigned int* bar;
    unsigned long long* cnt;  // [3] ring of worklist lengths
    int* maxc;
    int* err;
};

template <int G>
__global__ void __launch_bounds__(256, 5) k_color_persistent(int64_t n, const int64_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ colinds, Prio pr,
                                                          ColorState st) {
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & 31, grp = lane / G, sub = lane % G;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t fi0 = pr.iter_term(0);
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        st.W[v] = pr.word(0, fi0, v);
        st.cround[v] = 0x7fffffff;
        st.color[v] = -1;
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) st.cnt[threadIdx.x] = 0;
    grid_barrier(st.bar);
    const int32_t* cr = st.cround;
    const uint64_t* Wp = st.W;
    const int32_t* cl = st.color;
    int64_t m = n;
    for (int r = 0;; r++) {
        const int32_t* in = (r & 1) ? st.wl[1] : st.wl[0];  // no dynamic index into the parameter
        int32_t* out = (r & 1) ? st.wl[0] : st.wl[1];
        unsigned long long* ocnt = st.cnt + (r % 3);
        if (blockIdx.x == 0 && threadIdx.x == 0) st.cnt[(r + 1) % 3] = 0;
        int mc = -1;
        for (int64_t base = gwarp * RPW; base < m; base += nwarps * RPW) {
            const int64_t idx = base + grp;
            const bool valid = idx < m;
            int64_t v = 0, s = 0, e = 0;
            uint64_t wv = 0;
            if (valid) {
                v = (r == 0) ? idx : in[idx];
                s = rowptr[v];
                e = rowptr[v + 1];
                wv = st.W[v];
            }
            bool cand = true;
            uint64_t mask = 0;
            // batches of 8 entries per lane, three levels of independent
            // loads (column ids, rounds, then words or colours); a lane stops
            // at its first uncoloured neighbour with a smaller word
            if (valid)
                for (int64_t j0 = s + sub; j0 < e && cand; j0 += 8 * G) {
                    int32_t uu[8], ru[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int64_t j = j0 + (int64_t)q * G;
                        uu[q] = j < e ? colinds[j] : -1;
                    }
#pragma unroll
                    for (int q = 0; q < 8; q++) ru[q] = (uu[q] >= 0 && uu[q] != v) ? cr[uu[q]] : -1;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        if (ru[q] >= r) {
                            if (Wp[uu[q]] < wv) cand = false;
                        } else if (ru[q] >= 0) {
                            const int32_t cu = cl[uu[q]];
                            if (cu < 64) mask |= 1ull << cu;
                        }
                    }
                }
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const int oc = __shfl_xor_sync(kFull, (int)cand, off);  // every lane shuffles
                cand = cand && oc;
                mask |= __shfl_xor_sync(kFull, mask, off);
            }
            bool keep = false;
            if (valid && sub == 0) {
                if (cand) {
                    int32_t c;
                    if (mask != ~0ull) {
                        c = __ffsll((long long)~mask) - 1;
                    } else {  // more than 64 colours around: smallest free colour >= 64
                        c = 64;
                        for (;;) {
                            bool taken = false;
                            for (int64_t j = s; j < e && !taken; j++) {
                                const int32_t u = colinds[j];
                                if (u != v && st.cround[u] < r && st.color[u] == c) taken = true;
                            }
                            if (!taken) break;
                            c++;
                        }
                    }
                    st.color[v] = c;
                    st.cround[v] = r;
                    mc = max(mc, c);
                } else {
                    keep = true;
                }
            }
            const unsigned ball = __ballot_sync(kFull, keep);
            if (ball) {
                unsigned long long pos = 0;
                if (lane == 0) pos = atomicAdd(ocnt, (unsigned long long)__popc(ball));
                pos = __shfl_sync(kFull, pos, 0);
                if (keep) out[pos + __popc(ball & lanemask_lt())] = (int32_t)v;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mc = max(mc, __shfl_xor_sync(kFull, mc, off));
        if (lane == 0 && mc >= 0) atomicMax(st.maxc, mc);
        grid_barrier(st.bar);
        m = (int64_t)*(volatile unsigned long long*)ocnt;
        if (m == 0) break;
        if (r > n + 2) {  // every round colours at least the least uncoloured word
            if (blockIdx.x == 0 && threadIdx.x == 0) *st.err = 1;
            break;
        }
    }
}

// rows per cluster (pass 1) / placed at an atomically reserved slot (pass 2);
// lanes of a warp with the same key share one atomic (__match_any_sync: a
// colour histogram has ~20 keys for 10^6 entries)
__global__ void k_count_i32(int64_t n, const int32_t* __restrict__ key, unsigned long long* __restrict__ cnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const int32_t k = i < n ? key[i] : -1;
        const unsigned m = __match_any_sync(kFull, k);
        if (k >= 0 && !(m & lanemask_lt())) atomicAdd(&cnt[k], (unsigned long long)__popc(m));
    }
}
__global__ void k_scatter_i32(int64_t n, const int32_t* __restrict__ key, unsigned long long* __restrict__ cursor,
                              int32_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const int32_t k = i < n ? key[i] : -1;
        const unsigned m = __match_any_sync(kFull, k);
        const int leader = __ffs(m) - 1;
        unsigned long long pos = 0;
        if (k >= 0 && lane == leader) pos = atomicAdd(&cursor[k], (unsigned long long)__popc(m));
        pos = __shfl_sync(kFull, pos, leader);
        if (k >= 0) out[pos + __popc(m & lanemask_lt())] = (int32_t)i;
    }
}
// ascending rows inside each cluster: block bitonic of the segment in shared memory
constexpr int kSegMax = 4096;
__global__ void k_sort_segments(int64_t na, const int64_t* __restrict__ ptr, int32_t* __restrict__ rows, int* err) {
    __shared__ int32_t x[kSegMax];
    for (int64_t a = blockIdx.x; a < na; a += gridDim.x) {
        const int64_t s = ptr[a], len = ptr[a + 1] - s;
        if (len <= 1) continue;
        if (len > kSegMax) {
            if (threadIdx.x == 0) atomicOr(err, 1);
            continue;
        }
        int P = 1;
        while (P < len) P <<= 1;
        for (int i = threadIdx.x; i < P; i += blockDim.x) x[i] = i < len ? rows[s + i] : 0x7fffffff;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
                    const int lo = 2 * i - (i & (j - 1)), hi = lo + j;
                    const bool up = (lo & k) == 0;
                    const int32_t p = x[lo], q = x[hi];
                    if ((p > q) == up) {
                        x[lo] = q;
                        x[hi] = p;
                    }
                }
                __syncthreads();
            }
        for (int i = threadIdx.x; i < len; i += blockDim.x) rows[s + i] = x[i];
        __syncthreads();
    }
}
__global__ void k_diag(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                       const double* __restrict__ vals, double* __restrict__ diag, int* err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int64_t j = rowptr[i]; j < rowptr[i + 1]; j++)
            if (colinds[j] == i) d = vals[j];
        diag[i] = d;
        if (d == 0.0) atomicOr(err, 2);
    }
}
__global__ void k_iota(int64_t n, int32_t* __restrict__ x, int64_t* __restrict__ ptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) x[i] = (int32_t)i;
        ptr[i] = i;
    }
}

// One colour of a sweep: a warp per cluster of the colour.  The structure
// of the next row (its index, bounds, first 32 column ids and values, b_i,
// A_ii) is loaded while the current row gathers x, so a row costs one
// dependent gather + the lane reduction.
__global__ void k_cgs_color(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                            const double* __restrict__ vals, const double* __restrict__ diag,
                            const int64_t* __restrict__ cptr, const int32_t* __restrict__ crows,
                            const int32_t* __restrict__ cset, int64_t set_lo, int64_t set_hi,
                            const double* __restrict__ b, double* __restrict__ x, int backward) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = set_lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < set_hi; k += nw) {
        const int32_t a = cset[k];
        const int64_t r0 = cptr[a], r1 = cptr[a + 1], nr = r1 - r0;
        auto row_at = [&](int64_t t) { return (int64_t)crows[backward ? r1 - 1 - t : r0 + t]; };
        // structure of row t (lane-distributed first 32 entries)
        int64_t i = 0, s = 0, e = 0;
        int32_t cj = 0;
        double vj = 0.0, bi = 0.0, di = 1.0;
        auto load = [&](int64_t t, int64_t& ii, int64_t& ss, int64_t& ee, int32_t& c, double& v, double& bb,
                        double& dd) {
            ii = row_at(t);
            ss = rowptr[ii];
            ee = rowptr[ii + 1];
            c = 0;
            v = 0.0;
            if (ss + lane < ee) {
                c = colinds[ss + lane];
                v = vals[ss + lane];
            }
            bb = b[ii];
            dd = diag[ii];
        };
        if (nr > 0) load(0, i, s, e, cj, vj, bi, di);
        for (int64_t t = 0; t < nr; t++) {
            int64_t i2 = 0, s2 = 0, e2 = 0;
            int32_t cj2 = 0;
            double vj2 = 0.0, bi2 = 0.0, di2 = 1.0;
            if (t + 1 < nr) load(t + 1, i2, s2, e2, cj2, vj2, bi2, di2);
            double acc = (s + lane < e) ? vj * x[cj] : 0.0;
            for (int64_t j = s + 32 + lane; j < e; j += 32) acc += vals[j] * x[colinds[j]];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
            if (lane == 0) x[i] = x[i] + (bi - acc) / di;
            __syncwarp();
            i = i2;
            s = s2;
            e = e2;
            cj = cj2;
            vj = vj2;
            bi = bi2;
            di = di2;
        }
    }
}

// Point multicolor GS (every cluster one row): a thread per row of the colour.
// Point GS, one colour: G lanes per row (coalesced row reads, 8 independent
// gathers of x in flight per lane), lane-strided partial sums added by a
// shuffle tree (fixed order, so the sweep is deterministic).
template <int G>
__global__ void k_pgs_color(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                            const double* __restrict__ vals, const double* __restrict__ diag,
                            const int32_t* __restrict__ cset, int64_t set_lo, int64_t set_hi,
                            const double* __restrict__ b, double* __restrict__ x) {
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & 31, grp = lane / G, sub = lane % G;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = set_lo + gwarp * RPW; base < set_hi; base += nwarps * RPW) {
        const int64_t k = base + grp;
        const bool valid = k < set_hi;
        int64_t i = 0;
        double acc = 0.0;
        if (valid) {
            i = cset[k];
            const int64_t s = rowptr[i], e = rowptr[i + 1];
            for (int64_t j0 = s + sub; j0 < e; j0 += 8 * G) {
                int32_t c[8];
                double a[8], xv[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int64_t j = j0 + (int64_t)q * G;
                    c[q] = j < e ? colinds[j] : -1;
                    a[q] = j < e ? vals[j] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; q++) xv[q] = c[q] >= 0 ? x[c[q]] : 0.0;
#pragma unroll
                for (int q = 0; q < 8; q++) acc += a[q] * xv[q];
            }
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
        if (valid && sub == 0) x[i] = x[i] + (b[i] - acc) / diag[i];
    }
}

}  // namespace mis2k

using namespace mis2h;
using namespace mis2k;

struct mis2_cgs {
    int64_t n = 0, na = 0;
    int32_t ncolors = 0;
    bool point = false;
    mis2_graph g{};
    const double* vals = nullptr;
    std::vector<void*> allocs;
    double* diag = nullptr;
    int64_t* cptr = nullptr;   // [na+1] rows of cluster a: crows[cptr[a] .. cptr[a+1])
    int32_t* crows = nullptr;  // [n] ascending inside a cluster
    int32_t* cset = nullptr;   // [na] clusters grouped by colour
    std::vector<int64_t> csptr;  // host [ncolors+1]
};

namespace {

int cgs_alloc(mis2_cgs* h, void** p, size_t bytes) {
    MIS2_CUDA_TRY(cudaMalloc(p, bytes < 256 ? 256 : bytes));
    h->allocs.push_back(*p);
    return MIS2_OK;
}

unsigned grid_for(int64_t n, int sms) {
    int64_t b = (n + 255) / 256;
    if (b > (int64_t)sms * 16) b = (int64_t)sms * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

// the colouring (reading Q30); scratch carved from the caller's workspace
// (bytes_needed != NULL: sizing pass only)
int mis2h::color_graph(const mis2_graph& g, uint64_t seed, int32_t* color, int32_t* ncolors, void* ws, size_t ws_bytes,
                cudaStream_t s, size_t* bytes_needed) {
    const int64_t n = g.n;
    ColorState st;
    Carve c(ws, ws_bytes);
    st.W = c.take<uint64_t>((size_t)n + 1);
    st.cround = c.take<int32_t>((size_t)n + 1);
    st.wl[0] = c.take<int32_t>((size_t)n + 1);
    st.wl[1] = c.take<int32_t>((size_t)n + 1);
    char* ctr = c.take<char>(256);
    if (bytes_needed) {
        *bytes_needed = c.off;
        return MIS2_OK;
    }
    if (!c.ok()) {
        set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
        return MIS2_ENOMEM;
    }
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    if (n == 0) {
        *ncolors = 0;
        return MIS2_OK;
    }
    MIS2_CUDA_TRY(cudaMemsetAsync(ctr, 0, 256, s));
    st.color = color;
    st.bar = (unsigned int*)ctr;
    st.cnt = (unsigned long long*)(ctr + 64);
    st.maxc = (int*)(ctr + 128);
    st.err = (int*)(ctr + 132);
    MIS2_CUDA_TRY(cudaMemsetAsync(st.maxc, 0xff, sizeof(int), s));  // -1
    Prio pr{};
    pr.scheme = MIS2_SCHEME_XORSTAR;
    pr.b = bits_for(n);
    pr.seed = seed;
    pr.hi_mask = ~((1ull << pr.b) - 1ull);
    pr.n = n;
    const int G = choose_group(n, g.nnz, 0);
    void* fn;
    switch (G) {
        case 1: fn = (void*)k_color_persistent<1>; break;
        case 2: fn = (void*)k_color_persistent<2>; break;
        case 4: fn = (void*)k_color_persistent<4>; break;
        case 8: fn = (void*)k_color_persistent<8>; break;
        case 16: fn = (void*)k_color_persistent<16>; break;
        default: fn = (void*)k_color_persistent<32>; break;
    }
    int per_sm = 0;
    MIS2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
    int64_t grid = (int64_t)per_sm * di.sms;
    const int64_t need = (n + (256 / G) - 1) / (256 / G);
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    const mis2_graph gg = g;
    int64_t nn = n;
    void* args[] = {&nn, (void*)&gg.rowptr, (void*)&gg.colinds, &pr, &st};
    MIS2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(256), args, 0, s));
    count_launch();
    int hv[2] = {-1, 0};
    int rc = MIS2_OK;
    MIS2_CUDA_TRY(cudaMemcpyAsync(hv, st.maxc, sizeof(hv), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    if (hv[1]) {
        set_error("colouring did not terminate");
        rc = MIS2_EINTERNAL;
    } else {
        *ncolors = hv[0] + 1;
    }
    return rc;
}


extern "C" {

int mis2_color(const mis2_graph* g, uint64_t seed, int32_t* color, int32_t* ncolors, void* ws, size_t ws_bytes,
               void* stream) {
    reset_launches();
    if (!g || !ncolors || g->n < 0 || (g->n > 0 && (!color || !g->rowptr || !ws)) || g->n > 2147483645LL ||
        (g->rowptr_bits != 0 && g->rowptr_bits != 64)) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    return color_graph(*g, seed, color, ncolors, ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

int mis2_cgs_setup(const mis2_graph* g, const double* vals, const int32_t* labels, int64_t num_aggs,
                   const mis2_graph* coarse, uint64_t seed, mis2_cgs** out, void* stream) {
    reset_launches();
    if (!g || !out || g->n < 0 || (g->n > 0 && (!vals || !g->rowptr || !g->colinds)) ||
        (labels && (!coarse || num_aggs < 1 || coarse->n != num_aggs)) || g->n > 2147483645LL ||
        (g->rowptr_bits != 0 && g->rowptr_bits != 64) || (coarse && coarse->rowptr_bits != 0 && coarse->rowptr_bits != 64)) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    mis2_cgs* h = new mis2_cgs();
    h->n = g->n;
    h->g = *g;
    h->vals = vals;
    const bool point = labels == nullptr;
    h->point = point;
    h->na = point ? g->n : num_aggs;
    const int64_t n = h->n, na = h->na;
    auto fail = [&](int rc) {
        mis2_cgs_destroy(h);
        return rc;
    };
    void* p;
    int* err;
    int rc;
    int32_t* ccolor;
    unsigned long long* cnt;
    void* tmp;
    void* cws;
    size_t cws_bytes = 0;
    const int64_t nk = std::max<int64_t>(na, 64) + 2;
    const mis2_graph& cg = point ? *g : *coarse;
    if ((rc = color_graph(cg, seed, nullptr, nullptr, nullptr, 0, s, &cws_bytes)) != MIS2_OK) return fail(rc);
    // one allocation (owned by the handle) for its arrays and the setup
    // scratch, including the colouring's
    auto layout = [&](Carve& c) {
        cws = c.take<char>(cws_bytes);
        h->diag = c.take<double>((size_t)n + 1);
        h->cptr = c.take<int64_t>((size_t)na + 2);
        h->crows = c.take<int32_t>((size_t)n + 1);
        h->cset = c.take<int32_t>((size_t)na + 1);
        err = c.take<int>(16);
        ccolor = c.take<int32_t>((size_t)na + 1);
        cnt = c.take<unsigned long long>((size_t)nk);
        tmp = c.take<char>(scan64_ws_bytes(nk));
    };
    Carve dry(nullptr, 0);
    layout(dry);
    if ((rc = cgs_alloc(h, &p, dry.off)) != MIS2_OK) return fail(rc);
    Carve cv(p, dry.off);
    layout(cv);
    if (cudaMemsetAsync(err, 0, 64, s) != cudaSuccess) return fail(MIS2_ECUDA);
    if (n) {
        k_diag<<<grid_for(n, di.sms), 256, 0, s>>>(n, g->rowptr, g->colinds, vals, h->diag, err);
        count_launch();
    }
    // colour the coarse graph (point: the graph itself)
    if ((rc = color_graph(cg, seed, ccolor, &h->ncolors, cws, cws_bytes, s, nullptr)) != MIS2_OK) return fail(rc);
    // rows of each cluster, ascending
    if (point) {
        k_iota<<<grid_for(n + 1, di.sms), 256, 0, s>>>(n, h->crows, h->cptr);
        count_launch();
    } else if (n) {
        if (cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * nk, s) != cudaSuccess) return fail(MIS2_ECUDA);
        k_count_i32<<<grid_for(n, di.sms), 256, 0, s>>>(n, labels, cnt);
        count_launch();
        if ((rc = scan_counts64((const int64_t*)cnt, na, h->cptr, tmp, s)) != MIS2_OK) return fail(rc);
        if (cudaMemcpyAsync(cnt, h->cptr, sizeof(int64_t) * na, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return fail(MIS2_ECUDA);
        k_scatter_i32<<<grid_for(n, di.sms), 256, 0, s>>>(n, labels, cnt, h->crows);
        k_sort_segments<<<(unsigned)std::min<int64_t>(na, (int64_t)di.sms * 8), 256, 0, s>>>(na, h->cptr, h->crows, err);
        count_launch(2);
    }
    // clusters grouped by colour
    if (na) {
        if (cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * nk, s) != cudaSuccess) return fail(MIS2_ECUDA);
        k_count_i32<<<grid_for(na, di.sms), 256, 0, s>>>(na, ccolor, cnt);
        count_launch();
        std::vector<unsigned long long> hc(h->ncolors);
        if (cudaMemcpyAsync(hc.data(), cnt, sizeof(unsigned long long) * h->ncolors, cudaMemcpyDeviceToHost, s) !=
                cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fail(MIS2_ECUDA);
        h->csptr.assign(h->ncolors + 1, 0);
        for (int c = 0; c < h->ncolors; c++) h->csptr[c + 1] = h->csptr[c] + (int64_t)hc[c];
        if (cudaMemcpyAsync(cnt, h->csptr.data(), sizeof(int64_t) * h->ncolors, cudaMemcpyHostToDevice, s) !=
            cudaSuccess)
            return fail(MIS2_ECUDA);
        k_scatter_i32<<<grid_for(na, di.sms), 256, 0, s>>>(na, ccolor, cnt, h->cset);
        count_launch();
    }
    int herr = 0;
    if (cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(MIS2_ECUDA);
    if (herr & 2) {
        set_error("a diagonal entry A_ii is missing or zero");
        return fail(MIS2_EINVAL);
    }
    if (herr & 1) {
        set_error("a cluster has more than %d rows", kSegMax);
        return fail(MIS2_EINTERNAL);
    }
    *out = h;
    return MIS2_OK;
}

int mis2_cgs_ncolors(const mis2_cgs* h) { return h ? h->ncolors : -1; }

int mis2_cgs_apply(mis2_cgs* h, const double* b, double* x, int sweeps, int direction, void* stream) {
    reset_launches();
    if (!h || sweeps < 0 || direction < 0 || direction > 2 || (h->n > 0 && (!b || !x))) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    for (int sw = 0; sw < sweeps; sw++) {
        for (int pass = 0; pass < 2; pass++) {
            if (pass == 1 && direction != 0) break;
            const int backward = (direction == 2) || (direction == 0 && pass == 1);
            for (int ci = 0; ci < h->ncolors; ci++) {
                const int c = backward ? h->ncolors - 1 - ci : ci;
                const int64_t lo = h->csptr[c], hi = h->csptr[c + 1];
                if (hi <= lo) continue;
                if (h->point) {  // a thread per row
                    const double avg = h->n ? (double)h->g.nnz / (double)h->n : 0.0;
                    const int G = avg < 4 ? 1 : avg < 8 ? 2 : avg < 16 ? 4 : avg < 40 ? 8 : avg < 100 ? 16 : 32;
                    int64_t blocks = ((hi - lo) * G + 255) / 256;
                    if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
                    if (blocks < 1) blocks = 1;
                    const dim3 gb((unsigned)blocks), tb(256);
                    switch (G) {
                        case 1: k_pgs_color<1><<<gb, tb, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag, h->cset, lo, hi, b, x); break;
                        case 2: k_pgs_color<2><<<gb, tb, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag, h->cset, lo, hi, b, x); break;
                        case 4: k_pgs_color<4><<<gb, tb, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag, h->cset, lo, hi, b, x); break;
                        case 8: k_pgs_color<8><<<gb, tb, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag, h->cset, lo, hi, b, x); break;
                        case 16: k_pgs_color<16><<<gb, tb, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag, h->cset, lo, hi, b, x); break;
                        default: k_pgs_color<32><<<gb, tb, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag, h->cset, lo, hi, b, x); break;
                    }
                } else {
                    int64_t blocks = (hi - lo + 7) / 8;  // 8 warps per block, a warp per cluster
                    if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
                    k_cgs_color<<<(unsigned)blocks, 256, 0, s>>>(h->g.rowptr, h->g.colinds, h->vals, h->diag,
                                                                 h->cptr, h->crows, h->cset, lo, hi, b, x, backward);
                }
                count_launch();
            }
        }
    }
    MIS2_CUDA_TRY(cudaGetLastError());
    return MIS2_OK;
}

int mis2_cgs_destroy(mis2_cgs* h) {
    if (!h) return MIS2_OK;
    for (void* p : h->allocs) cudaFree(p);
    delete h;
    return MIS2_OK;
}

}  // extern "C"
