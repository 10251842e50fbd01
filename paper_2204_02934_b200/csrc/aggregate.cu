// aggregate.cu -- Alg. 3 "MIS-2 based Aggregation" (§III-B) on
// the device.  Both MIS-2 calls run the persistent kernel of mis2_core.cu;
// the phase bookkeeping is a handful of row-parallel kernels (G lanes per
// CSR row, as in the MIS-2 passes) plus two exclusive scans that number the
// aggregates in ascending root order (reading Q18).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace mis2k {

enum AggErr : int { kErrTwoRoots = 1, kErrPhase2Conflict = 2, kErrNoCandidate = 4 };

// warp-uniform loop over rows, G lanes per row
#define ROWS_BEGIN(G, n)                                                                   \
    constexpr int RPW = 32 / (G);                                                          \
    const int lane = threadIdx.x & 31, grp = lane / (G), sub = lane % (G);                 \
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);                         \
    const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);    \
    for (int64_t base = gwarp * RPW; base < (n); base += nwarps * RPW) {                   \
        const int64_t v = base + grp;                                                      \
        const bool valid = v < (n);

#define ROWS_END }

constexpr int kBatch = 8;  // gathers in flight per lane (row_batched)

// Phase 1: roots = MIS-2; every root and its neighbours get the
// root's id (pull form: each vertex looks for its unique root neighbour).
template <int G>
__global__ void k_phase1(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                         const uint8_t* __restrict__ in1, const int32_t* __restrict__ rid,
                         int32_t* __restrict__ labels, int32_t* __restrict__ roots, int* err) {
    ROWS_BEGIN(G, n)
    int found = -1;
    int bad = 0;
    const bool root = valid && in1[v];
    if (valid && !root)
        row_batched<G, kBatch>(rowptr[v], rowptr[v + 1], sub, colinds, [&](int32_t w) { return in1[w]; },
                               [&](int32_t w, uint8_t x) {
                                   if (w != v && x) {
                                       const int r = rid[w];
                                       if (found >= 0 && found != r) bad = 1;
                                       found = r;
                                   }
                               });
    // combine: all lanes that found a root must agree (roots are >= 3 apart)
    int mx = found, mn = found < 0 ? 0x7fffffff : found;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        mx = max(mx, __shfl_xor_sync(kFull, mx, off));
        mn = min(mn, __shfl_xor_sync(kFull, mn, off));
    }
    bad = group_or<G>(bad);
    if (valid && sub == 0) {
        if (root) {
            labels[v] = rid[v];
            if (roots) roots[rid[v]] = (int32_t)v;
        } else {
            labels[v] = mx;  // -1 when no root neighbour (UNAGG)
            if (bad || (mx >= 0 && mn != mx)) atomicOr(err, kErrTwoRoots);
        }
    }
    ROWS_END
}

// Phase 2 accept rule (reading Q16): an M2 root is accepted iff it has
// >= 2 neighbours w != v that are unaggregated after phase 1.
template <int G>
__global__ void k_phase2_accept(int64_t n, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ colinds, const uint8_t* __restrict__ in2,
                                const int32_t* __restrict__ labels, uint8_t* __restrict__ acc) {
    ROWS_BEGIN(G, n)
    const bool r = valid && in2[v];
    int cnt = 0;
    if (r)
        row_batched<G, kBatch>(rowptr[v], rowptr[v + 1], sub, colinds, [&](int32_t w) { return labels[w]; },
                               [&](int32_t w, int32_t x) { cnt += (w != v && x < 0); });
    cnt = group_sum<G>(cnt);
    if (valid && sub == 0) acc[v] = (r && cnt >= 2) ? 1 : 0;
    ROWS_END
}

// Phase 2 labels (reading Q17): accepted root v gets id n1 + aid[v];
// its unaggregated neighbours join it (pull form).
template <int G>
__global__ void k_phase2_label(int64_t n, const int64_t* __restrict__ rowptr,
                               const int32_t* __restrict__ colinds, const uint8_t* __restrict__ acc,
                               const int32_t* __restrict__ aid, const int32_t* __restrict__ d_n1,
                               int32_t* __restrict__ labels, int32_t* __restrict__ roots, int* err) {
    const int32_t n1 = *d_n1;
    ROWS_BEGIN(G, n)
    const bool un = valid && labels[v] < 0;
    const bool root = un && acc[v];
    int found = -1, bad = 0;
    if (un && !root)
        row_batched<G, kBatch>(rowptr[v], rowptr[v + 1], sub, colinds, [&](int32_t w) { return acc[w]; },
                               [&](int32_t w, uint8_t x) {
                                   if (w != v && x) {
                                       if (found >= 0 && found != aid[w]) bad = 1;
                                       found = aid[w];
                                   }
                               });
    int mx = found, mn = found < 0 ? 0x7fffffff : found;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        mx = max(mx, __shfl_xor_sync(kFull, mx, off));
        mn = min(mn, __shfl_xor_sync(kFull, mn, off));
    }
    bad = group_or<G>(bad);
    if (un && sub == 0) {
        if (root) {
            labels[v] = n1 + aid[v];
            if (roots) roots[n1 + aid[v]] = (int32_t)v;
        } else if (mx >= 0) {
            labels[v] = n1 + mx;
            if (bad || mn != mx) atomicOr(err, kErrPhase2Conflict);
        }
    }
    ROWS_END
}

// tent <- labels; aggsize(a) <- |{v : tent_v = a}|
__global__ void k_tent_size(int64_t n, const int32_t* __restrict__ labels, int32_t* __restrict__ tent,
                            int32_t* __restrict__ size, unsigned long long* leftovers) {
    int cnt = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = labels[v];
        tent[v] = a;
        if (a >= 0) atomicAdd(&size[a], 1);
        else cnt++;
    }
    cnt = group_sum<32>(cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(leftovers, (unsigned long long)cnt);
}

// candidate order for phase 3: larger coupling, then smaller aggsize, then
// smaller aggregate id (reading Q19)
__device__ __forceinline__ bool better(int c1, int s1, int a1, int c2, int s2, int a2) {
    if (a2 < 0) return a1 >= 0;
    if (a1 < 0) return false;
    if (c1 != c2) return c1 > c2;
    if (s1 != s2) return s1 < s2;
    return a1 < a2;
}

template <int G>
__device__ __forceinline__ void group_best(int& c, int& s, int& a) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        const int c2 = __shfl_xor_sync(kFull, c, off), s2 = __shfl_xor_sync(kFull, s, off),
                  a2 = __shfl_xor_sync(kFull, a, off);
        if (better(c2, s2, a2, c, s, a)) { c = c2; s = s2; a = a2; }
    }
}

constexpr int kHeavyDeg = 512;
#ifndef MIS2_P3LIST
#define MIS2_P3LIST 8
#endif
// distinct candidate aggregates kept per lane in phase 3 (C5 aggregation
// 18.4 / 20.4 / 26.1 ms with 8 / 12 / 16: register pressure beyond 8)
constexpr int kP3List = MIS2_P3LIST;

// Phase 3 for leftover rows of degree <= kHeavyDeg: each lane
// takes candidate entries and counts their coupling over the whole row.
template <int G>
__global__ void k_phase3(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                         const int32_t* __restrict__ tent, const int32_t* __restrict__ size,
                         int32_t* __restrict__ labels, int32_t* __restrict__ heavy, int* heavy_cnt, int* err) {
    ROWS_BEGIN(G, n)
    const bool left = valid && tent[v] < 0;
    int64_t s = 0, e = 0;
    if (left) { s = rowptr[v]; e = rowptr[v + 1]; }
    const bool is_heavy = left && (e - s) > kHeavyDeg;
    int bc = 0, bs = 0, ba = -1;
    bool done = false;
    {
        // one pass: each lane keeps the distinct candidate aggregates of its
        // entries (stride G) and their couplings in registers (a leftover sees
        // few aggregates); the group then adds up the lanes' counts by
        // shuffles.  A lane with more than 8 -> the group takes the quadratic
        // pass below.
        int32_t lab[kP3List];
        int cnt[kP3List];
        int nl = 0;
        bool overflow = false;
#pragma unroll
        for (int q = 0; q < kP3List; q++) {
            lab[q] = -1;
            cnt[q] = 0;
        }
        if (left && !is_heavy) {
            for (int64_t j0 = s + sub; j0 < e; j0 += 8 * G) {
                int32_t aa[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int64_t j = j0 + (int64_t)u * G;
                    aa[u] = -1;
                    if (j < e) {
                        const int32_t w = colinds[j];
                        aa[u] = (w != v) ? tent[w] : -1;
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int32_t a = aa[u];
                    if (a < 0) continue;
                    bool found = false;
#pragma unroll
                    for (int q = 0; q < kP3List; q++)
                        if (lab[q] == a) {
                            cnt[q]++;
                            found = true;
                        }
                    if (!found) {
                        if (nl < kP3List) {
#pragma unroll
                            for (int q = 0; q < kP3List; q++)
                                if (q == nl) {
                                    lab[q] = a;
                                    cnt[q] = 1;
                                }
                            nl++;
                        } else {
                            overflow = true;
                        }
                    }
                }
            }
        }
        int tot[kP3List];
#pragma unroll
        for (int q = 0; q < kP3List; q++) tot[q] = cnt[q];
#pragma unroll 1
        for (int r = 1; r < G; r++) {
            overflow |= __shfl_xor_sync(kFull, (int)overflow, r) != 0;
#pragma unroll
            for (int q2 = 0; q2 < kP3List; q2++) {
                const int32_t l2 = __shfl_xor_sync(kFull, lab[q2], r);
                const int c2 = __shfl_xor_sync(kFull, cnt[q2], r);
#pragma unroll
                for (int q = 0; q < kP3List; q++)
                    if (l2 >= 0 && lab[q] == l2) tot[q] += c2;
            }
        }
        if (left && !is_heavy && !overflow) {
#pragma unroll
            for (int q = 0; q < kP3List; q++)
                if (q < nl) {
                    const int sz = size[lab[q]];
                    if (better(tot[q], sz, lab[q], bc, bs, ba)) { bc = tot[q]; bs = sz; ba = lab[q]; }
                }
            done = true;
        }
    }
    if (left && !is_heavy && !done) {
        for (int64_t j = s + sub; j < e; j += G) {
            const int32_t u = colinds[j];
            const int32_t a = (u != v) ? tent[u] : -1;
            if (a < 0) continue;
            int c = 0;
            for (int64_t k = s; k < e; k++) {
                const int32_t x = colinds[k];
                c += (x != v && tent[x] == a);
            }
            const int sz = size[a];
            if (better(c, sz, a, bc, bs, ba)) { bc = c; bs = sz; ba = a; }
        }
    }
    group_best<G>(bc, bs, ba);
    if (left && sub == 0) {
        if (is_heavy) {
            heavy[atomicAdd(heavy_cnt, 1)] = (int32_t)v;
        } else if (ba < 0) {
            atomicOr(err, kErrNoCandidate);  // impossible by maximality of M1 (Q20)
        } else {
            labels[v] = ba;
        }
    }
    ROWS_END
}

// Phase 3 for heavy leftover rows: one block per row, coupling counted in a
// shared-memory hash table; labels are split into hash passes so any number
// of distinct candidates fits.
constexpr int kHashSlots = 4096;
// left != NULL (list form): heavy[] holds leftover-list positions, the
// choice goes to choice[position]; else heavy[] holds vertices -> labels.
__global__ void k_phase3_heavy(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                               const int32_t* __restrict__ tent, const int32_t* __restrict__ size,
                               int32_t* __restrict__ labels, const int32_t* __restrict__ heavy,
                               const int* heavy_cnt, int* err, const int32_t* __restrict__ left = nullptr,
                               int32_t* __restrict__ choice = nullptr) {
    __shared__ int32_t keys[kHashSlots];
    __shared__ int32_t cnts[kHashSlots];
    __shared__ int s_c[32], s_s[32], s_a[32];
    const int nh = *heavy_cnt;
    for (int h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t v = left ? left[heavy[h]] : heavy[h];
        const int64_t s = rowptr[v], e = rowptr[v + 1];
        const int64_t d = e - s;
        const int passes = (int)((d + kHashSlots / 2 - 1) / (kHashSlots / 2));
        int bc = 0, bs = 0, ba = -1;
        for (int pass = 0; pass < passes; pass++) {
            for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) { keys[i] = -1; cnts[i] = 0; }
            __syncthreads();
            for (int64_t j = s + threadIdx.x; j < e; j += blockDim.x) {
                const int32_t u = colinds[j];
                if (u == v) continue;
                const int32_t a = tent[u];
                if (a < 0) continue;
                const uint32_t hsh = (uint32_t)a * 2654435761u;
                if ((int)(hsh % (uint32_t)passes) != pass) continue;
                uint32_t slot = (hsh >> 7) & (kHashSlots - 1);
                for (;;) {
                    const int32_t prev = atomicCAS(&keys[slot], -1, a);
                    if (prev == -1 || prev == a) { atomicAdd(&cnts[slot], 1); break; }
                    slot = (slot + 1) & (kHashSlots - 1);
                }
            }
            __syncthreads();
            for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) {
                const int32_t a = keys[i];
                if (a >= 0) {
                    const int c = cnts[i], sz = size[a];
                    if (better(c, sz, a, bc, bs, ba)) { bc = c; bs = sz; ba = a; }
                }
            }
            __syncthreads();
        }
        group_best<32>(bc, bs, ba);
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) { s_c[warp] = bc; s_s[warp] = bs; s_a[warp] = ba; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                if (better(s_c[w], s_s[w], s_a[w], bc, bs, ba)) { bc = s_c[w]; bs = s_s[w]; ba = s_a[w]; }
            if (left) choice[heavy[h]] = ba;  // checked by k_scatter_choice
            else if (ba < 0) atomicOr(err, kErrNoCandidate);
            else labels[v] = ba;
        }
        __syncthreads();
    }
}

// Alg. 2 join: a vertex left unaggregated by phase 1 joins the
// aggregate of its smallest-id aggregated neighbour ("any neighbor", made
// deterministic -- reading Q28).
template <int G>
__global__ void k_basic_join(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                             const int32_t* __restrict__ tent, int32_t* __restrict__ labels, int* err) {
    ROWS_BEGIN(G, n)
    const bool left = valid && tent[v] < 0;
    int best = 0x7fffffff;
    if (left)
        for (int64_t j = rowptr[v] + sub; j < rowptr[v + 1]; j += G) {
            const int32_t u = colinds[j];
            if (u != v && tent[u] >= 0 && u < best) best = u;
        }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(kFull, best, off));
    if (left && sub == 0) {
        if (best == 0x7fffffff) atomicOr(err, kErrNoCandidate);  // impossible by maximality
        else labels[v] = tent[best];
    }
    ROWS_END
}

__global__ void k_finish(const int32_t* d_n1, const int32_t* d_n2, int64_t* out_na) {
    *out_na = (int64_t)*d_n1 + (int64_t)*d_n2;
}

// ---------------------------------------------------------------- list forms
// Single-GPU Alg. 3 works from ordered lists of roots instead of passes over
// all n rows: the roots push their aggregate id to their neighbours (roots
// are >= 3 apart, so no vertex is pushed twice -- checked), only the phase-2
// roots count their unaggregated neighbours, the aggregate sizes come out of
// the pushes (no histogram), and phase 3 visits the listed leftovers, whose
// choices are written by list position and scattered afterwards (so phase 3
// reads the labels themselves, frozen, and no copy of them is made).  A
// group of GL lanes takes one list entry at a time (GL from the average
// degree: short rows fill a warp with several entries); the groups of the
// grid stride over the list; list lengths are device scalars.
constexpr int kListWarps = 8;  // warps per block of the list kernels

template <int GL>
struct ListIdx {
    int64_t first, stride;
    int sub;
    __device__ __forceinline__ ListIdx() {
        const int64_t gid = (int64_t)blockIdx.x * (kListWarps * 32 / GL) + threadIdx.x / GL;
        first = gid;
        stride = (int64_t)gridDim.x * (kListWarps * 32 / GL);
        sub = threadIdx.x % GL;
    }
};
// every lane of a warp runs the same number of loop trips (the shuffles need
// the whole warp): the trip bound is the warp's largest group index
template <int GL>
__device__ __forceinline__ int64_t warp_trips(const ListIdx<GL>& li, int64_t cnt) {
    const int64_t wfirst = li.first - (int64_t)((threadIdx.x & 31) / GL);  // group 0 of this warp
    return cnt > wfirst ? (cnt - wfirst + li.stride - 1) / li.stride : 0;
}

// Phase 1: root R[i] gets aggregate i (ascending vertex order,
// Q18) and so do its neighbours; size[i] = 1 + |adj(R[i])|.  labels must be
// -1 (UNAGG) beforehand.
template <int GL>
__global__ void __launch_bounds__(32 * kListWarps) k_push_roots(const int32_t* __restrict__ R, const int32_t* d_cnt,
                                                                const int64_t* __restrict__ rowptr,
                                                                const int32_t* __restrict__ colinds,
                                                                int32_t* __restrict__ labels,
                                                                int32_t* __restrict__ size, int* err) {
    const ListIdx<GL> li;
    const int64_t cnt = *d_cnt, trips = warp_trips(li, cnt);
    int bad = 0;
    for (int64_t t = 0; t < trips; t++) {
        const int64_t i = li.first + t * li.stride;
        const bool ok = i < cnt;
        int c = 0;
        if (ok) {
            const int32_t r = R[i];
            if (li.sub == 0) labels[r] = (int32_t)i;
            const int64_t s = rowptr[r], e = rowptr[r + 1];
            for (int64_t j = s + li.sub; j < e; j += GL) {
                const int32_t w = colinds[j];
                if (w == r) continue;
                const int32_t old = atomicExch(&labels[w], (int32_t)i);
                bad |= old >= 0 && old != (int32_t)i;  // two roots within distance 2
                c++;
            }
        }
        c = group_sum<GL>(c);
        if (ok && li.sub == 0) size[i] = 1 + c;
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrTwoRoots);
}

// Phase 2 accept rule (Q16) for the phase-2 roots R2[i]: acc[i] =
// (>= 2 neighbours w != r unaggregated after phase 1); cnt2[i] = that count
template <int GL>
__global__ void __launch_bounds__(32 * kListWarps) k_accept_list(const int32_t* __restrict__ R2, const int32_t* d_cnt,
                                                                 const int64_t* __restrict__ rowptr,
                                                                 const int32_t* __restrict__ colinds,
                                                                 const int32_t* __restrict__ labels,
                                                                 uint8_t* __restrict__ acc) {
    const ListIdx<GL> li;
    const int64_t cnt = *d_cnt, trips = warp_trips(li, cnt);
    for (int64_t t = 0; t < trips; t++) {
        const int64_t i = li.first + t * li.stride;
        int c = 0;
        if (i < cnt) {
            const int32_t r = R2[i];
            const int64_t s = rowptr[r], e = rowptr[r + 1];
            for (int64_t j = s + li.sub; j < e; j += GL) {
                const int32_t w = colinds[j];
                c += (w != r && labels[w] < 0);
            }
        }
        c = group_sum<GL>(c);
        if (i < cnt && li.sub == 0) acc[i] = c >= 2 ? 1 : 0;
    }
}

// Phase 2 labels (Q17): accepted root A[j] gets aggregate n1 + j
// (ascending vertex order) and so do its unaggregated neighbours (no vertex
// has two: the phase-2 roots are >= 3 apart in the unaggregated subgraph);
// size[n1 + j] = 1 + the neighbours it took
template <int GL>
__global__ void __launch_bounds__(32 * kListWarps) k_push_accepted(const int32_t* __restrict__ A, const int32_t* d_cnt,
                                                                   const int32_t* d_n1,
                                                                   const int64_t* __restrict__ rowptr,
                                                                   const int32_t* __restrict__ colinds,
                                                                   int32_t* __restrict__ labels,
                                                                   int32_t* __restrict__ roots,
                                                                   int32_t* __restrict__ size, int* err) {
    const ListIdx<GL> li;
    const int64_t cnt = *d_cnt, trips = warp_trips(li, cnt);
    const int32_t n1 = *d_n1;
    int bad = 0;
    for (int64_t t = 0; t < trips; t++) {
        const int64_t i = li.first + t * li.stride;
        const bool ok = i < cnt;
        int c = 0;
        int32_t r = 0;
        const int32_t id = n1 + (int32_t)i;
        if (ok) {
            r = A[i];
            const int64_t s = rowptr[r], e = rowptr[r + 1];
            for (int64_t j = s + li.sub; j < e; j += GL) {
                const int32_t w = colinds[j];
                if (w == r) continue;
                const int32_t old = atomicCAS(&labels[w], -1, id);  // phase-1 labels (< n1) stay
                bad |= old >= n1 && old != id;                      // two accepted roots share a vertex
                c += old == -1;
            }
        }
        c = group_sum<GL>(c);
        if (ok && li.sub == 0) {
            labels[r] = id;
            roots[id] = r;
            size[id] = 1 + c;
        }
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrPhase2Conflict);
}

// the leftovers (label -1 after phase 2) listed, any order: each one's
// choice reads only the frozen labels and sizes.  A block takes a
// contiguous range, counts its leftovers, reserves them with ONE atomic
// (a warp-aggregated atomic per 32 rows serialises on the counter: C3 0.57
// ms) and writes them in order.
__global__ void k_leftovers(int64_t n, const int32_t* __restrict__ labels, int32_t* __restrict__ left,
                            unsigned long long* nleft) {
    constexpr int E = 8;  // consecutive vertices per thread per round
    __shared__ int s_w[33];
    __shared__ unsigned long long s_base;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    int c = 0;
    for (int64_t v = lo + t; v < hi; v += blockDim.x) c += labels[v] < 0;
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) s_w[warp] = c;
    __syncthreads();
    if (t == 0) {
        int tot = 0;
        for (int w = 0; w < nw; w++) tot += s_w[w];
        s_base = tot ? atomicAdd(nleft, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    unsigned long long run = s_base;
    for (int64_t b0 = lo; b0 < hi; b0 += (int64_t)blockDim.x * E) {
        const int64_t v0 = b0 + (int64_t)t * E;
        unsigned bits = 0;
#pragma unroll
        for (int k = 0; k < E; k++) bits |= (v0 + k < hi && labels[v0 + k] < 0) ? (1u << k) : 0u;
        const int mine = __popc(bits);
        int inc = mine;  // block exclusive scan of the per-thread counts
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, off);
            if (lane >= off) inc += y;
        }
        __syncthreads();
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        int wbase = 0, step = 0;
        for (int w = 0; w < nw; w++) {
            if (w < warp) wbase += s_w[w];
            step += s_w[w];
        }
        unsigned long long off = run + wbase + inc - mine;
#pragma unroll
        for (int k = 0; k < E; k++)
            if (bits & (1u << k)) left[off++] = (int32_t)(v0 + k);
        run += step;
    }
}

// Phase 3 (Q19) on the leftover list, a group of GL lanes per row
// of at most GL entries: lanes holding the same candidate aggregate find each
// other (__match_any_sync on (group, aggregate)), so every lane knows its
// candidate's coupling; the group keeps the best (max coupling, min aggsize,
// min id) and stores it at the row's list position.  Longer rows (<=
// kHeavyDeg) go to k_phase3_table, longer ones to k_phase3_heavy.
template <int GL>
__global__ void __launch_bounds__(32 * kListWarps) k_phase3_list(const int32_t* __restrict__ left,
                                                                 const unsigned long long* nleft,
                                                                 const int64_t* __restrict__ rowptr,
                                                                 const int32_t* __restrict__ colinds,
                                                                 const int32_t* __restrict__ labels,
                                                                 const int32_t* __restrict__ size,
                                                                 int32_t* __restrict__ choice,
                                                                 int32_t* __restrict__ longq, int* longq_cnt,
                                                                 int32_t* __restrict__ heavy, int* heavy_cnt) {
    // U list entries per group per trip, their loads interleaved (the chain
    // list -> rowptr -> colinds -> labels -> size is latency bound)
    constexpr int U = 1;  // 2 / 4 measured slower (C3 phase 3: 435 us at 1, 514 us at 4)
    const ListIdx<GL> li;
    const int64_t cnt = (int64_t)*nleft;
    const int64_t wfirst = li.first - (int64_t)((threadIdx.x & 31) / GL);
    const int64_t trips = cnt > wfirst ? (cnt - wfirst + li.stride * U - 1) / (li.stride * U) : 0;
    const uint64_t gtag = (uint64_t)(threadIdx.x / GL) << 32;
    for (int64_t t = 0; t < trips; t++) {
        int64_t i[U], s[U], e[U];
        int32_t v[U], a[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            i[u] = li.first + (t * U + u) * li.stride;
            v[u] = i[u] < cnt ? left[i[u]] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            s[u] = 0;
            e[u] = 0;
            if (v[u] >= 0) {
                s[u] = rowptr[v[u]];
                e[u] = rowptr[v[u] + 1];
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            a[u] = -1;
            if (v[u] >= 0 && e[u] - s[u] <= GL && s[u] + li.sub < e[u]) {
                const int32_t w = colinds[s[u] + li.sub];
                a[u] = (w != v[u]) ? w : -1;
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) a[u] = a[u] >= 0 ? labels[a[u]] : -1;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool short_row = v[u] >= 0 && e[u] - s[u] <= GL;
            if (v[u] >= 0 && !short_row && li.sub == 0) {
                if (e[u] - s[u] > kHeavyDeg) heavy[atomicAdd(heavy_cnt, 1)] = (int32_t)i[u];
                else longq[atomicAdd(longq_cnt, 1)] = (int32_t)i[u];
            }
            const unsigned grp = __match_any_sync(kFull, gtag | (uint32_t)a[u]);
            int bc = 0, bs = 0, ba = -1;
            if (a[u] >= 0) {
                bc = __popc(grp);
                bs = size[a[u]];
                ba = a[u];
            }
            group_best<GL>(bc, bs, ba);
            if (short_row && li.sub == 0) choice[i[u]] = ba;  // -1: no candidate (impossible)
        }
    }
}

// Phase 3 for the longer listed rows: a warp per row, the couplings of its
// candidate aggregates counted in the warp's shared-memory table (match
// groups of each 32-entry chunk add at once); a table overflow -> heavy.
#ifndef MIS2_P3_SLOTS
#define MIS2_P3_SLOTS 128
#endif
constexpr int kP3Slots = MIS2_P3_SLOTS;
// longq == nullptr: every listed leftover (rows mostly longer than the list
// kernel's groups: no listing pass, whose one append per row serialises on
// its counter -- C5 1.1 ms)
__global__ void __launch_bounds__(32 * kListWarps) k_phase3_table(const int32_t* __restrict__ left,
                                                                  const int32_t* __restrict__ longq, const int* longq_cnt,
                                                                  const unsigned long long* nleft,
                                                                  const int64_t* __restrict__ rowptr,
                                                                  const int32_t* __restrict__ colinds,
                                                                  const int32_t* __restrict__ labels,
                                                                  const int32_t* __restrict__ size,
                                                                  int32_t* __restrict__ choice,
                                                                  int32_t* __restrict__ heavy, int* heavy_cnt) {
    __shared__ int32_t tkey[kListWarps][kP3Slots];
    __shared__ int32_t tcnt[kListWarps][kP3Slots];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int32_t* key = tkey[wib];
    int32_t* cnt = tcnt[wib];
    const int64_t m = longq ? (int64_t)*longq_cnt : (int64_t)*nleft;
    for (int64_t q = (int64_t)blockIdx.x * kListWarps + wib; q < m; q += (int64_t)gridDim.x * kListWarps) {
        const int32_t i = longq ? longq[q] : (int32_t)q;
        const int32_t v = left[i];
        const int64_t s = rowptr[v], e = rowptr[v + 1];
#pragma unroll
        for (int k = 0; k < kP3Slots / 32; k++) {
            key[lane + 32 * k] = -1;
            cnt[lane + 32 * k] = 0;
        }
        __syncwarp();
        bool over = false;
        for (int64_t j0 = s; j0 < e; j0 += 32) {
            const int64_t j = j0 + lane;
            int32_t a = -1;
            if (j < e) {
                const int32_t w = colinds[j];
                a = (w != v) ? labels[w] : -1;
            }
            const unsigned grp = __match_any_sync(kFull, a);
            if (a >= 0 && lane == __ffs(grp) - 1) {
                unsigned h = ((unsigned)a * 2654435761u) % kP3Slots;
                bool placed = false;
                for (int probe = 0; probe < kP3Slots; probe++) {
                    const int32_t k = atomicCAS(&key[h], -1, a);
                    if (k == -1 || k == a) {
                        atomicAdd(&cnt[h], __popc(grp));
                        placed = true;
                        break;
                    }
                    h = (h + 1) % kP3Slots;
                }
                over |= !placed;
            }
        }
        __syncwarp();
        int bc = 0, bs = 0, ba = -1;
        if (!__any_sync(kFull, over)) {  // (uniform)
#pragma unroll
            for (int k = 0; k < kP3Slots / 32; k++) {
                const int32_t a = key[lane + 32 * k];
                if (a >= 0) {
                    const int c = cnt[lane + 32 * k], sz = size[a];
                    if (better(c, sz, a, bc, bs, ba)) { bc = c; bs = sz; ba = a; }
                }
            }
        }
        __syncwarp();
        const bool any_over = __any_sync(kFull, over);
        group_best<32>(bc, bs, ba);
        if (lane == 0) {
            if (any_over) heavy[atomicAdd(heavy_cnt, 1)] = i;
            else choice[i] = ba;
        }
    }
}

// ---- the induced subgraph of the unaggregated vertices (phase 2, Q15)
// act[v] = (labels[v] < 0)
__global__ void k_active_flags(int64_t n, const int32_t* __restrict__ labels, uint8_t* __restrict__ act) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        act[v] = labels[v] < 0;
}
// row i of the subgraph = vertex gid[i]: its active neighbours (self included if stored)
template <int GL>
__global__ void __launch_bounds__(32 * kListWarps) k_sub_len(const int32_t* __restrict__ gid, const int32_t* d_m,
                                                             const int64_t* __restrict__ rowptr,
                                                             const int32_t* __restrict__ colinds,
                                                             const uint8_t* __restrict__ act,
                                                             int64_t* __restrict__ len) {
    const ListIdx<GL> li;
    const int64_t cnt = *d_m, trips = warp_trips(li, cnt);
    for (int64_t t = 0; t < trips; t++) {
        const int64_t i = li.first + t * li.stride;
        int c = 0;
        if (i < cnt) {
            const int32_t v = gid[i];
            const int64_t s = rowptr[v], e = rowptr[v + 1];
            constexpr int U = 4;  // steps of the row in flight (the walk is latency bound)
            for (int64_t j0 = s + li.sub; j0 < e; j0 += (int64_t)GL * U) {
                int32_t w[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t j = j0 + (int64_t)u * GL;
                    w[u] = j < e ? colinds[j] : -1;
                }
#pragma unroll
                for (int u = 0; u < U; u++) c += w[u] >= 0 ? act[w[u]] : 0;
            }
        }
        c = group_sum<GL>(c);
        if (i < cnt && li.sub == 0) len[i] = c;
    }
}
// the subgraph's colinds: inv[w] of the active neighbours, in row order
template <int GL>
__global__ void __launch_bounds__(32 * kListWarps) k_sub_fill(const int32_t* __restrict__ gid, const int32_t* d_m,
                                                              const int64_t* __restrict__ rowptr,
                                                              const int32_t* __restrict__ colinds,
                                                              const uint8_t* __restrict__ act,
                                                              const int32_t* __restrict__ inv,
                                                              const int64_t* __restrict__ srow,
                                                              int32_t* __restrict__ scol) {
    const ListIdx<GL> li;
    const int64_t cnt = *d_m, trips = warp_trips(li, cnt);
    const int gbase_lane = (threadIdx.x & 31) & ~(GL - 1);
    const unsigned gmask = (GL == 32 ? kFull : ((1u << GL) - 1u)) << gbase_lane;
    for (int64_t t = 0; t < trips; t++) {
        const int64_t i = li.first + t * li.stride;
        const bool ok = i < cnt;
        int64_t s = 0, e = 0, o = 0;
        if (ok) {
            const int32_t v = gid[i];
            s = rowptr[v];
            e = rowptr[v + 1];
            o = srow[i];
        }
        // the group's lanes walk the row in strides of GL; each step's
        // active entries are placed by their rank among the group's lanes
        const int64_t steps = (e - s + GL - 1) / GL;
        int64_t maxsteps = steps;  // warp-wide: the ballots below need every lane
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const int64_t y = __shfl_xor_sync(kFull, maxsteps, off);
            maxsteps = y > maxsteps ? y : maxsteps;
        }
        constexpr int U = 4;  // steps in flight: colinds, then act, then inv of U steps
        for (int64_t k0 = 0; k0 < maxsteps; k0 += U) {
            int32_t w[U], x[U];
            bool a[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t j = s + (k0 + u) * GL + li.sub;
                w[u] = j < e ? colinds[j] : -1;
            }
#pragma unroll
            for (int u = 0; u < U; u++) a[u] = w[u] >= 0 && act[w[u]];
#pragma unroll
            for (int u = 0; u < U; u++) x[u] = a[u] ? inv[w[u]] : 0;
#pragma unroll
            for (int u = 0; u < U; u++) {
                const unsigned ball = __ballot_sync(kFull, a[u]) & gmask;
                if (a[u]) scol[o + __popc(ball & lanemask_lt())] = x[u];
                o += __popc(ball);
            }
        }
    }
}
// in_set of the whole graph from the subgraph's (inactive vertices: 0)
__global__ void k_scatter_in(const int32_t* __restrict__ gid, const int32_t* d_m, const uint8_t* __restrict__ in_sub,
                             uint8_t* __restrict__ in_full) {
    const int64_t m = *d_m;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        in_full[gid[i]] = in_sub[i];
}

// choices -> labels (after every phase-3 read of the frozen labels)
__global__ void k_scatter_choice(const int32_t* __restrict__ left, const unsigned long long* nleft,
                                 const int32_t* __restrict__ choice, int32_t* __restrict__ labels, int* err) {
    const int64_t m = (int64_t)*nleft;
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = choice[i];
        if (a < 0) bad = 1;  // impossible by maximality of M1 (Q20)
        else labels[left[i]] = a;
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrNoCandidate);
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

struct AggWs {
    Mis2Ws mis;
    uint8_t *in1, *in2, *acc;
    int32_t *rid, *aid, *tent, *size, *heavy, *left, *longq;
    int64_t *slen, *srow;  // induced subgraph of phase 2: row lengths, row pointers
    int32_t* scol;         // its colinds (<= nnz)
    void* scan_tmp;
    long long* scal;  // device scalars
};

static void carve_agg(Carve& c, int64_t n, int64_t nnz, int max_warps, AggWs* w) {
    carve_mis2(c, n, nnz, max_warps, &w->mis);
    w->in1 = c.take<uint8_t>((size_t)n + 1);
    w->in2 = c.take<uint8_t>((size_t)n + 1);
    w->acc = c.take<uint8_t>((size_t)n + 1);
    w->rid = c.take<int32_t>((size_t)n + 1);
    w->aid = c.take<int32_t>((size_t)n + 1);
    w->tent = c.take<int32_t>((size_t)n + 1);
    w->size = c.take<int32_t>((size_t)n + 1);
    w->heavy = c.take<int32_t>((size_t)n + 1);
    w->left = c.take<int32_t>((size_t)n + 1);
    w->longq = c.take<int32_t>((size_t)n + 1);
    w->slen = c.take<int64_t>((size_t)n + 1);
    w->srow = c.take<int64_t>((size_t)n + 2);
    w->scol = c.take<int32_t>((size_t)nnz + 1);
    w->scan_tmp = c.take<char>(std::max(scan_ws_bytes(n), scan64_ws_bytes(n)));
    w->scal = c.take<long long>(32);
}

// device scalar slots in AggWs::scal
enum { kCount1 = 0, kCount2 = 1, kNa = 2, kLeft = 3, kIters1 = 8, kIters2 = 9, kStatus1 = 10,
       kStatus2 = 11, kN1 = 12, kN2 = 13, kErr = 14, kHeavyCnt = 15 };

template <int G>
static void launch_rows(int64_t n, int sms, cudaStream_t s, int which, const mis2_graph& g, AggWs& w,
                        int32_t* labels, int32_t* roots) {
    int32_t* s32 = (int32_t*)w.scal;
    const int64_t rows_per_block = (int64_t)(kBlock / 32) * (32 / G);
    int64_t blocks = (n + rows_per_block - 1) / rows_per_block;
    const int64_t cap = (int64_t)sms * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    switch (which) {
        case 1:
            k_phase1<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.in1, w.rid, labels, roots,
                                                          &s32[2 * kErr]);
            break;
        case 2:
            k_phase2_accept<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.in2, labels, w.acc);
            break;
        case 3:
            k_phase2_label<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.acc, w.aid,
                                                                &s32[2 * kN1], labels, roots, &s32[2 * kErr]);
            break;
        case 4:
            k_phase3<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.tent, w.size, labels, w.heavy,
                                                          &s32[2 * kHeavyCnt], &s32[2 * kErr]);
            break;
        case 5:
            k_basic_join<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.tent, labels, &s32[2 * kErr]);
            break;
    }
    count_launch();
}

static void rows(int G, int64_t n, int sms, cudaStream_t s, int which, const mis2_graph& g, AggWs& w,
                 int32_t* labels, int32_t* roots) {
    switch (G) {
        case 1: launch_rows<1>(n, sms, s, which, g, w, labels, roots); break;
        case 2: launch_rows<2>(n, sms, s, which, g, w, labels, roots); break;
        case 4: launch_rows<4>(n, sms, s, which, g, w, labels, roots); break;
        case 8: launch_rows<8>(n, sms, s, which, g, w, labels, roots); break;
        case 16: launch_rows<16>(n, sms, s, which, g, w, labels, roots); break;
        default: launch_rows<32>(n, sms, s, which, g, w, labels, roots); break;
    }
}

// ---- raw-array launchers of the row kernels, for the partitioned driver
// (dist.cu): rows are a partition's owned rows, colinds are local indices
// and every array read through colinds holds the ghosts after the owned rows.
static int64_t row_blocks(int G, int64_t n, int sms) {
    const int64_t rows_per_block = (int64_t)(kBlock / 32) * (32 / G);
    int64_t blocks = (n + rows_per_block - 1) / rows_per_block;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    return blocks < 1 ? 1 : blocks;
}
#define AGG_DISPATCH(G, CALL)                  \
    switch (G) {                               \
        case 1: { constexpr int GG = 1; CALL; } break;  \
        case 2: { constexpr int GG = 2; CALL; } break;  \
        case 4: { constexpr int GG = 4; CALL; } break;  \
        case 8: { constexpr int GG = 8; CALL; } break;  \
        case 16: { constexpr int GG = 16; CALL; } break; \
        default: { constexpr int GG = 32; CALL; } break; \
    }
void agg_phase1(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* in1,
                const int32_t* rid, int32_t* labels, int* err, int sms, cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase1<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, in1, rid, labels, nullptr, err)));
    count_launch();
}
void agg_accept(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* in2,
                const int32_t* labels, uint8_t* acc, int sms, cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase2_accept<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, in2, labels, acc)));
    count_launch();
}
void agg_phase2_label(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* acc,
                      const int32_t* aid, const int32_t* d_n1, int32_t* labels, int* err, int sms, cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase2_label<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, acc, aid, d_n1, labels, nullptr, err)));
    count_launch();
}
void agg_tent_size(int64_t n, const int32_t* labels, int32_t* tent, int32_t* size, unsigned long long* left, int sms,
                   cudaStream_t s) {
    int64_t blocks = (n + kBlock - 1) / kBlock;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    if (blocks < 1) blocks = 1;
    k_tent_size<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, tent, size, left);
    count_launch();
}
void agg_phase3(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const int32_t* tent,
                const int32_t* size, int32_t* labels, int32_t* heavy, int* heavy_cnt, int* err, int sms,
                cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase3<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, tent, size, labels, heavy, heavy_cnt, err)));
    count_launch();
    k_phase3_heavy<<<sms * 4, kBlock, 0, s>>>(rowptr, colinds, tent, size, labels, heavy, heavy_cnt, err);
    count_launch();
}
#undef AGG_DISPATCH

// Large graphs run the phase-2 MIS-2 on the induced subgraph of the
// unaggregated vertices (below); small ones the masked call on G (the
// build's two host reads of the subgraph's size cost more than the smaller
// passes save: C2 0.88 ms masked, 0.97 ms on the subgraph; C3 11.1 -> 10.0
// ms, C5 14.8 -> 14.0 ms).  MIS2_AGG_SUB=0/1 forces (measurement knob).
static bool agg_use_sub(const mis2_graph& g) {
    bool use_sub = g.nnz >= (int64_t)1 << 26;
    if (const char* e = getenv("MIS2_AGG_SUB")) use_sub = atoi(e) != 0;
    return use_sub;
}

// All device work of Alg. 3 on stream s; the host reads the
// scalars afterwards (run_aggregate).
static int agg_enqueue(const mis2_graph& g, const mis2_opts& o, int32_t* labels, int32_t* roots, AggWs& w,
                       int64_t* ist1, int64_t* ist2, const DeviceInfo& di, cudaStream_t s) {
    const int64_t n = g.n;
    const int G = choose_group(g.n, g.nnz, o.group);
    int32_t* s32 = (int32_t*)w.scal;
    MIS2_CUDA_TRY(cudaMemsetAsync(w.scal, 0, 32 * sizeof(long long), s));

    // ---- phase 1: M1 = MIS2(G)
    MIS2_TRY(run_mis2(g, o, nullptr, w.in1, (int64_t*)&w.scal[kCount1], &s32[2 * kIters1],
                      &s32[2 * kStatus1], ist1, w.mis, s));
    const bool basic = (o.flags & MIS2_FLAG_BASIC) != 0;
    const unsigned lgrid = (unsigned)(di.sms * 8);  // list kernels: 8 warps per block
    // lanes per list entry: the average row length rounded up to a power of
    // two in [4, 32] (short rows: several entries per warp)
    const double avg = n > 0 ? (double)g.nnz / (double)n : 0.0;
    int GL = avg <= 4.0 ? 4 : (avg <= 8.0 ? 8 : (avg <= 16.0 ? 16 : 32));
    if (const char* e = getenv("MIS2_AGG_GL")) GL = atoi(e);  // measurement knob: 4 / 8 / 16 / 32
#define LIST_DISPATCH(gl, CALL)                             \
    switch (gl) {                                           \
        case 4: { constexpr int GLL = 4; CALL; } break;     \
        case 8: { constexpr int GLL = 8; CALL; } break;     \
        case 16: { constexpr int GLL = 16; CALL; } break;   \
        default: { constexpr int GLL = 32; CALL; } break;   \
    }
    int32_t* rl = roots ? roots : w.rid;            // roots in aggregate order (phase 1, then phase 2)
    if (basic) {
        MIS2_TRY(scan_flags(w.in1, n, w.rid, &s32[2 * kN1], w.scan_tmp, s));
        rows(G, n, di.sms, s, 1, g, w, labels, roots);
    } else {
        // roots listed in ascending vertex order = their aggregate ids (Q18); they push them
        MIS2_TRY(scan_flags_list(w.in1, n, nullptr, nullptr, rl, nullptr, &s32[2 * kN1], w.scan_tmp, s));
        MIS2_CUDA_TRY(cudaMemsetAsync(labels, 0xff, sizeof(int32_t) * (size_t)n, s));
        LIST_DISPATCH(GL, (k_push_roots<GLL><<<lgrid, 32 * kListWarps, 0, s>>>(rl, &s32[2 * kN1], g.rowptr, g.colinds,
                                                                            labels, w.size, &s32[2 * kErr])));
        count_launch();
    }

    if (basic) {
        // ---- Alg. 2: every leftover joins an adjacent phase-1 aggregate
        MIS2_CUDA_TRY(cudaMemsetAsync(w.size, 0, sizeof(int32_t) * ((size_t)n + 1), s));
        int64_t blocks = (n + kBlock - 1) / kBlock;
        if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
        if (blocks < 1) blocks = 1;
        k_tent_size<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, w.tent, w.size,
                                                        (unsigned long long*)&w.scal[kLeft]);
        count_launch();
        rows(G, n, di.sms, s, 5, g, w, labels, roots);
        k_finish<<<1, 1, 0, s>>>(&s32[2 * kN1], &s32[2 * kN2], (int64_t*)&w.scal[kNa]);
        count_launch();
    } else {

    // ---- phase 2: M2 = MIS2(G \ aggregated) on the same ids / seed (Q15)
    if (!agg_use_sub(g)) {
        MIS2_TRY(run_mis2(g, o, labels, w.in2, (int64_t*)&w.scal[kCount2], &s32[2 * kIters2], &s32[2 * kStatus2],
                          ist2, w.mis, s));
    } else {
    // The induced subgraph of the unaggregated vertices itself: its
    // rows hold only unaggregated neighbours (C2: 44% of the rows, 17% of
    // the entries), row i is vertex gid[i] (aid), whose original id the
    // hash, the packing width b (of the whole graph) and the M id fields use
    // -- the same iteration as the masked call on G, on less data.
    {
        int64_t blocks = (n + kBlock - 1) / kBlock;
        if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
        if (blocks < 1) blocks = 1;
        k_active_flags<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, w.acc);
        count_launch();
    }
    int32_t* gid = w.aid;   // rows of the subgraph -> vertices (ascending)
    int32_t* inv = w.rid;   // vertices -> rows (active ones); w.rid is free until phase 2's pushes
    int32_t* d_m = &s32[2 * kN2 + 1];
    MIS2_TRY(scan_flags_list(w.acc, n, nullptr, inv, gid, nullptr, d_m, w.scan_tmp, s));
    // the subgraph build is latency bound: several rows per warp (GL <= 8)
    // (C3, 7-entry rows, GS = 2 / 4 / 8: 12.5 / 8.8 / 9.4 ms; C5, 81-entry
    // rows, 4 / 8 / 16: 12.4 / 12.0 / 12.5 ms)
    int GS = GL <= 8 ? 4 : 8;
    if (const char* e = getenv("MIS2_SUB_G")) GS = atoi(e);  // measurement knob: 4 / 8 / 16 / 32
    LIST_DISPATCH(GS, (k_sub_len<GLL><<<lgrid, 32 * kListWarps, 0, s>>>(gid, d_m, g.rowptr, g.colinds, w.acc,
                                                                      w.slen)));
    count_launch();
    int64_t hm[2] = {0, 0};
    {
        int32_t m32 = 0;
        MIS2_CUDA_TRY(cudaMemcpyAsync(&m32, d_m, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));  // the subgraph's size sizes its launches
        hm[0] = m32;
    }
    MIS2_TRY(scan_counts64(w.slen, hm[0], w.srow, w.scan_tmp, s));
    LIST_DISPATCH(GS, (k_sub_fill<GLL><<<lgrid, 32 * kListWarps, 0, s>>>(gid, d_m, g.rowptr, g.colinds, w.acc, inv,
                                                                       w.srow, w.scol)));
    count_launch();
    MIS2_CUDA_TRY(cudaMemcpyAsync(&hm[1], w.srow + hm[0], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    {
        mis2_graph gs{hm[0], hm[1], w.srow, w.scol};
        const SubGraph sub{gid, inv, n};
        MIS2_TRY(run_mis2(gs, o, nullptr, w.in1, (int64_t*)&w.scal[kCount2], &s32[2 * kIters2], &s32[2 * kStatus2],
                          ist2, w.mis, s, &sub));
        MIS2_CUDA_TRY(cudaMemsetAsync(w.in2, 0, (size_t)n, s));
        k_scatter_in<<<(unsigned)(di.sms * 8), kBlock, 0, s>>>(gid, d_m, w.in1, w.in2);
        count_launch();
    }
    }  // use_sub
    // the phase-2 roots in vertex order (aid), their acceptance (acc, by
    // list position), the accepted ones in vertex order (tent) -> aggregates
    // n1, n1 + 1, ...; their sizes come out of the pushes
    MIS2_TRY(scan_flags_list(w.in2, n, nullptr, nullptr, w.aid, nullptr, &s32[2 * kN2 + 1], w.scan_tmp, s));
    LIST_DISPATCH(GL, (k_accept_list<GLL><<<lgrid, 32 * kListWarps, 0, s>>>(w.aid, &s32[2 * kN2 + 1], g.rowptr,
                                                                          g.colinds, labels, w.acc)));
    count_launch();
    MIS2_TRY(scan_flags_list(w.acc, n, &s32[2 * kN2 + 1], nullptr, w.tent, w.aid, &s32[2 * kN2], w.scan_tmp, s));
    LIST_DISPATCH(GL, (k_push_accepted<GLL><<<lgrid, 32 * kListWarps, 0, s>>>(w.tent, &s32[2 * kN2], &s32[2 * kN1],
                                                                            g.rowptr, g.colinds, labels, rl, w.size,
                                                                            &s32[2 * kErr])));
    count_launch();

    // ---- phase 3: max coupling / min size / min id over the frozen labels;
    // choices by leftover-list position (tent), scattered at the end
    {
        int64_t blocks = (n + kBlock - 1) / kBlock;
        if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
        if (blocks < 1) blocks = 1;
        k_leftovers<<<(unsigned)(di.sms * 4), kBlock, 0, s>>>(n, labels, w.left, (unsigned long long*)&w.scal[kLeft]);
        count_launch();
    }
    const unsigned long long* nleft = (const unsigned long long*)&w.scal[kLeft];
    // rows mostly longer than 32 entries (C5: 81): every leftover goes
    // straight to the table kernel (a warp per row)
    const bool all_long = avg > 32.0;
    if (!all_long)
        LIST_DISPATCH(GL, (k_phase3_list<GLL><<<lgrid, 32 * kListWarps, 0, s>>>(
                              w.left, nleft, g.rowptr, g.colinds, labels, w.size, w.tent, w.longq,
                              &s32[2 * kHeavyCnt + 1], w.heavy, &s32[2 * kHeavyCnt])));
    k_phase3_table<<<lgrid, 32 * kListWarps, 0, s>>>(w.left, all_long ? nullptr : w.longq, &s32[2 * kHeavyCnt + 1],
                                                     nleft, g.rowptr, g.colinds, labels, w.size, w.tent, w.heavy,
                                                     &s32[2 * kHeavyCnt]);
    k_phase3_heavy<<<di.sms * 4, kBlock, 0, s>>>(g.rowptr, g.colinds, labels, w.size, labels, w.heavy,
                                                &s32[2 * kHeavyCnt], &s32[2 * kErr], w.left, w.tent);
    k_scatter_choice<<<(unsigned)(di.sms * 8), kBlock, 0, s>>>(w.left, nleft, w.tent, labels, &s32[2 * kErr]);
    count_launch(all_long ? 3 : 4);
    k_finish<<<1, 1, 0, s>>>(&s32[2 * kN1], &s32[2 * kN2], (int64_t*)&w.scal[kNa]);
    count_launch();
    }  // Alg. 3
    MIS2_CUDA_TRY(cudaGetLastError());
    return MIS2_OK;
}

// ---- CUDA-graph replay of repeated aggregate() calls
// Alg. 3 is ~20 launches whose sizes depend only on (n, nnz, options), so a
// call on the same graph, outputs and workspace as an earlier one replays
// the captured launch sequence (one graph launch instead of ~20 kernel
// launches and their gaps) on a private stream joined to the caller's by
// events -- from the second call with the same key on (a one-off call, e.g.
// a level of the multilevel loop, pays no capture).  Only sequences without
// host reads are captured: the masked
// phase-2 call (not the induced subgraph, whose size the host reads), no
// skew test (8n <= 64 MB), no per-iteration statistics.  MIS2_AGG_GRAPH=0:
// never (measurement knob).
struct AggGraphKey {
    int64_t n, nnz;
    const void *rowptr, *colinds, *labels, *roots, *ws;
    size_t ws_bytes;
    uint64_t seed;
    int32_t scheme, max_iters, group;
    uint32_t flags;
    bool operator==(const AggGraphKey& k) const { return memcmp(this, &k, sizeof(k)) == 0; }
};
struct AggGraph {
    AggGraphKey key;
    cudaGraphExec_t exec;
    int64_t launches;
    int dev;
};
static std::mutex g_agg_mu;
static AggGraph g_agg_cache[4];
static int g_agg_n = 0, g_agg_next = 0;
static cudaStream_t g_agg_stream[64];
static cudaEvent_t g_agg_ev[64][2];

static int agg_graph_run(const mis2_graph& g, const mis2_opts& o, int32_t* labels, int32_t* roots, AggWs& w,
                         void* ws, size_t ws_bytes, const DeviceInfo& di, cudaStream_t s, bool* done) {
    *done = false;
    if (const char* e = getenv("MIS2_AGG_GRAPH"))
        if (atoi(e) == 0) return MIS2_OK;
    int dev = 0;
    MIS2_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return MIS2_OK;
    {  // the caller is capturing its own graph: stay a plain sequence inside it
        cudaStreamCaptureStatus cs_status = cudaStreamCaptureStatusNone;
        MIS2_CUDA_TRY(cudaStreamIsCapturing(s, &cs_status));
        if (cs_status != cudaStreamCaptureStatusNone) return MIS2_OK;
    }
    AggGraphKey key;
    memset(&key, 0, sizeof(key));
    key.n = g.n;
    key.nnz = g.nnz;
    key.rowptr = g.rowptr;
    key.colinds = g.colinds;
    key.labels = labels;
    key.roots = roots;
    key.ws = ws;
    key.ws_bytes = ws_bytes;
    key.seed = o.seed;
    key.scheme = o.scheme;
    key.max_iters = o.max_iters;
    key.group = o.group;
    key.flags = o.flags;
    std::lock_guard<std::mutex> lock(g_agg_mu);
    if (!g_agg_stream[dev]) {
        MIS2_CUDA_TRY(cudaStreamCreateWithFlags(&g_agg_stream[dev], cudaStreamNonBlocking));
        MIS2_CUDA_TRY(cudaEventCreateWithFlags(&g_agg_ev[dev][0], cudaEventDisableTiming));
        MIS2_CUDA_TRY(cudaEventCreateWithFlags(&g_agg_ev[dev][1], cudaEventDisableTiming));
    }
    cudaStream_t cs = g_agg_stream[dev];
    AggGraph* hit = nullptr;
    for (int i = 0; i < g_agg_n; i++)
        if (g_agg_cache[i].dev == dev && g_agg_cache[i].key == key) hit = &g_agg_cache[i];
    if (!hit) {  // first call with this key: run directly, capture on the next one
        AggGraph& slot = g_agg_cache[g_agg_n < 4 ? g_agg_n++ : (g_agg_next++ & 3)];
        if (slot.exec) cudaGraphExecDestroy(slot.exec);
        slot.key = key;
        slot.exec = nullptr;
        slot.launches = 0;
        slot.dev = dev;
        return MIS2_OK;
    }
    MIS2_CUDA_TRY(cudaEventRecord(g_agg_ev[dev][0], s));
    MIS2_CUDA_TRY(cudaStreamWaitEvent(cs, g_agg_ev[dev][0], 0));
    if (!hit->exec) {
        reset_launches();
        MIS2_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
        const int rc = agg_enqueue(g, o, labels, roots, w, nullptr, nullptr, di, cs);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ie = (rc == MIS2_OK && ce == cudaSuccess) ? cudaGraphInstantiate(&exec, graph, 0)
                                                                    : cudaErrorUnknown;
        if (graph) cudaGraphDestroy(graph);
        if (ie != cudaSuccess) {  // not capturable here: the caller runs the sequence directly
            (void)cudaGetLastError();
            MIS2_CUDA_TRY(cudaStreamWaitEvent(s, g_agg_ev[dev][0], 0));
            return MIS2_OK;
        }
        hit->exec = exec;
        hit->launches = mis2_last_launch_count();
    }
    MIS2_CUDA_TRY(cudaGraphLaunch(hit->exec, cs));
    MIS2_CUDA_TRY(cudaEventRecord(g_agg_ev[dev][1], cs));
    MIS2_CUDA_TRY(cudaStreamWaitEvent(s, g_agg_ev[dev][1], 0));
    reset_launches();
    count_launch((int)hit->launches);
    *done = true;
    return MIS2_OK;
}

int run_aggregate(const mis2_graph& g, const mis2_opts& o, int32_t* labels, int64_t* num_aggs, int32_t* roots,
                  int64_t* stats, void* ws, size_t ws_bytes, cudaStream_t s, size_t* bytes_needed) {
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    Carve c(ws, ws_bytes);
    AggWs w;
    carve_agg(c, g.n, g.nnz, max_coop_warps(di), &w);
    if (bytes_needed) { *bytes_needed = c.off; return MIS2_OK; }
    if (!c.ok()) { set_error("workspace too small: need %zu bytes", c.off); return MIS2_ENOMEM; }
    const int64_t n = g.n;

    // per-iteration worklist statistics of both MIS-2 calls (MIS2_FLAG_ITER_STATS)
    const bool iter_stats = stats && (o.flags & MIS2_FLAG_ITER_STATS) && !(o.flags & MIS2_FLAG_TIMELINE);
    const int64_t mi = max_iters_for(n, o.max_iters);
    int64_t* ist1 = iter_stats ? stats + 8 : nullptr;
    int64_t* ist2 = iter_stats ? stats + 8 + 6 * mi : nullptr;
    if (iter_stats) memset(stats + 8, 0, sizeof(int64_t) * 12 * (size_t)mi);

    bool done = false;
    const bool graphable = !iter_stats && !(o.flags & MIS2_FLAG_TIMELINE) && !agg_use_sub(g) &&
                           (double)g.n * 8.0 <= 64.0 * 1048576.0 && g.n > 0;
    if (graphable) MIS2_TRY(agg_graph_run(g, o, labels, roots, w, ws, ws_bytes, di, s, &done));
    if (!done) MIS2_TRY(agg_enqueue(g, o, labels, roots, w, ist1, ist2, di, s));

    long long h[32];
    MIS2_CUDA_TRY(cudaMemcpyAsync(h, w.scal, sizeof(h), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    const int32_t* h32 = (const int32_t*)h;
    if (h32[2 * kStatus1] != MIS2_OK || h32[2 * kStatus2] != MIS2_OK) {
        set_error("MIS-2 did not converge within max_iters");
        return MIS2_ENOTCONVERGED;
    }
    if (h32[2 * kErr] != 0) {
        set_error("aggregation invariant failed (flags 0x%x): input graph not symmetric?", h32[2 * kErr]);
        return MIS2_EINTERNAL;
    }
    *num_aggs = h[kNa];
    if (stats) {
        stats[0] = h[kCount1];
        stats[1] = h32[2 * kIters1];
        stats[2] = h[kCount2];
        stats[3] = h32[2 * kIters2];
        stats[4] = h32[2 * kN2];
        stats[5] = h[kLeft];
        stats[6] = h32[2 * kN1];
        stats[7] = h[kNa];
    }
    return MIS2_OK;
}

}  // namespace mis2h
