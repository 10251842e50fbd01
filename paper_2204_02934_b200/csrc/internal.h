// internal.h -- host-side internals of libmis2.so (not part of the ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/mis2.h"

namespace mis2h {

// thread-local error detail + launch counter (abi.cu)
void set_error(const char* fmt, ...);
void count_launch(int k = 1);
void reset_launches();

#define MIS2_CUDA_TRY(expr)                                                              \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            ::mis2h::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                               cudaGetErrorString(_e));                                  \
            return MIS2_ECUDA;                                                           \
        }                                                                                \
    } while (0)

#define MIS2_TRY(expr)           \
    do {                         \
        int _rc = (expr);        \
        if (_rc != MIS2_OK) return _rc; \
    } while (0)

// bump allocator over the caller's workspace (256-byte aligned pieces)
struct Carve {
    char* base;
    size_t cap;
    size_t off = 0;
    bool dry;  // sizing pass: no base pointer
    Carve(void* b, size_t c) : base((char*)b), cap(c), dry(b == nullptr) {}
    template <class T>
    T* take(size_t count) {
        size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        if (bytes == 0) bytes = 256;
        T* p = dry ? nullptr : (T*)(base + off);
        off += bytes;
        return p;
    }
    bool ok() const { return dry || off <= cap; }
};

struct DeviceInfo {
    int device;
    int sms;
    size_t smem_optin;
};
int device_info(DeviceInfo* out);

constexpr int kStatsMaxIters = 400;

// MIS-2 state carved from the workspace
struct Mis2Ws {
    uint64_t* T;
    uint32_t* M;
    int32_t* L1[2];
    int32_t* L2[2];
    int32_t* heavy;
    unsigned int* mark;
    int32_t* gq;        // global queue of deferred rows (skewed graphs, mis2_kernel.cuh MIS2_GQ)
    uint8_t* oflag;     // push-form Decide state (mis2_core.cu)
    uint32_t* cnt;
    uint32_t* degc;
    uint32_t* K;        // 32-bit column keys (mis2_core.cu kkey)
    unsigned long long* ctrl;  // [80]: [0]=barrier, [5]=IN count, [8]=max degree,
                               // [16], [32] = the two counters of grid_sync_sum, [64..67] deferred-row queue
    unsigned long long* maxdeg;  // skew test of run_mis2
    long long* dstats;         // [kStatsMaxIters * 6]
    long long* scal;           // [8] host-visible scalars of mis2()/mis2_host()
};
void carve_mis2(Carve& c, int64_t n, int64_t nnz, int max_warps, Mis2Ws* w);
int max_coop_warps(const DeviceInfo& d);

// Runs Alg. 1 on the device.  labels != NULL restricts to {v : labels[v] < 0}
// (phase 2 of Alg. 3, reading Q15).  Writes in_set, *d_count, *d_iters,
// *d_status (device).  stats_host optional (synchronises).
// sub != NULL: g is an induced subgraph whose row v is vertex gid[v] of a
// graph of n_full vertices (hash ids, the packing width b and the M id
// fields use the original ids; inv maps them back to rows)
struct SubGraph {
    const int32_t* gid;
    const int32_t* inv;
    int64_t n_full;
};
int run_mis2(const mis2_graph& g, const mis2_opts& o, const int32_t* labels, uint8_t* in_set,
             int64_t* d_count, int32_t* d_iters, int32_t* d_status, int64_t* stats_host,
             const Mis2Ws& w, cudaStream_t s, const SubGraph* sub = nullptr);

int choose_group(int64_t n, int64_t nnz, int requested);
int max_iters_for(int64_t n, int requested);
int bits_for(int64_t n);

// ---- partitioned (multi-GPU) MIS-2: device state of one partition
struct PartDev {
    int64_t n_global, n_own, n_ghost, gbase, nnz;
    const int64_t* rowptr;   // device, local rows, n_own + 1
    const int32_t* colinds;  // device, LOCAL indices: owned [0, n_own), ghosts [n_own, n_own + n_ghost)
    const int32_t* labels;   // phase-2 mask or null
    uint64_t* T;             // n_own + n_ghost
    uint32_t* M;             // n_own + n_ghost
    int32_t* L1[2];
    int32_t* L2[2];
    int32_t* heavy;          // n_own deferred long rows
    uint8_t* in_set;         // n_own
    int G, scheme, hshift;
    uint64_t seed;
    // halo pushes (mis2_kernel.cuh PartK): owned row send_src[i] -> partition send_peer[i], index send_dst[i]
    int64_t nsend;
    const int64_t* send_csp;       // [n_own / 8 + 2] entries per 8-row group (sorted by row)
    const int32_t* send_src;
    const int32_t* send_peer;
    const int64_t* send_dst;
    unsigned int* bar;             // partition barrier counter
    unsigned long long* acc;       // [2]
    unsigned long long* box;       // [2 * P] mailboxes
    unsigned long long* rel;       // [1]
    int gpart;                     // global partition id
};
// Alg. 1 over the local partitions parts[0..nl) (one cooperative launch);
// peer_T / peer_M / peer_box: every partition's arrays as seen from this
// device (P entries); sys_scope: peers on other GPUs.  epoch: last partition-barrier epoch, updated.
// Writes *count (global), *iters; returns MIS2_OK / MIS2_ENOTCONVERGED.
int dist_mis2_launch(const std::vector<PartDev>& parts, const std::vector<uint64_t*>& peer_T,
                     const std::vector<uint32_t*>& peer_M, const std::vector<unsigned long long*>& peer_box,
                     bool sys_scope, int G, int max_iters, unsigned int* epoch, void* dev_scratch, int64_t* count,
                     int32_t* iters, cudaStream_t s);
size_t dist_scratch_bytes(int nlocal);
int debug_read(void* ws, size_t ws_bytes, int64_t n, long long* out, int64_t count);

// aggregation / coarsening / validation (aggregate.cu, coarsen.cu)
int run_aggregate(const mis2_graph& g, const mis2_opts& o, int32_t* labels, int64_t* num_aggs,
                  int32_t* roots, int64_t* stats, void* ws, size_t ws_bytes, cudaStream_t s,
                  size_t* bytes_needed);
int run_coarsen(const mis2_graph& g, const int32_t* labels, int64_t na, int64_t* c_rowptr,
                int32_t* c_colinds, int64_t cap, int64_t* c_nnz, void* ws, size_t ws_bytes,
                cudaStream_t s, size_t* bytes_needed);
int run_validate(const mis2_graph& g, void* ws, size_t ws_bytes, cudaStream_t s, size_t* bytes_needed);
// Alg. 4 setup colouring (cgs.cu, reading Q30)
int color_graph(const mis2_graph& g, uint64_t seed, int32_t* color, int32_t* ncolors, void* ws, size_t ws_bytes,
                cudaStream_t s, size_t* bytes_needed);

// aggregation row kernels on raw arrays (aggregate.cu), for the partitioned driver
void agg_phase1(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* in1,
                const int32_t* rid, int32_t* labels, int* err, int sms, cudaStream_t s);
void agg_accept(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* in2,
                const int32_t* labels, uint8_t* acc, int sms, cudaStream_t s);
void agg_phase2_label(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* acc,
                      const int32_t* aid, const int32_t* d_n1, int32_t* labels, int* err, int sms, cudaStream_t s);
void agg_tent_size(int64_t n, const int32_t* labels, int32_t* tent, int32_t* size, unsigned long long* left, int sms,
                   cudaStream_t s);
void agg_phase3(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const int32_t* tent,
                const int32_t* size, int32_t* labels, int32_t* heavy, int* heavy_cnt, int* err, int sms,
                cudaStream_t s);

// device-wide exclusive scan of 0/1 (uint8) flags -> int32 prefix, total to *d_total
size_t scan_ws_bytes(int64_t n);
// the same over the first min(n, *d_n) flags (d_n: device count or null),
// also (list non-null) the ordered compaction list[prefix[i]] = map ? map[i]
// : i of the set flags (prefix may be null)
int scan_flags_list(const uint8_t* flags, int64_t n, const int32_t* d_n, int32_t* prefix, int32_t* list,
                    const int32_t* map, int32_t* d_total, void* tmp, cudaStream_t s);
int scan_flags(const uint8_t* flags, int64_t n, int32_t* prefix, int32_t* d_total, void* tmp,
               cudaStream_t s);
// int64 exclusive scan of int64 counts (n entries) -> out[n+1]
size_t scan64_ws_bytes(int64_t n);
int scan_counts64(const int64_t* counts, int64_t n, int64_t* out, void* tmp, cudaStream_t s);

}  // namespace mis2h
