// dist.cu -- MIS-2 over a 1-D row partition.
//
// Every phase of Alg. 1 is a pure per-vertex function of the previous
// phase's arrays, the hash uses global ids and the packing uses the
// global n (Eq. 1), so any row partition reproduces the single-GPU result
// bit for bit provided each partition sees, before each phase, the current
// values of the vertices its rows reference:
//   before Refresh Column : T of the ghosts (owned by other partitions)
//   before Decide         : M of the ghosts
//   after Decide          : sum of |worklist_1| over all partitions
// Partition q owns rows [n*q/P, n*(q+1)/P); its local index space is
// [owned | ghosts], ghosts sorted by global id (hence grouped by owner), so a
// received halo lands directly in T / M without an unpack step.
//
// Transports: NCCL (one process per GPU; grouped ncclSend/ncclRecv for the
// halos, ncclAllReduce for the count; libnccl is dlopen'ed so the library
// loads without it), and LOCAL (all partitions in one process on the current
// device; halos copied device to device) -- the local transport runs the
// complete partitioned algorithm on one GPU, which is how it is tested.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "nccl.h"

using namespace mis2h;

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
        nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

int nccl_api(NcclApi** out) {
    static NcclApi api;
    if (!api.h) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            set_error("cannot dlopen libnccl.so.2: %s", dlerror());
            return MIS2_ENCCL;
        }
#define SYM(f)                                                              \
    api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f));         \
    if (!api.f) {                                                           \
        set_error("libnccl lacks nccl" #f);                                 \
        return MIS2_ENCCL;                                                  \
    }
        SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(Send) SYM(Recv) SYM(GroupStart) SYM(GroupEnd)
        SYM(AllReduce) SYM(AllGather) SYM(GetErrorString)
#undef SYM
        api.h = h;
    }
    *out = &api;
    return MIS2_OK;
}

#define NCCL_TRY(api, expr)                                                               \
    do {                                                                                  \
        ncclResult_t _r = (expr);                                                         \
        if (_r != ncclSuccess) {                                                          \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, (api)->GetErrorString(_r)); \
            return MIS2_ENCCL;                                                            \
        }                                                                                 \
    } while (0)

// ------------------------------------------------------------------ plan
inline int64_t part_lo(int64_t n, int P, int q) { return n * q / P; }

struct HostPart {
    int64_t lo = 0, hi = 0, n_own = 0, nnz = 0;
    std::vector<int64_t> rowptr;     // local rows, rebased
    std::vector<int32_t> colinds;    // local indices
    std::vector<int64_t> ghosts;     // global ids, sorted
    std::vector<int64_t> recv_cnt;   // per owner
    std::vector<int64_t> recv_off;   // [P+1] into the ghost slots
    std::vector<int32_t> send_idx;   // owned local indices, grouped by destination
    std::vector<int64_t> send_cnt;   // per destination
    std::vector<int64_t> send_off;   // [P+1]
};

// ghost discovery + local colinds (pure host)
int plan_local(int64_t n, int P, int q, const int64_t* rowptr, const int32_t* colinds, HostPart& hp) {
    hp.lo = part_lo(n, P, q);
    hp.hi = part_lo(n, P, q + 1);
    hp.n_own = hp.hi - hp.lo;
    hp.nnz = rowptr[hp.n_own] - rowptr[0];
    hp.rowptr.resize(hp.n_own + 1);
    for (int64_t i = 0; i <= hp.n_own; i++) hp.rowptr[i] = rowptr[i] - rowptr[0];
    std::vector<int64_t> g;
    for (int64_t j = 0; j < hp.nnz; j++) {
        const int64_t c = colinds[rowptr[0] + j];
        if (c < 0 || c >= n) {
            set_error("column index %lld out of range", (long long)c);
            return MIS2_EGRAPH;
        }
        if (c < hp.lo || c >= hp.hi) g.push_back(c);
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    hp.ghosts = g;
    hp.recv_cnt.assign(P, 0);
    for (int64_t c : g) {
        int o = (int)((c * P) / n);  // owner: largest q with n*q/P <= c
        while (o + 1 <= P - 1 && part_lo(n, P, o + 1) <= c) o++;
        while (o > 0 && part_lo(n, P, o) > c) o--;
        hp.recv_cnt[o]++;
    }
    hp.recv_off.assign(P + 1, 0);
    for (int o = 0; o < P; o++) hp.recv_off[o + 1] = hp.recv_off[o] + hp.recv_cnt[o];
    hp.colinds.resize(hp.nnz);
    for (int64_t j = 0; j < hp.nnz; j++) {
        const int64_t c = colinds[rowptr[0] + j];
        if (c >= hp.lo && c < hp.hi) hp.colinds[j] = (int32_t)(c - hp.lo);
        else hp.colinds[j] = (int32_t)(hp.n_own + (std::lower_bound(g.begin(), g.end(), c) - g.begin()));
    }
    return MIS2_OK;
}

// requests[o] = ghost ids this part wants from owner o -> send lists of the owner
void finish_sends(HostPart& owner, const std::vector<std::vector<int64_t>>& wanted_by, int P) {
    owner.send_cnt.assign(P, 0);
    owner.send_off.assign(P + 1, 0);
    owner.send_idx.clear();
    for (int d = 0; d < P; d++) {
        owner.send_cnt[d] = (int64_t)wanted_by[d].size();
        owner.send_off[d + 1] = owner.send_off[d] + owner.send_cnt[d];
        for (int64_t id : wanted_by[d]) owner.send_idx.push_back((int32_t)(id - owner.lo));
    }
}

__global__ void k_pack_u32(const uint32_t* __restrict__ src, const int32_t* __restrict__ idx, int64_t cnt,
                           uint32_t* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

__global__ void k_pack_u8(const uint8_t* __restrict__ src, const int32_t* __restrict__ idx, int64_t cnt,
                          uint8_t* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}
// x[v] += off for v < n (local prefix -> global aggregate numbering)
__global__ void k_add_i32(int32_t* __restrict__ x, int64_t n, int32_t off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] += off;
}
__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }
// labels of the stacked per-part coarse rows: row i is coarse row i mod na
__global__ void k_mod_labels(int32_t* __restrict__ lab, int64_t n, int64_t na) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        lab[i] = (int32_t)(i % na);
}
// dst[i] = src[i] + off (int64), i < cnt
__global__ void k_shift_i64(const int64_t* __restrict__ src, int64_t cnt, int64_t off, int64_t* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] + off;
}

}  // namespace

// ------------------------------------------------------------------ handles
// per-part state of the partitioned aggregation (allocated on first use)
struct AggPart {
    uint8_t *in1 = nullptr, *in2 = nullptr, *acc = nullptr;  // [n_own + n_ghost]
    int32_t *rid = nullptr, *aid = nullptr, *lab = nullptr, *tent = nullptr;  // [n_own + n_ghost]
    int32_t* size = nullptr;   // [n_global + 1] aggregate sizes (LOCAL: one array shared by all parts)
    int32_t* heavy = nullptr;  // [n_own]
    void* scan_tmp = nullptr;
    long long* scal = nullptr; // [16]: 0 n_local(int32 at 0), 1 err, 2 heavy_cnt, 3 leftovers, 4 n1 (int32)
};
struct mis2_comm {
    bool local = false;
    int nparts = 1;  // P
    int rank = 0;    // NCCL rank (local: unused)
    NcclApi* api = nullptr;
    ncclComm_t nccl = nullptr;
    int64_t n_global = 0;
    std::vector<HostPart> hp;   // local: P parts; NCCL: 1 (this rank)
    std::vector<PartDev> dev;   // same
    std::vector<void*> allocs;
    std::vector<uint64_t*> sendT;          // packed-halo scratch of exchange_arr (aggregation passes)
    std::vector<int32_t*> send_idx_d;
    std::vector<AggPart> agg;              // partitioned aggregation state
    // the partitioned MIS-2 kernel's view of every partition (P entries):
    // local transport -> the other parts' device buffers; NCCL -> the other
    // ranks' buffers mapped over NVLink (CUDA IPC)
    std::vector<uint64_t*> peer_T;
    std::vector<uint32_t*> peer_M;
    std::vector<unsigned long long*> peer_box;
    std::vector<void*> ipc_opened;
    unsigned int epoch = 0;                // last partition-barrier epoch (advances identically on every rank)
    void* dscratch = nullptr;              // kernel parameter block + results
    int64_t* d_counts = nullptr;           // [2 * (P + 1)] allgather buffers of gather_counts
    std::vector<std::pair<void*, size_t>> pool;  // coarsening scratch (DevBuf slots), kept across calls
};

static int dev_alloc(mis2_comm* c, void** p, size_t bytes) {
    MIS2_CUDA_TRY(cudaMalloc(p, bytes < 256 ? 256 : bytes));
    c->allocs.push_back(*p);
    return MIS2_OK;
}

static void free_parts(mis2_comm* c) {
    if (!c->ipc_opened.empty()) cudaDeviceSynchronize();  // peers' kernels may still reference the mappings
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    c->ipc_opened.clear();
    for (void* p : c->allocs) cudaFree(p);
    c->allocs.clear();
    for (auto& e : c->pool)
        if (e.first) cudaFree(e.first);
    c->pool.clear();
    c->hp.clear();
    c->dev.clear();
    c->sendT.clear();
    c->send_idx_d.clear();
    c->agg.clear();
    c->peer_T.clear();
    c->peer_M.clear();
    c->peer_box.clear();
    c->dscratch = nullptr;
    c->d_counts = nullptr;
}

// upload one planned part
static int upload_part(mis2_comm* c, const HostPart& h, PartDev& d, cudaStream_t s) {
    memset(&d, 0, sizeof(d));
    d.n_global = c->n_global;
    d.n_own = h.n_own;
    d.n_ghost = (int64_t)h.ghosts.size();
    d.gbase = h.lo;
    d.nnz = h.nnz;
    d.G = choose_group(h.n_own, h.nnz, 0);
    const int64_t nt = d.n_own + d.n_ghost + 1;
    void* p;
    MIS2_TRY(dev_alloc(c, &p, sizeof(int64_t) * (d.n_own + 1)));
    d.rowptr = (const int64_t*)p;
    MIS2_CUDA_TRY(cudaMemcpyAsync(p, h.rowptr.data(), sizeof(int64_t) * (d.n_own + 1), cudaMemcpyHostToDevice, s));
    MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (h.nnz + 1)));
    d.colinds = (const int32_t*)p;
    if (h.nnz) MIS2_CUDA_TRY(cudaMemcpyAsync(p, h.colinds.data(), sizeof(int32_t) * h.nnz, cudaMemcpyHostToDevice, s));
    MIS2_TRY(dev_alloc(c, &p, sizeof(uint64_t) * nt));
    d.T = (uint64_t*)p;
    MIS2_TRY(dev_alloc(c, &p, sizeof(uint32_t) * nt));
    d.M = (uint32_t*)p;
    for (int i = 0; i < 2; i++) {
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (d.n_own + 1)));
        d.L1[i] = (int32_t*)p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (d.n_own + 1)));
        d.L2[i] = (int32_t*)p;
    }
    // partition barrier state (mis2_kernel.cuh part_sync); the mailboxes get
    // their own allocation (other ranks map it over NVLink)
    MIS2_TRY(dev_alloc(c, &p, 256 + sizeof(unsigned long long) * 4));
    MIS2_CUDA_TRY(cudaMemsetAsync(p, 0, 256 + sizeof(unsigned long long) * 4, s));
    d.bar = (unsigned int*)p;
    d.acc = (unsigned long long*)((char*)p + 256);
    d.rel = d.acc + 2;
    MIS2_TRY(dev_alloc(c, &p, sizeof(unsigned long long) * 2 * c->nparts));
    MIS2_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(unsigned long long) * 2 * c->nparts, s));
    d.box = (unsigned long long*)p;
    MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (d.n_own + 1)));
    d.heavy = (int32_t*)p;
    const int64_t ns = (int64_t)h.send_idx.size();
    MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (ns + 1)));
    c->send_idx_d.push_back((int32_t*)p);
    if (ns) MIS2_CUDA_TRY(cudaMemcpyAsync(p, h.send_idx.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    MIS2_TRY(dev_alloc(c, &p, sizeof(uint64_t) * (ns + 1)));
    c->sendT.push_back((uint64_t*)p);
    return MIS2_OK;
}

// halo pushes of part `me` (owned row -> peer, index in the peer's T / M):
// its send list to peer q lands at q's ghost slots n_own_q + recv_off_q[me] + k
static int upload_sends(mis2_comm* c, const HostPart& h, PartDev& d, int me, const std::vector<int64_t>& n_own_of,
                        const std::vector<int64_t>& recv_off_me_of, cudaStream_t s) {
    const int P = c->nparts;
    const int64_t ns = (int64_t)h.send_idx.size();
    struct E {
        int32_t src, peer;
        int64_t dst;
    };
    std::vector<E> ent(ns);
    for (int q = 0; q < P; q++)
        for (int64_t k = 0; k < h.send_cnt[q]; k++) {
            const int64_t i = h.send_off[q] + k;
            ent[i] = E{h.send_idx[i], q, n_own_of[q] + recv_off_me_of[q] + k};
        }
    (void)me;
    // sorted by owned row: a block pushes the entries of the rows it owns
    std::stable_sort(ent.begin(), ent.end(), [](const E& a, const E& b) { return a.src < b.src; });
    std::vector<int32_t> src(ns), peer(ns);
    std::vector<int64_t> dst(ns);
    for (int64_t i = 0; i < ns; i++) {
        src[i] = ent[i].src;
        peer[i] = ent[i].peer;
        dst[i] = ent[i].dst;
    }
    const int64_t ngrp = d.n_own / 8 + 2;
    std::vector<int64_t> csp(ngrp + 1, 0);
    for (int64_t i = 0; i < ns; i++) csp[src[i] / 8 + 1]++;
    for (int64_t g = 0; g < ngrp; g++) csp[g + 1] += csp[g];
    void* p;
    MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (ns + 1)));
    d.send_src = (const int32_t*)p;
    if (ns) MIS2_CUDA_TRY(cudaMemcpyAsync(p, src.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (ns + 1)));
    d.send_peer = (const int32_t*)p;
    if (ns) MIS2_CUDA_TRY(cudaMemcpyAsync(p, peer.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    MIS2_TRY(dev_alloc(c, &p, sizeof(int64_t) * (ns + 1)));
    d.send_dst = (const int64_t*)p;
    if (ns) MIS2_CUDA_TRY(cudaMemcpyAsync(p, dst.data(), sizeof(int64_t) * ns, cudaMemcpyHostToDevice, s));
    MIS2_TRY(dev_alloc(c, &p, sizeof(int64_t) * (ngrp + 1)));
    d.send_csp = (const int64_t*)p;
    MIS2_CUDA_TRY(cudaMemcpyAsync(p, csp.data(), sizeof(int64_t) * (ngrp + 1), cudaMemcpyHostToDevice, s));
    d.nsend = ns;
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));  // the host vectors go out of scope
    return MIS2_OK;
}

// ------------------------------------------------------------------ halo exchange
// ghost values of a per-part array of es-byte elements (1 or 4): arr[i] is
// part i's local array [owned | ghosts]; the send buffers of T are scratch
static int exchange_arr(mis2_comm* c, const std::vector<void*>& arr, int es, cudaStream_t s) {
    const int P = c->nparts;
    const int L = (int)c->dev.size();
    for (int i = 0; i < L; i++) {
        const int64_t ns = (int64_t)c->hp[i].send_idx.size();
        if (!ns) continue;
        const int blocks = (int)std::min<int64_t>((ns + 255) / 256, 1024);
        if (es == 1) k_pack_u8<<<blocks, 256, 0, s>>>((const uint8_t*)arr[i], c->send_idx_d[i], ns, (uint8_t*)c->sendT[i]);
        else k_pack_u32<<<blocks, 256, 0, s>>>((const uint32_t*)arr[i], c->send_idx_d[i], ns, (uint32_t*)c->sendT[i]);
        count_launch();
    }
    MIS2_CUDA_TRY(cudaGetLastError());
    if (c->local) {
        for (int p = 0; p < P; p++) {
            char* dst = (char*)arr[p];
            for (int q = 0; q < P; q++) {
                const int64_t cnt = c->hp[p].recv_cnt[q];
                if (!cnt || q == p) continue;
                const char* src = (const char*)c->sendT[q] + es * c->hp[q].send_off[p];
                MIS2_CUDA_TRY(cudaMemcpyAsync(dst + es * (c->dev[p].n_own + c->hp[p].recv_off[q]), src, es * cnt,
                                              cudaMemcpyDeviceToDevice, s));
            }
        }
        return MIS2_OK;
    }
    const HostPart& h = c->hp[0];
    const PartDev& d = c->dev[0];
    const ncclDataType_t ty = es == 1 ? ncclUint8 : ncclInt32;
    char* dst = (char*)arr[0];
    const char* sb = (const char*)c->sendT[0];
    NCCL_TRY(c->api, c->api->GroupStart());
    for (int q = 0; q < P; q++) {
        if (q == c->rank) continue;
        if (h.send_cnt[q]) NCCL_TRY(c->api, c->api->Send(sb + es * h.send_off[q], h.send_cnt[q], ty, q, c->nccl, s));
        if (h.recv_cnt[q])
            NCCL_TRY(c->api, c->api->Recv(dst + es * (d.n_own + h.recv_off[q]), h.recv_cnt[q], ty, q, c->nccl, s));
    }
    NCCL_TRY(c->api, c->api->GroupEnd());
    return MIS2_OK;
}

// per-part int64 values -> all of them on the host, in part order
static int gather_counts(mis2_comm* c, const std::vector<int64_t>& mine, std::vector<int64_t>& all, cudaStream_t s) {
    const int P = c->nparts;
    all.assign(P, 0);
    if (c->local) {
        for (int p = 0; p < P; p++) all[p] = mine[p];
        return MIS2_OK;
    }
    int64_t* d_in = c->d_counts;  // allocated with the graph: no allocation per call
    int64_t* d_all = c->d_counts + 1;
    MIS2_CUDA_TRY(cudaMemcpyAsync(d_in, &mine[0], sizeof(int64_t), cudaMemcpyHostToDevice, s));
    NCCL_TRY(c->api, c->api->AllGather(d_in, d_all, 1, ncclInt64, c->nccl, s));
    MIS2_CUDA_TRY(cudaMemcpyAsync(all.data(), d_all, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    return MIS2_OK;
}

extern "C" {

int mis2_plan_part(int64_t n_global, int nparts, int part, const int64_t* rowptr_local, const int32_t* colinds_global,
                   int64_t* n_ghost, int64_t* ghost_ids, int64_t* req_counts, int32_t* colinds_local) {
    reset_launches();
    if (n_global < 0 || nparts < 1 || part < 0 || part >= nparts || !rowptr_local || !n_ghost || !req_counts) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    HostPart hp;
    MIS2_TRY(plan_local(n_global, nparts, part, rowptr_local, colinds_global, hp));
    *n_ghost = (int64_t)hp.ghosts.size();
    for (int q = 0; q < nparts; q++) req_counts[q] = hp.recv_cnt[q];
    if (ghost_ids) memcpy(ghost_ids, hp.ghosts.data(), sizeof(int64_t) * hp.ghosts.size());
    if (colinds_local) memcpy(colinds_local, hp.colinds.data(), sizeof(int32_t) * hp.colinds.size());
    return MIS2_OK;
}

int mis2_comm_unique_id(uint8_t* id128) {
    reset_launches();
    NcclApi* api;
    MIS2_TRY(nccl_api(&api));
    ncclUniqueId u;
    NCCL_TRY(api, api->GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    memcpy(id128, &u, 128);
    return MIS2_OK;
}

int mis2_comm_init_nccl(const uint8_t* id128, int nranks, int rank, mis2_comm** out) {
    reset_launches();
    if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    NcclApi* api;
    MIS2_TRY(nccl_api(&api));
    mis2_comm* c = new mis2_comm();
    c->api = api;
    c->nparts = nranks;
    c->rank = rank;
    ncclUniqueId u;
    memcpy(&u, id128, 128);
    ncclResult_t r = api->CommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
        set_error("ncclCommInitRank: %s", api->GetErrorString(r));
        delete c;
        return MIS2_ENCCL;
    }
    *out = c;
    return MIS2_OK;
}

int mis2_comm_init_local(int nparts, mis2_comm** out) {
    reset_launches();
    if (nparts < 1 || !out) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    mis2_comm* c = new mis2_comm();
    c->local = true;
    c->nparts = nparts;
    *out = c;
    return MIS2_OK;
}

int mis2_comm_destroy(mis2_comm* c) {
    if (!c) return MIS2_OK;
    free_parts(c);
    if (c->nccl && c->api) c->api->CommDestroy(c->nccl);
    delete c;
    return MIS2_OK;
}

int mis2_comm_set_graph(mis2_comm* c, int64_t n_global, const int64_t* rowptr_h, const int32_t* colinds_h,
                        void* stream) {
    reset_launches();
    if (!c || n_global < 0 || !rowptr_h || n_global > 2147483645LL) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    free_parts(c);
    c->n_global = n_global;
    const int P = c->nparts;
    if (c->local) {
        c->hp.resize(P);
        for (int q = 0; q < P; q++) {
            const int64_t lo = part_lo(n_global, P, q);
            MIS2_TRY(plan_local(n_global, P, q, rowptr_h + lo, colinds_h, c->hp[q]));
        }
        // owner q sends to p the ghosts p requests from q (ascending ids)
        for (int q = 0; q < P; q++) {
            std::vector<std::vector<int64_t>> wanted(P);
            for (int p = 0; p < P; p++) {
                if (p == q) continue;
                const HostPart& hpp = c->hp[p];
                wanted[p].assign(hpp.ghosts.begin() + hpp.recv_off[q], hpp.ghosts.begin() + hpp.recv_off[q + 1]);
            }
            finish_sends(c->hp[q], wanted, P);
        }
    } else {
        c->hp.resize(1);
        HostPart& h = c->hp[0];
        MIS2_TRY(plan_local(n_global, P, c->rank, rowptr_h, colinds_h, h));
        // all-to-all of the request lists: counts (allgather), then ids
        std::vector<int64_t> cnt_all((size_t)P * P, 0);
        int64_t *d_cnt, *d_all;
        MIS2_CUDA_TRY(cudaMalloc(&d_cnt, sizeof(int64_t) * P));
        MIS2_CUDA_TRY(cudaMalloc(&d_all, sizeof(int64_t) * P * P));
        MIS2_CUDA_TRY(cudaMemcpyAsync(d_cnt, h.recv_cnt.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, s));
        NCCL_TRY(c->api, c->api->AllGather(d_cnt, d_all, P, ncclInt64, c->nccl, s));
        MIS2_CUDA_TRY(cudaMemcpyAsync(cnt_all.data(), d_all, sizeof(int64_t) * P * P, cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
        cudaFree(d_cnt);
        cudaFree(d_all);
        int64_t tot_in = 0;
        for (int p = 0; p < P; p++) tot_in += (p == c->rank) ? 0 : cnt_all[(size_t)p * P + c->rank];
        int64_t *d_req, *d_in;
        MIS2_CUDA_TRY(cudaMalloc(&d_req, sizeof(int64_t) * (h.ghosts.size() + 1)));
        MIS2_CUDA_TRY(cudaMalloc(&d_in, sizeof(int64_t) * (tot_in + 1)));
        if (!h.ghosts.empty())
            MIS2_CUDA_TRY(cudaMemcpyAsync(d_req, h.ghosts.data(), sizeof(int64_t) * h.ghosts.size(),
                                          cudaMemcpyHostToDevice, s));
        std::vector<int64_t> in_off(P + 1, 0);
        for (int p = 0; p < P; p++) in_off[p + 1] = in_off[p] + ((p == c->rank) ? 0 : cnt_all[(size_t)p * P + c->rank]);
        NCCL_TRY(c->api, c->api->GroupStart());
        for (int q = 0; q < P; q++) {
            if (q == c->rank) continue;
            if (h.recv_cnt[q]) NCCL_TRY(c->api, c->api->Send(d_req + h.recv_off[q], h.recv_cnt[q], ncclInt64, q, c->nccl, s));
            const int64_t k = in_off[q + 1] - in_off[q];
            if (k) NCCL_TRY(c->api, c->api->Recv(d_in + in_off[q], k, ncclInt64, q, c->nccl, s));
        }
        NCCL_TRY(c->api, c->api->GroupEnd());
        std::vector<int64_t> in(tot_in);
        if (tot_in) MIS2_CUDA_TRY(cudaMemcpyAsync(in.data(), d_in, sizeof(int64_t) * tot_in, cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
        cudaFree(d_req);
        cudaFree(d_in);
        std::vector<std::vector<int64_t>> wanted(P);
        for (int p = 0; p < P; p++) wanted[p].assign(in.begin() + in_off[p], in.begin() + in_off[p + 1]);
        finish_sends(h, wanted, P);
    }
    c->dev.resize(c->hp.size());
    for (size_t i = 0; i < c->hp.size(); i++) MIS2_TRY(upload_part(c, c->hp[i], c->dev[i], s));
    {
        void* p;
        MIS2_TRY(dev_alloc(c, &p, dist_scratch_bytes((int)c->dev.size())));
        c->dscratch = p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int64_t) * 2 * (P + 1)));
        c->d_counts = (int64_t*)p;
    }
    c->peer_T.assign(P, nullptr);
    c->peer_M.assign(P, nullptr);
    c->peer_box.assign(P, nullptr);
    if (c->local) {
        // every part's buffers are on this device: the halo pushes and the
        // mailbox posts of the partitioned kernel are plain device stores
        std::vector<int64_t> n_own_of(P);
        for (int q = 0; q < P; q++) {
            n_own_of[q] = c->dev[q].n_own;
            c->peer_T[q] = c->dev[q].T;
            c->peer_M[q] = c->dev[q].M;
            c->peer_box[q] = c->dev[q].box;
            c->dev[q].gpart = q;
        }
        for (int q = 0; q < P; q++) {
            std::vector<int64_t> roff(P);  // where q's sends land in each peer
            for (int d = 0; d < P; d++) roff[d] = c->hp[d].recv_off[q];
            MIS2_TRY(upload_sends(c, c->hp[q], c->dev[q], q, n_own_of, roff, s));
        }
    } else {
        // one part per rank: its peers' T / M / mailboxes are mapped over
        // NVLink (CUDA IPC; handles and ghost layouts allgathered over NCCL)
        const int me = c->rank;
        PartDev& d = c->dev[0];
        d.gpart = me;
        // layout: [n_own, recv_off[0..P)] of every rank
        std::vector<int64_t> lay((size_t)(P + 1)), lay_all((size_t)(P + 1) * P);
        lay[0] = d.n_own;
        for (int q = 0; q < P; q++) lay[1 + q] = c->hp[0].recv_off[q];
        cudaIpcMemHandle_t hs[3];
        MIS2_CUDA_TRY(cudaIpcGetMemHandle(&hs[0], d.T));
        MIS2_CUDA_TRY(cudaIpcGetMemHandle(&hs[1], d.M));
        MIS2_CUDA_TRY(cudaIpcGetMemHandle(&hs[2], d.box));
        const size_t hb = sizeof(hs), lb = sizeof(int64_t) * (P + 1);
        void* buf;
        MIS2_CUDA_TRY(cudaMalloc(&buf, (hb + lb) * (P + 1)));
        char* mine = (char*)buf;
        char* all = mine + hb + lb;
        MIS2_CUDA_TRY(cudaMemcpyAsync(mine, hs, hb, cudaMemcpyHostToDevice, s));
        MIS2_CUDA_TRY(cudaMemcpyAsync(mine + hb, lay.data(), lb, cudaMemcpyHostToDevice, s));
        NCCL_TRY(c->api, c->api->AllGather(mine, all, hb + lb, ncclUint8, c->nccl, s));
        std::vector<char> host((hb + lb) * P);
        MIS2_CUDA_TRY(cudaMemcpyAsync(host.data(), all, (hb + lb) * P, cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
        cudaFree(buf);
        std::vector<int64_t> n_own_of(P), roff(P);
        for (int q = 0; q < P; q++) {
            const char* rec = host.data() + (hb + lb) * q;
            const int64_t* ql = (const int64_t*)(rec + hb);
            n_own_of[q] = ql[0];
            roff[q] = ql[1 + me];  // where my sends land in q
            if (q == me) {
                c->peer_T[q] = d.T;
                c->peer_M[q] = d.M;
                c->peer_box[q] = d.box;
                continue;
            }
            cudaIpcMemHandle_t qh[3];
            memcpy(qh, rec, hb);
            void* ptr[3];
            for (int k = 0; k < 3; k++) {
                MIS2_CUDA_TRY(cudaIpcOpenMemHandle(&ptr[k], qh[k], cudaIpcMemLazyEnablePeerAccess));
                c->ipc_opened.push_back(ptr[k]);
            }
            c->peer_T[q] = (uint64_t*)ptr[0];
            c->peer_M[q] = (uint32_t*)ptr[1];
            c->peer_box[q] = (unsigned long long*)ptr[2];
        }
        MIS2_TRY(upload_sends(c, c->hp[0], d, me, n_own_of, roff, s));
    }
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    return MIS2_OK;
}

}  // extern "C"

// Alg. 1 over the partition (one launch of the partitioned persistent
// kernel, mis2_kernel.cuh mis2_dist_persistent).  in_sets[i] = part i's
// owned mask; labels[i] (or empty) = part i's phase-2 mask (active iff < 0,
// owned rows).
static int dist_mis2_run(mis2_comm* c, const mis2_opts& opt, const std::vector<uint8_t*>& in_sets,
                         const std::vector<const int32_t*>& labels, int64_t* count, int32_t* iters, cudaStream_t s) {
    const int max_iters = max_iters_for(c->n_global, opt.max_iters);
    const int L = (int)c->dev.size();
    int64_t n_loc = 0, nnz_loc = 0;
    for (int i = 0; i < L; i++) {
        PartDev& d = c->dev[i];
        d.seed = opt.seed;
        d.scheme = opt.scheme;
        d.hshift = (opt.flags & MIS2_FLAG_WORD32) ? 32 : 0;
        d.labels = labels.empty() ? nullptr : labels[i];
        d.in_set = in_sets[i];
        n_loc += d.n_own;
        nnz_loc += d.nnz;
    }
    // one lane-group width for every local part (the persistent kernel is
    // one launch); the ranks of the NCCL transport each choose from their
    // own rows, which only changes the work split, never the result
    const int G = opt.group ? opt.group : choose_group(n_loc, nnz_loc, 0);
    return dist_mis2_launch(c->dev, c->peer_T, c->peer_M, c->peer_box, !c->local, G, max_iters, &c->epoch,
                            c->dscratch, count, iters, s);
}

static int agg_alloc(mis2_comm* c) {
    if (!c->agg.empty()) return MIS2_OK;
    const int L = (int)c->dev.size();
    c->agg.resize(L);
    int32_t* shared_size = nullptr;
    for (int i = 0; i < L; i++) {
        AggPart& a = c->agg[i];
        const PartDev& d = c->dev[i];
        const int64_t nl = d.n_own + d.n_ghost + 1;
        void* p;
        MIS2_TRY(dev_alloc(c, &p, nl)); a.in1 = (uint8_t*)p;
        MIS2_TRY(dev_alloc(c, &p, nl)); a.in2 = (uint8_t*)p;
        MIS2_TRY(dev_alloc(c, &p, nl)); a.acc = (uint8_t*)p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * nl)); a.rid = (int32_t*)p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * nl)); a.aid = (int32_t*)p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * nl)); a.lab = (int32_t*)p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * nl)); a.tent = (int32_t*)p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (d.n_own + 1))); a.heavy = (int32_t*)p;
        MIS2_TRY(dev_alloc(c, &p, scan_ws_bytes(d.n_own))); a.scan_tmp = p;
        MIS2_TRY(dev_alloc(c, &p, sizeof(long long) * 16)); a.scal = (long long*)p;
        if (!c->local || i == 0) {
            MIS2_TRY(dev_alloc(c, &p, sizeof(int32_t) * (c->n_global + 1)));
            shared_size = (int32_t*)p;
        }
        a.size = shared_size;  // LOCAL: every part adds into the one global histogram
    }
    return MIS2_OK;
}

// Alg. 3 over the partition, bit-identical to mis2_aggregate():
// the two MIS-2 calls run partitioned; roots are numbered by a global
// exclusive prefix (per-part counts gathered); every array read through a
// neighbour is completed with its ghost values before the pass that reads
// it; the aggregate sizes of phase 3 are summed over the parts.
static int dist_aggregate_run(mis2_comm* c, const mis2_opts& opt, const std::vector<int32_t*>& labels_out,
                              int64_t* num_aggs, int64_t* stats, cudaStream_t s) {
    MIS2_TRY(agg_alloc(c));
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    const int L = (int)c->dev.size();
    std::vector<void*> v_in1(L), v_acc(L), v_rid(L), v_aid(L), v_lab(L);
    std::vector<uint8_t*> in1(L), in2(L);
    std::vector<const int32_t*> labs(L);
    for (int i = 0; i < L; i++) {
        AggPart& a = c->agg[i];
        v_in1[i] = a.in1; v_acc[i] = a.acc; v_rid[i] = a.rid; v_aid[i] = a.aid; v_lab[i] = a.lab;
        in1[i] = a.in1; in2[i] = a.in2; labs[i] = a.lab;
        MIS2_CUDA_TRY(cudaMemsetAsync(a.scal, 0, sizeof(long long) * 16, s));
    }
    auto scal_i32 = [&](int i, int slot) { return (int32_t*)&c->agg[i].scal[slot]; };
    // local counts (int32 device scalar at slot) -> global exclusive offsets and the total
    auto offsets = [&](int slot, std::vector<int64_t>& off, int64_t& total) -> int {
        std::vector<int64_t> mine(L, 0);
        for (int i = 0; i < L; i++) {
            int32_t v = 0;
            MIS2_CUDA_TRY(cudaMemcpyAsync(&v, scal_i32(i, slot), sizeof(v), cudaMemcpyDeviceToHost, s));
            MIS2_CUDA_TRY(cudaStreamSynchronize(s));
            mine[i] = v;
        }
        std::vector<int64_t> all;
        MIS2_TRY(gather_counts(c, mine, all, s));
        const int P = c->nparts;
        std::vector<int64_t> ex(P + 1, 0);
        for (int q = 0; q < P; q++) ex[q + 1] = ex[q] + all[q];
        off.assign(L, 0);
        for (int i = 0; i < L; i++) off[i] = ex[c->local ? i : c->rank];
        total = ex[P];
        return MIS2_OK;
    };

    // ---- phase 1: M1 = MIS2(G); roots numbered in vertex order; pull labels
    int64_t cnt1 = 0, cnt2 = 0;
    int32_t it1 = 0, it2 = 0;
    MIS2_TRY(dist_mis2_run(c, opt, in1, {}, &cnt1, &it1, s));
    for (int i = 0; i < L; i++)
        MIS2_TRY(scan_flags(c->agg[i].in1, c->dev[i].n_own, c->agg[i].rid, scal_i32(i, 0), c->agg[i].scan_tmp, s));
    std::vector<int64_t> off1;
    int64_t n1 = 0;
    MIS2_TRY(offsets(0, off1, n1));
    for (int i = 0; i < L; i++) {
        const int64_t no = c->dev[i].n_own;
        if (off1[i] && no) {
            k_add_i32<<<(unsigned)std::min<int64_t>((no + 255) / 256, 4096), 256, 0, s>>>(c->agg[i].rid, no, (int32_t)off1[i]);
            count_launch();
        }
    }
    MIS2_TRY(exchange_arr(c, v_in1, 1, s));
    MIS2_TRY(exchange_arr(c, v_rid, 4, s));
    for (int i = 0; i < L; i++) {
        const PartDev& d = c->dev[i];
        agg_phase1(d.G, d.n_own, d.rowptr, d.colinds, c->agg[i].in1, c->agg[i].rid, c->agg[i].lab,
                   (int*)scal_i32(i, 2), di.sms, s);
    }
    // ---- phase 2: M2 = MIS2(G \ aggregated) (reading Q15); accept >= 2 unaggregated neighbours
    MIS2_TRY(dist_mis2_run(c, opt, in2, labs, &cnt2, &it2, s));
    MIS2_TRY(exchange_arr(c, v_lab, 4, s));
    for (int i = 0; i < L; i++) {
        const PartDev& d = c->dev[i];
        agg_accept(d.G, d.n_own, d.rowptr, d.colinds, c->agg[i].in2, c->agg[i].lab, c->agg[i].acc, di.sms, s);
        MIS2_TRY(scan_flags(c->agg[i].acc, d.n_own, c->agg[i].aid, scal_i32(i, 0), c->agg[i].scan_tmp, s));
    }
    std::vector<int64_t> off2;
    int64_t n2 = 0;
    MIS2_TRY(offsets(0, off2, n2));
    for (int i = 0; i < L; i++) {
        const int64_t no = c->dev[i].n_own;
        if (off2[i] && no) {
            k_add_i32<<<(unsigned)std::min<int64_t>((no + 255) / 256, 4096), 256, 0, s>>>(c->agg[i].aid, no, (int32_t)off2[i]);
            count_launch();
        }
        k_set_i32<<<1, 1, 0, s>>>(scal_i32(i, 8), (int32_t)n1);
        count_launch();
    }
    MIS2_TRY(exchange_arr(c, v_acc, 1, s));
    MIS2_TRY(exchange_arr(c, v_aid, 4, s));
    for (int i = 0; i < L; i++) {
        const PartDev& d = c->dev[i];
        agg_phase2_label(d.G, d.n_own, d.rowptr, d.colinds, c->agg[i].acc, c->agg[i].aid, scal_i32(i, 8),
                         c->agg[i].lab, (int*)scal_i32(i, 2), di.sms, s);
    }
    // ---- phase 3: frozen labels (ghosts too); sizes summed over the parts
    MIS2_TRY(exchange_arr(c, v_lab, 4, s));
    const int64_t na = n1 + n2;
    for (int i = 0; i < L; i++) {
        if (!c->local || i == 0) MIS2_CUDA_TRY(cudaMemsetAsync(c->agg[i].size, 0, sizeof(int32_t) * (na + 1), s));
    }
    for (int i = 0; i < L; i++) {
        const PartDev& d = c->dev[i];
        AggPart& a = c->agg[i];
        agg_tent_size(d.n_own, a.lab, a.tent, a.size, (unsigned long long*)&a.scal[3], di.sms, s);
        if (d.n_ghost)
            MIS2_CUDA_TRY(cudaMemcpyAsync(a.tent + d.n_own, a.lab + d.n_own, sizeof(int32_t) * d.n_ghost,
                                          cudaMemcpyDeviceToDevice, s));
    }
    if (!c->local && na > 0)
        NCCL_TRY(c->api, c->api->AllReduce(c->agg[0].size, c->agg[0].size, (size_t)na, ncclInt32, ncclSum, c->nccl, s));
    for (int i = 0; i < L; i++) {
        const PartDev& d = c->dev[i];
        AggPart& a = c->agg[i];
        agg_phase3(d.G, d.n_own, d.rowptr, d.colinds, a.tent, a.size, a.lab, a.heavy, (int*)scal_i32(i, 4),
                   (int*)scal_i32(i, 2), di.sms, s);
        if (d.n_own)
            MIS2_CUDA_TRY(cudaMemcpyAsync(labels_out[i], a.lab, sizeof(int32_t) * d.n_own, cudaMemcpyDeviceToDevice, s));
    }
    MIS2_CUDA_TRY(cudaGetLastError());
    // errors and leftovers over all parts
    long long err = 0, left = 0;
    for (int i = 0; i < L; i++) {
        long long h[16];
        MIS2_CUDA_TRY(cudaMemcpyAsync(h, c->agg[i].scal, sizeof(h), cudaMemcpyDeviceToHost, s));
        MIS2_CUDA_TRY(cudaStreamSynchronize(s));
        err |= ((const int32_t*)h)[2];
        left += h[3];
    }
    if (!c->local) {
        std::vector<int64_t> e1(1, err), l1(1, left), ea, la;
        MIS2_TRY(gather_counts(c, e1, ea, s));
        MIS2_TRY(gather_counts(c, l1, la, s));
        err = 0;
        left = 0;
        for (int64_t x : ea) err |= x;
        for (int64_t x : la) left += x;
    }
    if (err) {
        set_error("aggregation invariant failed (flags 0x%llx): input graph not symmetric?", (long long)err);
        return MIS2_EINTERNAL;
    }
    *num_aggs = na;
    if (stats) {
        stats[0] = cnt1;
        stats[1] = it1;
        stats[2] = cnt2;
        stats[3] = it2;
        stats[4] = n2;
        stats[5] = left;
        stats[6] = n1;
        stats[7] = na;
    }
    return MIS2_OK;
}

extern "C" {

int mis2_dist_mis2(mis2_comm* c, const mis2_opts* o, uint8_t* in_set, int64_t* count, int32_t* iters, void* stream) {
    reset_launches();
    if (!c || !count || !iters || c->dev.empty()) {
        set_error("bad arguments (graph not set?)");
        return MIS2_EINVAL;
    }
    if (c->n_global > 0 && !in_set) {
        set_error("null in_set");
        return MIS2_EINVAL;
    }
    mis2_opts def;
    mis2_opts_default(&def);
    const mis2_opts& opt = o ? *o : def;
    if (opt.prio_override) {
        set_error("prio_override is not supported by the partitioned driver");
        return MIS2_EINVAL;
    }
    if ((opt.flags & MIS2_FLAG_WORD32) && bits_for(c->n_global) > 31) {
        set_error("MIS2_FLAG_WORD32 needs ceil(log2(n + 2)) <= 31");
        return MIS2_EINVAL;
    }
    std::vector<uint8_t*> ins(c->dev.size());
    for (size_t i = 0; i < c->dev.size(); i++) ins[i] = c->local ? in_set + c->hp[i].lo : in_set;
    return dist_mis2_run(c, opt, ins, {}, count, iters, (cudaStream_t)stream);
}

// device scratch of the coarsening steps: slot k of the communicator's
// pool, grown when a call needs more and kept for the next call (no
// allocation per call once the sizes have been seen; freed with the graph)
struct DevBuf {
    void* p = nullptr;
    mis2_comm* c = nullptr;
    int slot = 0;
    DevBuf() = default;
    DevBuf(mis2_comm* cc, int k) : c(cc), slot(k) {}
    int alloc(size_t bytes) {
        if (bytes < 256) bytes = 256;
        if ((int)c->pool.size() <= slot) c->pool.resize(slot + 1, {nullptr, 0});
        auto& e = c->pool[slot];
        if (e.second < bytes) {
            if (e.first) cudaFree(e.first);
            e = {nullptr, 0};
            if (cudaMalloc(&e.first, bytes) != cudaSuccess) {
                set_error("cudaMalloc(%zu) failed", bytes);
                return MIS2_ECUDA;
            }
            e.second = bytes;
        }
        p = e.first;
        return MIS2_OK;
    }
};
enum { kSlotWsPart = 0, kSlotSrow, kSlotSlab, kSlotScol, kSlotArow, kSlotPcol, kSlotAcol, kSlotWsMerge, kSlotPart0 };

// coarse rows (per-part edges) of one part: run_coarsen on its rows with the
// labels of its ghosts filled in (the coarse rows of aggregates it does not
// touch stay empty)
static int part_coarse(mis2_comm* c, const PartDev& d, const int32_t* lab, int64_t na, DevBuf& crow, DevBuf& ccol,
                       int64_t& nnz, cudaStream_t s) {
    mis2_graph gl{d.n_own, d.nnz, d.rowptr, d.colinds};
    mis2_graph gs{std::max<int64_t>(d.n_own, na), d.nnz, nullptr, nullptr};
    size_t wsb = 0;
    MIS2_TRY(run_coarsen(gs, nullptr, 0, nullptr, nullptr, 0, nullptr, nullptr, 0, s, &wsb));
    DevBuf ws(c, kSlotWsPart);
    MIS2_TRY(ws.alloc(wsb));
    MIS2_TRY(crow.alloc(sizeof(int64_t) * (na + 1)));
    int rc = run_coarsen(gl, lab, na, (int64_t*)crow.p, nullptr, 0, &nnz, ws.p, wsb, s, nullptr);
    if (rc != MIS2_ERANGE && rc != MIS2_OK) return rc;
    MIS2_TRY(ccol.alloc(sizeof(int32_t) * (nnz + 1)));
    return run_coarsen(gl, lab, na, (int64_t*)crow.p, (int32_t*)ccol.p, nnz, &nnz, ws.p, wsb, s, nullptr);
}

// The coarse graph of a partitioned graph, replicated on every part:
// each part builds the coarse rows its fine rows contribute (ghost labels
// exchanged first), the per-part coarse CSRs are stacked (allgather; LOCAL:
// already on the device) and merged by one more coarsening of the stacked
// graph with row label i mod na -- the union of each coarse row's edge sets,
// sorted and deduplicated: exactly mis2_coarsen() of the whole graph.
static int dist_coarsen_run(mis2_comm* c, const std::vector<const int32_t*>& labels_in, int64_t na, int64_t* c_rowptr,
                            int32_t* c_colinds, int64_t cap, int64_t* c_nnz, cudaStream_t s) {
    MIS2_TRY(agg_alloc(c));
    const int L = (int)c->dev.size();
    const int P = c->nparts;
    std::vector<void*> v_lab(L);
    for (int i = 0; i < L; i++) {
        v_lab[i] = c->agg[i].lab;
        if (c->dev[i].n_own)
            MIS2_CUDA_TRY(cudaMemcpyAsync(c->agg[i].lab, labels_in[i], sizeof(int32_t) * c->dev[i].n_own,
                                          cudaMemcpyDeviceToDevice, s));
    }
    MIS2_TRY(exchange_arr(c, v_lab, 4, s));
    std::vector<DevBuf> crow, ccol;
    for (int i = 0; i < L; i++) {
        crow.emplace_back(c, kSlotPart0 + 2 * i);
        ccol.emplace_back(c, kSlotPart0 + 2 * i + 1);
    }
    std::vector<int64_t> nnz(L, 0);
    for (int i = 0; i < L; i++) MIS2_TRY(part_coarse(c, c->dev[i], c->agg[i].lab, na, crow[i], ccol[i], nnz[i], s));
    // stacked graph: P * na rows
    std::vector<int64_t> all_nnz;
    MIS2_TRY(gather_counts(c, nnz, all_nnz, s));
    int64_t tot = 0, mx = 0;
    for (int64_t x : all_nnz) {
        tot += x;
        mx = std::max(mx, x);
    }
    const int64_t ns = (int64_t)P * na;
    DevBuf srow(c, kSlotSrow), scol(c, kSlotScol), slab(c, kSlotSlab), arow(c, kSlotArow), pcol(c, kSlotPcol),
        acol(c, kSlotAcol);
    MIS2_TRY(srow.alloc(sizeof(int64_t) * (ns + 1)));
    MIS2_TRY(slab.alloc(sizeof(int32_t) * (ns + 1)));
    MIS2_TRY(scol.alloc(sizeof(int32_t) * (tot + 1)));
    int64_t* sr = (int64_t*)srow.p;
    const unsigned gb = (unsigned)std::min<int64_t>((na + 256) / 256 + 1, 4096);
    // the coarse CSR of every part: on the device already (LOCAL) or
    // allgathered (NCCL: row pointers, and the columns padded to the largest
    // part's count -- only the first all_nnz[p] entries of a part are used)
    std::vector<const int64_t*> prow(P);
    std::vector<const int32_t*> pcolp(P);
    if (c->local) {
        for (int p = 0; p < P; p++) {
            prow[p] = (const int64_t*)crow[p].p;
            pcolp[p] = (const int32_t*)ccol[p].p;
        }
    } else {
        MIS2_TRY(arow.alloc(sizeof(int64_t) * (na + 1) * P));
        MIS2_TRY(pcol.alloc(sizeof(int32_t) * (mx + 1)));
        MIS2_TRY(acol.alloc(sizeof(int32_t) * ((mx + 1) * P)));
        if (nnz[0]) MIS2_CUDA_TRY(cudaMemcpyAsync(pcol.p, ccol[0].p, sizeof(int32_t) * nnz[0], cudaMemcpyDeviceToDevice, s));
        NCCL_TRY(c->api, c->api->AllGather(crow[0].p, arow.p, (size_t)(na + 1), ncclInt64, c->nccl, s));
        NCCL_TRY(c->api, c->api->AllGather(pcol.p, acol.p, (size_t)(mx + 1), ncclInt32, c->nccl, s));
        for (int p = 0; p < P; p++) {
            prow[p] = (const int64_t*)arow.p + (int64_t)p * (na + 1);
            pcolp[p] = (const int32_t*)acol.p + (int64_t)p * (mx + 1);
        }
    }
    // stacked graph: part p's coarse rows are rows [p*na, (p+1)*na), its
    // columns the contiguous range [off_p, off_p + all_nnz[p]) -- every row
    // ends where the next begins, the last at tot
    int64_t off = 0;
    for (int p = 0; p < P; p++) {
        k_shift_i64<<<gb, 256, 0, s>>>(prow[p], na, off, sr + (int64_t)p * na);
        count_launch();
        if (all_nnz[p])
            MIS2_CUDA_TRY(cudaMemcpyAsync((int32_t*)scol.p + off, pcolp[p], sizeof(int32_t) * all_nnz[p],
                                          cudaMemcpyDeviceToDevice, s));
        off += all_nnz[p];
    }
    MIS2_CUDA_TRY(cudaMemcpyAsync(sr + ns, &tot, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));  // `tot` is a host stack value
    k_mod_labels<<<(unsigned)std::min<int64_t>((ns + 255) / 256 + 1, 4096), 256, 0, s>>>((int32_t*)slab.p, ns, na);
    count_launch();
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    mis2_graph gm{ns, tot, sr, (const int32_t*)scol.p};
    size_t wsb = 0;
    MIS2_TRY(run_coarsen(gm, nullptr, 0, nullptr, nullptr, 0, nullptr, nullptr, 0, s, &wsb));
    DevBuf ws(c, kSlotWsMerge);
    MIS2_TRY(ws.alloc(wsb));
    return run_coarsen(gm, (const int32_t*)slab.p, na, c_rowptr, c_colinds, cap, c_nnz, ws.p, wsb, s, nullptr);
}

int mis2_dist_coarsen(mis2_comm* c, const int32_t* labels, int64_t num_aggs, int64_t* c_rowptr, int32_t* c_colinds,
                      int64_t cap, int64_t* c_nnz, void* stream) {
    reset_launches();
    if (!c || c->dev.empty() || !c_rowptr || !c_nnz || cap < 0 || num_aggs < 0 || (c->n_global > 0 && !labels)) {
        set_error("bad arguments (graph not set?)");
        return MIS2_EINVAL;
    }
    if (c->n_global > 0 && num_aggs == 0) {
        set_error("num_aggs out of range");
        return MIS2_EINVAL;
    }
    if (c->n_global == 0) {
        *c_nnz = 0;
        return cudaMemsetAsync(c_rowptr, 0, sizeof(int64_t) * (num_aggs + 1), (cudaStream_t)stream) == cudaSuccess
                   ? MIS2_OK
                   : MIS2_ECUDA;
    }
    std::vector<const int32_t*> ins(c->dev.size());
    for (size_t i = 0; i < c->dev.size(); i++) ins[i] = c->local ? labels + c->hp[i].lo : labels;
    return dist_coarsen_run(c, ins, num_aggs, c_rowptr, c_colinds, cap, c_nnz, (cudaStream_t)stream);
}

int mis2_dist_aggregate(mis2_comm* c, const mis2_opts* o, int32_t* labels, int64_t* num_aggs, int64_t* stats,
                        void* stream) {
    reset_launches();
    if (!c || !num_aggs || c->dev.empty()) {
        set_error("bad arguments (graph not set?)");
        return MIS2_EINVAL;
    }
    if (c->n_global > 0 && !labels) {
        set_error("null labels");
        return MIS2_EINVAL;
    }
    mis2_opts def;
    mis2_opts_default(&def);
    const mis2_opts& opt = o ? *o : def;
    if (opt.prio_override || (opt.flags & MIS2_FLAG_BASIC)) {
        set_error("prio_override / MIS2_FLAG_BASIC are not supported by the partitioned driver");
        return MIS2_EINVAL;
    }
    if ((opt.flags & MIS2_FLAG_WORD32) && bits_for(c->n_global) > 31) {
        set_error("MIS2_FLAG_WORD32 needs ceil(log2(n + 2)) <= 31");
        return MIS2_EINVAL;
    }
    std::vector<int32_t*> outs(c->dev.size());
    for (size_t i = 0; i < c->dev.size(); i++) outs[i] = c->local ? labels + c->hp[i].lo : labels;
    return dist_aggregate_run(c, opt, outs, num_aggs, stats, (cudaStream_t)stream);
}

int mis2_comm_part_info(mis2_comm* c, int part, int64_t* lo, int64_t* hi, int64_t* n_ghost) {
    if (!c || part < 0 || part >= (int)c->hp.size()) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    if (lo) *lo = c->hp[part].lo;
    if (hi) *hi = c->hp[part].hi;
    if (n_ghost) *n_ghost = (int64_t)c->hp[part].ghosts.size();
    return MIS2_OK;
}

}  // extern "C"
