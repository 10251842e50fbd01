// abi.cu -- the extern "C" entry points declared in include/mis2.h.
// Argument checking, workspace carving, error strings.  All compute is in
// mis2_core.cu / aggregate.cu / coarsen.cu / validate.cu / scan.cu.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include <algorithm>

#include "internal.h"

namespace mis2h {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
void count_launch(int k) { g_launches += k; }
void reset_launches() { g_launches = 0; }

int device_info(DeviceInfo* out) {
    int dev = 0;
    MIS2_CUDA_TRY(cudaGetDevice(&dev));
    static thread_local int cached_dev = -1;
    static thread_local DeviceInfo cached;
    if (cached_dev != dev) {
        int sms = 0, optin = 0;
        MIS2_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MIS2_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        cached.device = dev;
        cached.sms = sms;
        cached.smem_optin = (size_t)optin;
        cached_dev = dev;
    }
    *out = cached;
    return MIS2_OK;
}

static int check_graph(const mis2_graph* g, bool rowptr32_ok = false) {
    if (!g) { set_error("graph is NULL"); return MIS2_EINVAL; }
    if (g->rowptr_bits != 0 && g->rowptr_bits != 64 && !(g->rowptr_bits == 32 && rowptr32_ok)) {
        set_error("rowptr_bits %d not supported here (0/64%s)", g->rowptr_bits, rowptr32_ok ? " or 32" : "");
        return MIS2_EINVAL;
    }
    if (g->rowptr_bits == 32 && g->nnz > 2147483647LL) { set_error("rowptr_bits 32 needs nnz < 2^31"); return MIS2_EINVAL; }
    if (g->n < 0 || g->n > 2147483645LL) { set_error("n out of range [0, 2^31-3]: %lld", (long long)g->n); return MIS2_EINVAL; }
    if (g->nnz < 0) { set_error("nnz < 0"); return MIS2_EINVAL; }
    if (g->n > 0 && (!g->rowptr || (g->nnz > 0 && !g->colinds))) { set_error("null rowptr/colinds"); return MIS2_EINVAL; }
    return MIS2_OK;
}

static int check_opts(const mis2_opts* o, int64_t n) {
    if (!o) return MIS2_OK;
    if (o->scheme < 0 || o->scheme > 2) { set_error("bad scheme %d", o->scheme); return MIS2_EINVAL; }
    if (o->group != 0 && o->group != 1 && o->group != 2 && o->group != 4 && o->group != 8 && o->group != 16 &&
        o->group != 32) {
        set_error("group must be 0 (auto) or a power of two <= 32, got %d", o->group);
        return MIS2_EINVAL;
    }
    if (o->prio_override && o->prio_iters < 0) { set_error("prio_iters < 0"); return MIS2_EINVAL; }
    if ((o->flags & MIS2_FLAG_WORD32) && bits_for(n) > 31) {
        set_error("MIS2_FLAG_WORD32 needs ceil(log2(n + 2)) <= 31");
        return MIS2_EINVAL;
    }
    return MIS2_OK;
}

static size_t mis2_bytes(int64_t n, int64_t nnz) {
    DeviceInfo di;
    if (device_info(&di) != MIS2_OK) di.sms = 148;
    Carve c(nullptr, 0);
    Mis2Ws w;
    carve_mis2(c, n, nnz, max_coop_warps(di), &w);
    return c.off;
}

// int32 row pointers (rowptr_bits = 32): widened to int64 into the last
// 8(n+1) bytes (256-aligned) of the workspace, which the op then does not
// use (mis2_workspace_size includes them for every op).
__global__ void k_widen_rowptr(int64_t cnt, const int32_t* __restrict__ src, int64_t* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
static size_t widen_bytes(int64_t n) { return ((sizeof(int64_t) * ((size_t)n + 1) + 255) & ~size_t(255)) + 256; }
static int widen_graph(const mis2_graph* g, void* ws, size_t* ws_bytes, mis2_graph* out, cudaStream_t s) {
    *out = *g;
    out->rowptr_bits = 64;
    if (g->rowptr_bits != 32 || g->n == 0) return MIS2_OK;
    const size_t need = widen_bytes(g->n);
    if (*ws_bytes < need) { set_error("workspace too small for the widened int32 rowptr"); return MIS2_ENOMEM; }
    const size_t at = (*ws_bytes - need + 255) & ~size_t(255);
    int64_t* dst = (int64_t*)((char*)ws + at);
    const int64_t cnt = g->n + 1;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    const int64_t blocks = std::min<int64_t>((cnt + 255) / 256, (int64_t)di.sms * 8);
    k_widen_rowptr<<<(unsigned)blocks, 256, 0, s>>>(cnt, g->rowptr32, dst);
    count_launch();
    MIS2_CUDA_TRY(cudaGetLastError());
    out->rowptr = dst;
    *ws_bytes = *ws_bytes - need;
    return MIS2_OK;
}

}  // namespace mis2h

using namespace mis2h;

static int workspace_size_op(int64_t n, int64_t nnz, int32_t op, size_t* bytes);

extern "C" {

void mis2_opts_default(mis2_opts* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->scheme = MIS2_SCHEME_XORSTAR;
}

int mis2_workspace_size(int64_t n, int64_t nnz, int32_t op, size_t* bytes) {
    if (!bytes || n < 0 || nnz < 0) { set_error("bad arguments"); return MIS2_EINVAL; }
    reset_launches();
    const int rc = workspace_size_op(n, nnz, op, bytes);
    if (rc == MIS2_OK) *bytes += widen_bytes(n);
    return rc;
}

int mis2_validate_graph(const mis2_graph* g, void* ws, size_t ws_bytes, void* stream) {
    reset_launches();
    MIS2_TRY(check_graph(g, true));
    if (!ws) { set_error("workspace is NULL"); return MIS2_EINVAL; }
    mis2_graph gw;
    MIS2_TRY(widen_graph(g, ws, &ws_bytes, &gw, (cudaStream_t)stream));
    return run_validate(gw, ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

}  // extern "C"

static int workspace_size_op(int64_t n, int64_t nnz, int32_t op, size_t* bytes) {
    mis2_graph g{n, nnz, {nullptr}, nullptr, 0, 0};
    switch (op) {
        case MIS2_OP_MIS2: *bytes = mis2_bytes(n, nnz); return MIS2_OK;
        case MIS2_OP_MIS2_HOST: {
            DeviceInfo di;
            MIS2_TRY(device_info(&di));
            Carve c(nullptr, 0);
            Mis2Ws w;
            carve_mis2(c, n, nnz, max_coop_warps(di), &w);
            c.take<int64_t>((size_t)n + 1);
            c.take<int32_t>((size_t)nnz);
            c.take<uint8_t>((size_t)n + 1);
            *bytes = c.off;
            return MIS2_OK;
        }
        case MIS2_OP_AGGREGATE: return run_aggregate(g, mis2_opts{}, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, bytes);
        case MIS2_OP_COARSEN: return run_coarsen(g, nullptr, 0, nullptr, nullptr, 0, nullptr, nullptr, 0, 0, bytes);
        case MIS2_OP_VALIDATE: return run_validate(g, nullptr, 0, 0, bytes);
        case MIS2_OP_COLOR: return color_graph(g, 0, nullptr, nullptr, nullptr, 0, 0, bytes);
    }
    set_error("unknown op %d", op);
    return MIS2_EINVAL;
}

extern "C" {

int mis2_async(const mis2_graph* g, const mis2_opts* o, uint8_t* in_set, int64_t* d_count, int32_t* d_iters,
               int32_t* d_status, void* ws, size_t ws_bytes, void* stream) {
    reset_launches();
    MIS2_TRY(check_graph(g, true));
    MIS2_TRY(check_opts(o, g->n));
    if (!d_count || !d_iters || !d_status || (g->n > 0 && !in_set) || !ws) {
        set_error("null output or workspace");
        return MIS2_EINVAL;
    }
    mis2_opts def;
    mis2_opts_default(&def);
    const mis2_opts& opt = o ? *o : def;
    cudaStream_t s = (cudaStream_t)stream;
    mis2_graph gw;
    MIS2_TRY(widen_graph(g, ws, &ws_bytes, &gw, s));
    g = &gw;
    if (opt.flags & MIS2_FLAG_VALIDATE) MIS2_TRY(run_validate(*g, ws, ws_bytes, s, nullptr));
    Carve c(ws, ws_bytes);
    Mis2Ws w;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    carve_mis2(c, g->n, g->nnz, max_coop_warps(di), &w);
    if (!c.ok()) { set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes); return MIS2_ENOMEM; }
    return run_mis2(*g, opt, nullptr, in_set, d_count, d_iters, d_status, nullptr, w, s);
}

int mis2(const mis2_graph* g, const mis2_opts* o, uint8_t* in_set, int64_t* count, int32_t* iters,
         int64_t* stats, void* ws, size_t ws_bytes, void* stream) {
    reset_launches();
    MIS2_TRY(check_graph(g, true));
    MIS2_TRY(check_opts(o, g->n));
    if (!count || !iters || (g->n > 0 && !in_set) || !ws) { set_error("null output or workspace"); return MIS2_EINVAL; }
    mis2_opts def;
    mis2_opts_default(&def);
    const mis2_opts& opt = o ? *o : def;
    cudaStream_t s = (cudaStream_t)stream;
    mis2_graph gw;
    MIS2_TRY(widen_graph(g, ws, &ws_bytes, &gw, s));
    g = &gw;
    if (opt.flags & MIS2_FLAG_VALIDATE) MIS2_TRY(run_validate(*g, ws, ws_bytes, s, nullptr));
    Carve c(ws, ws_bytes);
    Mis2Ws w;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    carve_mis2(c, g->n, g->nnz, max_coop_warps(di), &w);
    int64_t* scal = (int64_t*)w.scal;
    if (!c.ok()) { set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes); return MIS2_ENOMEM; }
    int32_t* s32 = (int32_t*)(scal + 1);
    MIS2_TRY(run_mis2(*g, opt, nullptr, in_set, scal, s32, s32 + 1, stats, w, s));
    int64_t h[2];
    MIS2_CUDA_TRY(cudaMemcpyAsync(h, scal, sizeof(h), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    *count = h[0];
    *iters = ((int32_t*)&h[1])[0];
    const int32_t st = ((int32_t*)&h[1])[1];
    if (st != MIS2_OK) { set_error("MIS-2 did not converge within max_iters"); return st; }
    return MIS2_OK;
}

int mis2_host(int64_t n, int64_t nnz, const int64_t* rowptr_h, const int32_t* colinds_h, const mis2_opts* o,
              uint8_t* in_set_h, int64_t* count, int32_t* iters, void* ws, size_t ws_bytes, void* stream) {
    reset_launches();
    if (n < 0 || nnz < 0 || (n > 0 && (!rowptr_h || !in_set_h)) || (nnz > 0 && !colinds_h) || !count || !iters || !ws) {
        set_error("bad arguments");
        return MIS2_EINVAL;
    }
    mis2_opts def;
    mis2_opts_default(&def);
    const mis2_opts& opt = o ? *o : def;
    MIS2_TRY(check_opts(&opt, n));
    cudaStream_t s = (cudaStream_t)stream;
    Carve c(ws, ws_bytes);
    Mis2Ws w;
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    carve_mis2(c, n, nnz, max_coop_warps(di), &w);
    int64_t* d_rowptr = c.take<int64_t>((size_t)n + 1);
    int32_t* d_col = c.take<int32_t>((size_t)nnz);
    uint8_t* d_in = c.take<uint8_t>((size_t)n + 1);
    int64_t* scal = (int64_t*)w.scal;
    if (!c.ok()) { set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes); return MIS2_ENOMEM; }
    MIS2_CUDA_TRY(cudaMemcpyAsync(d_rowptr, rowptr_h, sizeof(int64_t) * ((size_t)n + 1), cudaMemcpyHostToDevice, s));
    if (nnz > 0)
        MIS2_CUDA_TRY(cudaMemcpyAsync(d_col, colinds_h, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice, s));
    mis2_graph g{n, nnz, d_rowptr, d_col};
    if (opt.flags & MIS2_FLAG_VALIDATE) MIS2_TRY(run_validate(g, ws, ws_bytes, s, nullptr));
    int32_t* s32 = (int32_t*)(scal + 1);
    MIS2_TRY(run_mis2(g, opt, nullptr, d_in, scal, s32, s32 + 1, nullptr, w, s));
    if (n > 0) MIS2_CUDA_TRY(cudaMemcpyAsync(in_set_h, d_in, (size_t)n, cudaMemcpyDeviceToHost, s));
    int64_t h[2];
    MIS2_CUDA_TRY(cudaMemcpyAsync(h, scal, sizeof(h), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    *count = h[0];
    *iters = ((int32_t*)&h[1])[0];
    const int32_t st = ((int32_t*)&h[1])[1];
    if (st != MIS2_OK) { set_error("MIS-2 did not converge within max_iters"); return st; }
    return MIS2_OK;
}

int mis2_aggregate(const mis2_graph* g, const mis2_opts* o, int32_t* labels, int64_t* num_aggs, int32_t* roots,
                   int64_t* stats, void* ws, size_t ws_bytes, void* stream) {
    reset_launches();
    MIS2_TRY(check_graph(g, true));
    MIS2_TRY(check_opts(o, g->n));
    if (!num_aggs || (g->n > 0 && !labels) || !ws) { set_error("null output or workspace"); return MIS2_EINVAL; }
    mis2_opts def;
    mis2_opts_default(&def);
    const mis2_opts& opt = o ? *o : def;
    cudaStream_t s = (cudaStream_t)stream;
    mis2_graph gw;
    MIS2_TRY(widen_graph(g, ws, &ws_bytes, &gw, s));
    g = &gw;
    if (opt.flags & MIS2_FLAG_VALIDATE) MIS2_TRY(run_validate(*g, ws, ws_bytes, s, nullptr));
    if (opt.prio_override) { set_error("prio_override is only supported by mis2()"); return MIS2_EINVAL; }
    return run_aggregate(*g, opt, labels, num_aggs, roots, stats, ws, ws_bytes, s, nullptr);
}

int mis2_coarsen(const mis2_graph* g, const int32_t* labels, int64_t num_aggs, int64_t* c_rowptr, int32_t* c_colinds,
                 int64_t cap, int64_t* c_nnz, void* ws, size_t ws_bytes, void* stream) {
    reset_launches();
    MIS2_TRY(check_graph(g, true));
    if (!c_nnz || !c_rowptr || (g->n > 0 && !labels) || !ws || cap < 0) { set_error("bad arguments"); return MIS2_EINVAL; }
    mis2_graph gw;
    MIS2_TRY(widen_graph(g, ws, &ws_bytes, &gw, (cudaStream_t)stream));
    g = &gw;
    return run_coarsen(*g, labels, num_aggs, c_rowptr, c_colinds, cap, c_nnz, ws, ws_bytes, (cudaStream_t)stream,
                       nullptr);
}

int64_t mis2_last_launch_count(void) { return g_launches; }

// measurement aid (not in mis2.h): copies the instrumentation words a
// MIS2_FLAG_TIMELINE run with MIS2_DBG_IT set left in the workspace
int mis2_debug_read(void* ws, size_t ws_bytes, int64_t n, long long* out, int64_t count) {
    return debug_read(ws, ws_bytes, n, out, count);
}

const char* mis2_strerror(int status) {
    switch (status) {
        case MIS2_OK: return "ok";
        case MIS2_EINVAL: return "invalid argument";
        case MIS2_ENOMEM: return "workspace too small";
        case MIS2_ECUDA: return "CUDA error";
        case MIS2_ENCCL: return "NCCL error";
        case MIS2_EGRAPH: return "graph violates the input contract";
        case MIS2_ENOTCONVERGED: return "not converged within max_iters";
        case MIS2_ERANGE: return "output capacity too small";
        case MIS2_EINTERNAL: return "internal invariant failed";
    }
    return "unknown status";
}

const char* mis2_last_error(void) { return g_err; }

const char* mis2_version(void) { return "libmis2 0.1 sm_100a (persistent MIS-2, Alg. 1/3, coarsen)"; }

}  // extern "C"
