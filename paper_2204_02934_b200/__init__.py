"""B200-native MIS-2 / MIS-2 aggregation / coarsening (arXiv 2204.02934).

Thin Python binding over the C ABI of ``libmis2.so`` (include/mis2.h):
argument marshalling only -- torch CUDA tensors become device pointers and
``torch.cuda.current_stream()`` becomes the cudaStream_t.  Every step of the
hot path runs in the sm_100a kernels of ``csrc/``.  There is no CPU fallback:
without the library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

__all__ = ["mis2", "mis2_async", "mis2_host", "aggregate", "coarsen", "validate_graph", "multilevel",
           "Mis2Error", "lib", "SCHEMES", "EXPORTS", "workspace"]

SCHEMES = {"xorstar": 0, "fixed": 1, "xor": 2}
OP_MIS2, OP_AGGREGATE, OP_COARSEN, OP_MIS2_HOST, OP_VALIDATE, OP_COLOR = 0, 1, 2, 3, 4, 5
OK, EINVAL, ENOMEM, ECUDA, ENCCL, EGRAPH, ENOTCONVERGED, ERANGE, EINTERNAL = 0, -1, -2, -3, -4, -5, -6, -7, -9
FLAG_VALIDATE = 1
FLAG_TIMELINE = 2
FLAG_BASIC = 4
FLAG_PUSH_DECIDE = 8
FLAG_PULL_DECIDE = 16
DECIDE = {"auto": 0, "push": FLAG_PUSH_DECIDE, "pull": FLAG_PULL_DECIDE}
FLAG_KEYS = 32
FLAG_NO_KEYS = 64
KEYS = {"auto": 0, "on": FLAG_KEYS, "off": FLAG_NO_KEYS}
FLAG_WORD32 = 128
FLAG_ITER_STATS = 256
WORD_BITS = {64: 0, 32: FLAG_WORD32}

# every symbol include/mis2.h declares
EXPORTS = ["mis2_opts_default", "mis2_workspace_size", "mis2", "mis2_async", "mis2_host", "mis2_aggregate",
           "mis2_coarsen", "mis2_validate_graph", "mis2_last_launch_count", "mis2_strerror", "mis2_last_error",
           "mis2_version", "mis2_comm_unique_id", "mis2_comm_init_nccl", "mis2_comm_init_local",
           "mis2_comm_set_graph", "mis2_dist_mis2", "mis2_dist_aggregate", "mis2_dist_coarsen", "mis2_comm_part_info", "mis2_comm_destroy",
           "mis2_plan_part", "mis2_color", "mis2_cgs_setup", "mis2_cgs_ncolors", "mis2_cgs_apply", "mis2_cgs_destroy"]


class Mis2Error(RuntimeError):
    def __init__(self, rc: int, where: str, detail: str = ""):
        super().__init__(f"{where}: {rc} {detail}")
        self.rc = rc


class _Graph(ctypes.Structure):
    # the C struct's rowptr / rowptr32 union is one pointer; rowptr_bits says which
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("rowptr", ctypes.c_void_p),
                ("colinds", ctypes.c_void_p), ("rowptr_bits", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _Opts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("max_iters", ctypes.c_int32), ("scheme", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("group", ctypes.c_int32), ("prio_override", ctypes.c_void_p),
                ("prio_iters", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None


def lib():
    """Load (building in-tree first if sources are newer) libmis2.so."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if os.environ.get("MIS2_LIB_PATH"):  # measurement only: A/B another build of the same ABI
            path = os.environ["MIS2_LIB_PATH"]
        elif _build.stale() and os.path.exists(_build.NVCC):
            path = _build.build()
        if not os.path.exists(path):
            raise ImportError(f"libmis2.so not built ({path}); run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        P, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
        L.mis2_workspace_size.argtypes = [I64, I64, I32, ctypes.POINTER(SZ)]
        L.mis2.argtypes = [P, P, P, P, P, P, P, SZ, P]
        L.mis2_async.argtypes = [P, P, P, P, P, P, P, SZ, P]
        L.mis2_host.argtypes = [I64, I64, P, P, P, P, P, P, P, SZ, P]
        L.mis2_aggregate.argtypes = [P, P, P, P, P, P, P, SZ, P]
        L.mis2_coarsen.argtypes = [P, P, I64, P, P, I64, P, P, SZ, P]
        L.mis2_validate_graph.argtypes = [P, P, SZ, P]
        L.mis2_dist_aggregate.argtypes = [P, P, P, P, P, P]
        L.mis2_dist_coarsen.argtypes = [P, P, I64, P, P, I64, P, P]
        L.mis2_color.argtypes = [P, ctypes.c_uint64, P, P, P, SZ, P]
        L.mis2_cgs_setup.argtypes = [P, P, P, I64, P, ctypes.c_uint64, P, P]
        L.mis2_cgs_ncolors.argtypes = [P]
        L.mis2_cgs_apply.argtypes = [P, P, P, I32, I32, P]
        L.mis2_cgs_destroy.argtypes = [P]
        L.mis2_last_launch_count.restype = I64
        L.mis2_strerror.restype = ctypes.c_char_p
        L.mis2_strerror.argtypes = [ctypes.c_int]
        L.mis2_last_error.restype = ctypes.c_char_p
        L.mis2_version.restype = ctypes.c_char_p
        L.mis2_opts_default.argtypes = [P]
        L.mis2_comm_unique_id.argtypes = [P]
        L.mis2_comm_init_nccl.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]
        L.mis2_comm_init_local.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
        L.mis2_comm_set_graph.argtypes = [P, I64, P, P, P]
        L.mis2_dist_mis2.argtypes = [P, P, P, P, P, P]
        L.mis2_comm_part_info.argtypes = [P, ctypes.c_int, P, P, P]
        L.mis2_comm_destroy.argtypes = [P]
        L.mis2_plan_part.argtypes = [I64, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P]
        for name in ("mis2", "mis2_async", "mis2_host", "mis2_aggregate", "mis2_coarsen", "mis2_validate_graph",
                     "mis2_workspace_size", "mis2_comm_unique_id", "mis2_comm_init_nccl", "mis2_comm_init_local",
                     "mis2_comm_set_graph", "mis2_dist_mis2", "mis2_comm_part_info", "mis2_comm_destroy",
                     "mis2_plan_part"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int, where: str, allow=()):
    if rc != OK and rc not in allow:
        L = lib()
        raise Mis2Error(rc, where, f"{L.mis2_strerror(rc).decode()}: {L.mis2_last_error().decode()}")
    return rc


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2204_02934_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


_ws_cache: dict = {}


def workspace(op: int, n: int, nnz: int):
    """Device workspace tensor for `op` (cached per device and size)."""
    torch = _torch()
    sz = ctypes.c_size_t(0)
    _check(lib().mis2_workspace_size(n, nnz, op, ctypes.byref(sz)), "mis2_workspace_size")
    dev = torch.cuda.current_device()
    key = (dev, op)
    t = _ws_cache.get(key)
    if t is None or t.numel() < sz.value:
        t = torch.empty(max(sz.value, 256), dtype=torch.uint8, device=f"cuda:{dev}")
        _ws_cache[key] = t
    return t, sz.value


def _graph(rowptr, colinds):
    """CSR tensors -> the C struct: rowptr int64 or int32 (rowptr_bits 32), colinds int32."""
    torch = _torch()
    assert rowptr.is_cuda and colinds.is_cuda, "rowptr/colinds must be CUDA tensors"
    assert rowptr.dtype in (torch.int64, torch.int32) and colinds.dtype == torch.int32
    assert rowptr.is_contiguous() and colinds.is_contiguous()
    n = rowptr.numel() - 1
    nnz = colinds.numel()
    bits = 32 if rowptr.dtype == torch.int32 else 64
    return _Graph(n, nnz, rowptr.data_ptr(), colinds.data_ptr() if nnz else None, bits, 0), n, nnz


def _opts(seed=0, scheme="xorstar", max_iters=0, group=0, validate=False, prio_override=None, decide="auto",
          keys="auto", word_bits=64):
    o = _Opts()
    lib().mis2_opts_default(ctypes.byref(o))
    o.seed = seed & ((1 << 64) - 1)
    o.scheme = SCHEMES[scheme]
    o.max_iters = max_iters
    o.group = group
    o.flags = (FLAG_VALIDATE if validate else 0) | DECIDE[decide] | KEYS[keys] | WORD_BITS[word_bits]
    if prio_override is not None:
        o.prio_override = prio_override.data_ptr()
        o.prio_iters = prio_override.shape[0]
    return o


@dataclass
class Mis2Result:
    in_set: "object"          # torch.uint8 CUDA tensor [n]
    count: int
    iterations: int
    rc: int = OK
    stats: np.ndarray | None = None
    launches: int = 0
    extra: dict | None = None  # timeline: init_us / final_us


def mis2(rowptr, colinds, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0, group: int = 0,
         validate: bool = False, prio_override=None, stats: bool = False, allow_partial: bool = False,
         out=None, timeline: bool = False, decide: str = "auto", keys: str = "auto",
         word_bits: int = 64) -> Mis2Result:
    """Alg. 1 through ``mis2()`` of the C ABI."""
    torch = _torch()
    g, n, nnz = _graph(rowptr, colinds)
    if prio_override is not None:
        prio_override = prio_override.to(device=rowptr.device, dtype=torch.int64).contiguous()
    o = _opts(seed, scheme, max_iters, group, validate, prio_override, decide, keys, word_bits)
    ws, wsb = workspace(OP_MIS2, n, nnz)
    in_set = out if out is not None else torch.empty(max(n, 1), dtype=torch.uint8, device=rowptr.device)
    cnt, its = ctypes.c_int64(0), ctypes.c_int32(0)
    st = None
    b = (n + 1).bit_length()
    mi = max_iters if max_iters > 0 else 10 * b + 20
    if stats:
        st = np.zeros((mi, 6), dtype=np.int64)
    elif timeline:
        o.flags |= FLAG_TIMELINE
        st = np.zeros(2 * mi + 2, dtype=np.int64)
    rc = lib().mis2(ctypes.byref(g), ctypes.byref(o), in_set.data_ptr(), ctypes.byref(cnt), ctypes.byref(its),
                    st.ctypes.data if st is not None else None, ws.data_ptr(), wsb, _stream())
    launches = int(lib().mis2_last_launch_count())
    _check(rc, "mis2", allow=(ENOTCONVERGED,) if allow_partial else ())
    extra = None
    if timeline:
        # kernel entry -> first phase (init), last phase -> kernel end (output)
        extra = {"init_us": float(st[0] - st[2 * mi]) / 1e3, "final_us": float(st[2 * mi + 1] - st[2 * its.value]) / 1e3}
        st = np.diff(st[: 2 * its.value + 1]) / 1e3  # microseconds per phase
    elif st is not None:
        st = st[: its.value].copy()
    return Mis2Result(in_set[:n], int(cnt.value), int(its.value), rc, st, launches, extra)


def mis2_async(rowptr, colinds, in_set, d_scalars, seed: int = 0, scheme: str = "xorstar", group: int = 0,
               max_iters: int = 0, decide: str = "auto"):
    """Enqueue MIS-2 without synchronising; d_scalars = int64 CUDA tensor [2]
    receiving count and (iterations | status << 32)."""
    g, n, nnz = _graph(rowptr, colinds)
    o = _opts(seed, scheme, max_iters, group, decide=decide)
    ws, wsb = workspace(OP_MIS2, n, nnz)
    p = d_scalars.data_ptr()
    rc = lib().mis2_async(ctypes.byref(g), ctypes.byref(o), in_set.data_ptr(), p, p + 8, p + 12, ws.data_ptr(),
                          wsb, _stream())
    _check(rc, "mis2_async")
    return int(lib().mis2_last_launch_count())


def mis2_host(rowptr_h: np.ndarray, colinds_h: np.ndarray, in_set_h: np.ndarray, seed: int = 0,
              scheme: str = "xorstar", group: int = 0, ws=None):
    """End-to-end MIS-2 from HOST arrays (copies inside the call)."""
    n = rowptr_h.shape[0] - 1
    nnz = colinds_h.shape[0]
    o = _opts(seed, scheme, 0, group)
    if ws is None:
        ws, wsb = workspace(OP_MIS2_HOST, n, nnz)
    else:
        ws, wsb = ws
    cnt, its = ctypes.c_int64(0), ctypes.c_int32(0)

    def hp(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    rc = lib().mis2_host(n, nnz, hp(rowptr_h), hp(colinds_h), ctypes.byref(o), hp(in_set_h), ctypes.byref(cnt),
                         ctypes.byref(its), ws.data_ptr(), wsb, _stream())
    _check(rc, "mis2_host")
    return int(cnt.value), int(its.value)


@dataclass
class AggResult:
    labels: "object"   # torch.int32 CUDA [n]
    num_aggs: int
    roots: "object"    # torch.int32 CUDA [num_aggs]
    stats: dict
    iter_stats: tuple | None = None  # (phase-1 MIS-2, masked phase-2 MIS-2) worklist statistics


def aggregate(rowptr, colinds, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0, group: int = 0,
              validate: bool = False, basic: bool = False, decide: str = "auto", keys: str = "auto",
              word_bits: int = 64, iter_stats: bool = False) -> AggResult:
    """Alg. 3, or Alg. 2 with basic=True,
    through ``mis2_aggregate()``."""
    torch = _torch()
    g, n, nnz = _graph(rowptr, colinds)
    o = _opts(seed, scheme, max_iters, group, validate, decide=decide, keys=keys, word_bits=word_bits)
    if basic:
        o.flags |= FLAG_BASIC
    mi = max_iters if max_iters > 0 else 10 * (n + 1).bit_length() + 20
    if iter_stats:
        o.flags |= FLAG_ITER_STATS
    ws, wsb = workspace(OP_AGGREGATE, n, nnz)
    labels = torch.empty(max(n, 1), dtype=torch.int32, device=rowptr.device)
    roots = torch.empty(max(n, 1), dtype=torch.int32, device=rowptr.device)
    na = ctypes.c_int64(0)
    st = np.zeros(8 + (12 * mi if iter_stats else 0), dtype=np.int64)
    rc = lib().mis2_aggregate(ctypes.byref(g), ctypes.byref(o), labels.data_ptr(), ctypes.byref(na),
                              roots.data_ptr(), st.ctypes.data, ws.data_ptr(), wsb, _stream())
    _check(rc, "mis2_aggregate")
    keys = ["mis1", "iters1", "mis2", "iters2", "accepted2", "leftovers", "n1", "num_aggs"]
    summary = dict(zip(keys, map(int, st[:8])))
    its = None
    if iter_stats:
        a = st[8:8 + 6 * mi].reshape(mi, 6)[: summary["iters1"]].copy()
        b = st[8 + 6 * mi:].reshape(mi, 6)[: summary["iters2"]].copy()
        its = (a, b)
    return AggResult(labels[:n], int(na.value), roots[: na.value], summary, its)


def coarsen(rowptr, colinds, labels, num_aggs: int):
    """Coarse graph through ``mis2_coarsen()`` (two-call)."""
    torch = _torch()
    g, n, nnz = _graph(rowptr, colinds)
    ws, wsb = workspace(OP_COARSEN, n, nnz)
    crow = torch.empty(num_aggs + 1, dtype=torch.int64, device=rowptr.device)
    cnnz = ctypes.c_int64(0)
    L = lib()
    # one call with a capacity guess (coarse graphs are far sparser than the
    # fine one); the two-call convention (MIS2_ERANGE + exact size) otherwise
    cap = max(4096, min(nnz, num_aggs * num_aggs), nnz // 8) if nnz else 1
    ccol = torch.empty(cap, dtype=torch.int32, device=rowptr.device)
    rc = L.mis2_coarsen(ctypes.byref(g), labels.data_ptr(), num_aggs, crow.data_ptr(), ccol.data_ptr(), cap,
                        ctypes.byref(cnnz), ws.data_ptr(), wsb, _stream())
    if rc == ERANGE:
        ccol = torch.empty(max(cnnz.value, 1), dtype=torch.int32, device=rowptr.device)
        rc = L.mis2_coarsen(ctypes.byref(g), labels.data_ptr(), num_aggs, crow.data_ptr(), ccol.data_ptr(),
                            ccol.numel(), ctypes.byref(cnnz), ws.data_ptr(), wsb, _stream())
    _check(rc, "mis2_coarsen")
    return crow, ccol[: cnnz.value]


def validate_graph(rowptr, colinds) -> None:
    g, n, nnz = _graph(rowptr, colinds)
    ws, wsb = workspace(OP_VALIDATE, n, nnz)
    _check(lib().mis2_validate_graph(ctypes.byref(g), ws.data_ptr(), wsb, _stream()), "mis2_validate_graph")


def multilevel(rowptr, colinds, threshold: int = 1000, max_levels: int = 32, seed: int = 0):
    """Repeated aggregation + coarsening until n < threshold or no reduction
    (reading Q22).  Returns [(n, nnz, num_aggs)], final CSR,
    and the per-level label tensors."""
    levels, labels_all = [], []
    rp, ci = rowptr, colinds
    for _ in range(max_levels):
        n = rp.numel() - 1
        if n < threshold:
            break
        agg = aggregate(rp, ci, seed=seed)
        levels.append((n, ci.numel(), agg.num_aggs))
        labels_all.append(agg.labels)
        if agg.num_aggs == n:
            break
        rp, ci = coarsen(rp, ci, agg.labels, agg.num_aggs)
    return levels, (rp, ci), labels_all


# ---------------------------------------------------------------- partitioned
def plan_part(n_global: int, nparts: int, part: int, rowptr_local: np.ndarray, colinds_global: np.ndarray):
    """Host-only partition planner (C ABI ``mis2_plan_part``): returns
    (ghost global ids, requests per owner, colinds in the local index space)."""
    L = lib()
    rowptr_local = np.ascontiguousarray(rowptr_local, dtype=np.int64)
    colinds_global = np.ascontiguousarray(colinds_global, dtype=np.int32)
    ng = ctypes.c_int64(0)
    req = np.zeros(nparts, dtype=np.int64)
    _check(L.mis2_plan_part(n_global, nparts, part, rowptr_local.ctypes.data, colinds_global.ctypes.data,
                            ctypes.byref(ng), None, req.ctypes.data, None), "mis2_plan_part")
    ghosts = np.zeros(max(ng.value, 1), dtype=np.int64)
    nnz = int(rowptr_local[-1] - rowptr_local[0])
    loc = np.zeros(max(nnz, 1), dtype=np.int32)
    _check(L.mis2_plan_part(n_global, nparts, part, rowptr_local.ctypes.data, colinds_global.ctypes.data,
                            ctypes.byref(ng), ghosts.ctypes.data, req.ctypes.data, loc.ctypes.data), "mis2_plan_part")
    return ghosts[: ng.value], req, loc[:nnz]


def comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().mis2_comm_unique_id(buf), "mis2_comm_unique_id")
    return bytes(buf)


class Comm:
    """Partitioned MIS-2 driver (C ABI ``mis2_comm_*`` / ``mis2_dist_mis2``).

    ``Comm.local(P)``: P partitions in this process on the current device.
    ``Comm.nccl(uid, world, rank)``: one partition per process/GPU over NCCL."""

    def __init__(self, handle, local: bool, nparts: int):
        self.h, self.local, self.nparts = handle, local, nparts
        self.n_global = 0

    @classmethod
    def local_parts(cls, nparts: int):
        h = ctypes.c_void_p()
        _check(lib().mis2_comm_init_local(nparts, ctypes.byref(h)), "mis2_comm_init_local")
        return cls(h, True, nparts)

    @classmethod
    def nccl(cls, uid: bytes, world: int, rank: int):
        h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().mis2_comm_init_nccl(buf, world, rank, ctypes.byref(h)), "mis2_comm_init_nccl")
        return cls(h, False, world)

    def set_graph(self, n_global: int, rowptr_h: np.ndarray, colinds_h: np.ndarray):
        rowptr_h = np.ascontiguousarray(rowptr_h, dtype=np.int64)
        colinds_h = np.ascontiguousarray(colinds_h, dtype=np.int32)
        if colinds_h.shape[0] == 0:
            colinds_h = np.zeros(1, dtype=np.int32)
        _check(lib().mis2_comm_set_graph(self.h, n_global, rowptr_h.ctypes.data, colinds_h.ctypes.data, _stream()),
               "mis2_comm_set_graph")
        self.n_global = n_global
        return self

    def part_info(self, part: int = 0):
        lo, hi, ng = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        _check(lib().mis2_comm_part_info(self.h, part, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(ng)),
               "mis2_comm_part_info")
        return lo.value, hi.value, ng.value

    def mis2(self, in_set, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0, group: int = 0,
             word_bits: int = 64):
        o = _opts(seed, scheme, max_iters, group, word_bits=word_bits)
        cnt, its = ctypes.c_int64(0), ctypes.c_int32(0)
        _check(lib().mis2_dist_mis2(self.h, ctypes.byref(o), in_set.data_ptr(), ctypes.byref(cnt), ctypes.byref(its),
                                    _stream()), "mis2_dist_mis2")
        return int(cnt.value), int(its.value)

    def aggregate(self, labels, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0, group: int = 0,
                  word_bits: int = 64):
        """Alg. 3 over the partition (``mis2_dist_aggregate``): fills ``labels``
        (int32 CUDA tensor: this rank's rows, or all rows for local parts)
        with global aggregate ids; returns (num_aggs, stats dict)."""
        o = _opts(seed, scheme, max_iters, group, word_bits=word_bits)
        na = ctypes.c_int64(0)
        st = np.zeros(8, dtype=np.int64)
        _check(lib().mis2_dist_aggregate(self.h, ctypes.byref(o), labels.data_ptr(), ctypes.byref(na),
                                         st.ctypes.data, _stream()), "mis2_dist_aggregate")
        keys = ["mis1", "iters1", "mis2", "iters2", "accepted2", "leftovers", "n1", "num_aggs"]
        return int(na.value), dict(zip(keys, map(int, st)))

    def coarsen(self, labels, num_aggs: int):
        """Coarse graph of the partitioned graph (``mis2_dist_coarsen``),
        replicated on every rank: (crow int64, ccol int32) CUDA tensors."""
        torch = _torch()
        dev = labels.device
        crow = torch.empty(num_aggs + 1, dtype=torch.int64, device=dev)
        cnnz = ctypes.c_int64(0)
        L = lib()
        rc = L.mis2_dist_coarsen(self.h, labels.data_ptr(), num_aggs, crow.data_ptr(), None, 0, ctypes.byref(cnnz),
                                 _stream())
        _check(rc, "mis2_dist_coarsen(count)", allow=(ERANGE,))
        ccol = torch.empty(max(cnnz.value, 1), dtype=torch.int32, device=dev)
        rc = L.mis2_dist_coarsen(self.h, labels.data_ptr(), num_aggs, crow.data_ptr(), ccol.data_ptr(), ccol.numel(),
                                 ctypes.byref(cnnz), _stream())
        _check(rc, "mis2_dist_coarsen")
        return crow, ccol[: cnnz.value]

    def multilevel(self, labels, threshold: int = 1000, max_levels: int = 32, seed: int = 0):
        """Multilevel coarsening of the partitioned graph (NEXT-3): level 0
        aggregated and coarsened over the partition (mis2_dist_aggregate +
        mis2_dist_coarsen), the replicated coarse graph (~1/70 of the fine
        one on the elasticity graphs) continued on this GPU by ``multilevel``.
        ``labels`` receives the level-0 labels.  Returns the same
        (levels, final CSR) as ``multilevel`` on the whole graph."""
        n = self.n_global
        if n < threshold:
            return [], None
        na, _ = self.aggregate(labels, seed=seed)
        levels = [(n, None, na)]
        if na == n or max_levels <= 1:
            return levels, None
        crow, ccol = self.coarsen(labels, na)
        more, fin, _ = multilevel(crow, ccol, threshold=threshold, max_levels=max_levels - 1, seed=seed)
        return levels + more, fin

    def close(self):
        if self.h:
            lib().mis2_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- Alg. 4
def color(rowptr, colinds, seed: int = 0):
    """Deterministic greedy colouring (``mis2_color``, reading Q30): returns
    (int32 CUDA colours, ncolors)."""
    torch = _torch()
    g, n, nnz = _graph(rowptr, colinds)
    out = torch.empty(max(n, 1), dtype=torch.int32, device=rowptr.device)
    nc = ctypes.c_int32(0)
    ws, wsb = workspace(OP_COLOR, n, nnz)
    _check(lib().mis2_color(ctypes.byref(g), seed & ((1 << 64) - 1), out.data_ptr(), ctypes.byref(nc),
                            ws.data_ptr(), wsb, _stream()), "mis2_color")
    return out[:n], int(nc.value)


class ClusterSGS:
    """Alg. 4 cluster multicolor Gauss-Seidel (``mis2_cgs_*``): clusters =
    ``labels`` (e.g. ``aggregate``) coloured on their coarse graph, or
    point multicolor GS when ``labels`` is None.  ``apply`` runs sweeps in
    place on a float64 CUDA vector."""

    DIRS = {"symmetric": 0, "forward": 1, "backward": 2}

    def __init__(self, rowptr, colinds, vals, labels=None, num_aggs: int = 0, coarse=None, seed: int = 0):
        self._keep = (rowptr, colinds, vals, labels, coarse)
        g, n, nnz = _graph(rowptr, colinds)
        self.n = n
        cg = None
        if labels is not None:
            if coarse is None:
                coarse = coarsen(rowptr, colinds, labels, num_aggs)
                self._keep = (rowptr, colinds, vals, labels, coarse)
            cg, _, _ = _graph(*coarse)
        h = ctypes.c_void_p()
        _check(lib().mis2_cgs_setup(ctypes.byref(g), vals.data_ptr(), labels.data_ptr() if labels is not None else None,
                                    num_aggs, ctypes.byref(cg) if cg is not None else None,
                                    seed & ((1 << 64) - 1), ctypes.byref(h), _stream()), "mis2_cgs_setup")
        self.h = h
        self.ncolors = int(lib().mis2_cgs_ncolors(h))

    def apply(self, b, x=None, sweeps: int = 1, direction: str = "symmetric"):
        torch = _torch()
        if x is None:
            x = torch.zeros(max(self.n, 1), dtype=torch.float64, device=b.device)
        _check(lib().mis2_cgs_apply(self.h, b.data_ptr(), x.data_ptr(), sweeps, self.DIRS[direction], _stream()),
               "mis2_cgs_apply")
        return x

    def close(self):
        if getattr(self, "h", None):
            lib().mis2_cgs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
