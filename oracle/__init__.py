"""Serial CPU oracle for the MIS-2 hot path (arXiv 2204.02934) -- TEST
INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA product path (paper_2204_02934_b200/) and neither imports the other; the
only common dependency is the seeded input generator module ``mis2gen``.

The arithmetic lives in oracle.c (plain C, serial, in the paper's order; see
its header for the passage each function follows).  This file only compiles
it, marshals numpy arrays, and adds the multilevel loop of P:26-28 (§I,
"apply coarsening recursively until ... smaller than some threshold").

Pinned by tests/test_oracle_*.py.  The exact
in-set masks/labels at config scale are pinned only through those properties
plus GPU == oracle; no function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, EINVAL, ENOMEM, ENOTCONVERGED, EASSERT, ERANGE = 0, -1, -2, -6, -9, -7
SCHEMES = {"xorstar": 0, "fixed": 1, "xor": 2}
WORD32 = 0x10  # scheme modifier: status words of width 32 (reading Q32)


def _scheme(scheme: str, word_bits: int) -> int:
    if word_bits not in (32, 64):
        raise ValueError(word_bits)
    return SCHEMES[scheme] | (WORD32 if word_bits == 32 else 0)
IN = 0
OUT = (1 << 64) - 1
UNAGG = -1


class OracleError(RuntimeError):
    def __init__(self, rc, msg=""):
        super().__init__(f"oracle rc={rc} {msg}")
        self.rc = rc


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-Wno-unused-variable", "-shared",
                               "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, i64, i32, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        lib.orc_xorshift64.argtypes = [u64]; lib.orc_xorshift64.restype = u64
        lib.orc_xorshift64star.argtypes = [u64]; lib.orc_xorshift64star.restype = u64
        lib.orc_h.argtypes = [ctypes.c_int, u64, u64, u64]; lib.orc_h.restype = u64
        lib.orc_bits.argtypes = [i64]; lib.orc_bits.restype = ctypes.c_int
        lib.orc_pack.argtypes = [u64, i64, ctypes.c_int]; lib.orc_pack.restype = u64
        lib.orc_word.argtypes = [ctypes.c_int, u64, i64, u64, ctypes.c_int]; lib.orc_word.restype = u64
        lib.orc_mis2.argtypes = [i64, p, p, u64, ctypes.c_int, i32, p, p, i32, p, p, p, p, p, p]
        lib.orc_mis2.restype = ctypes.c_int
        lib.orc_aggregate.argtypes = [i64, p, p, u64, ctypes.c_int, i32, p, p, p, p]
        lib.orc_aggregate.restype = ctypes.c_int
        lib.orc_coarsen_basic.argtypes = [i64, p, p, u64, ctypes.c_int, i32, p, p]
        lib.orc_coarsen_basic.restype = ctypes.c_int
        lib.orc_coarsen.argtypes = [i64, p, p, p, i64, p, p, i64, p]
        lib.orc_coarsen.restype = ctypes.c_int
        lib.orc_color_jp.argtypes = [i64, p, p, u64, p, p]
        lib.orc_color_jp.restype = ctypes.c_int
        lib.orc_cluster_sgs.argtypes = [i64, p, p, p, p, i64, p, i32, p, p, ctypes.c_int, ctypes.c_int]
        lib.orc_cluster_sgs.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _csr(rowptr, colinds):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colinds = np.ascontiguousarray(colinds, dtype=np.int32)
    if colinds.shape[0] == 0:
        colinds = np.zeros(1, dtype=np.int32)
    return rowptr, colinds


# --- §V-A / §V-C scalars --------------------------------------------------
def xorshift64(x: int) -> int:
    return int(_load().orc_xorshift64(x))


def xorshift64star(x: int) -> int:
    return int(_load().orc_xorshift64star(x))


def h(it: int, v: int, seed: int = 0, scheme: str = "xorstar") -> int:
    return int(_load().orc_h(SCHEMES[scheme], it, v, seed))


def bits(n: int) -> int:
    return int(_load().orc_bits(n))


def pack(priority: int, vid: int, b: int) -> int:
    return int(_load().orc_pack(priority, vid, b))


def word(it: int, v: int, n: int, seed: int = 0, scheme: str = "xorstar", word_bits: int = 64) -> int:
    return int(_load().orc_word(_scheme(scheme, word_bits), it, v, seed, bits(n)))


# --- Alg. 1 ---------------------------------------------------------------
@dataclass
class Mis2Result:
    in_set: np.ndarray
    count: int
    iterations: int
    rc: int = OK
    stats: np.ndarray | None = None   # [iters, 6]: |wl1| |wl2| E1 E2 |N[wl1]| |N[wl2]|
    T: np.ndarray | None = None
    M: np.ndarray | None = None


def mis2(rowptr, colinds, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0,
         active=None, prio_override=None, stats: bool = False, state: bool = False,
         allow_partial: bool = False, word_bits: int = 64) -> Mis2Result:
    """Alg. 1 on CSR (rowptr int64, colinds int32); word_bits = the
    status-word width W (64, or the paper's 32: reading Q32)."""
    lib = _load()
    rowptr, colinds = _csr(rowptr, colinds)
    n = rowptr.shape[0] - 1
    b = lib.orc_bits(n)
    mi = max_iters if max_iters > 0 else 10 * b + 20
    in_set = np.zeros(max(n, 1), dtype=np.uint8)
    cnt = ctypes.c_int64(0)
    its = ctypes.c_int32(0)
    st = np.zeros((mi, 6), dtype=np.int64) if stats else None
    T = np.zeros(max(n, 1), dtype=np.uint64) if state else None
    M = np.zeros(max(n, 1), dtype=np.uint64) if state else None
    act = None if active is None else np.ascontiguousarray(active, dtype=np.uint8)
    po, pi = None, 0
    if prio_override is not None:
        po = np.ascontiguousarray(prio_override, dtype=np.uint64)
        pi = po.shape[0]
        po = po.reshape(-1)
    rc = lib.orc_mis2(n, _p(rowptr), _p(colinds), seed, _scheme(scheme, word_bits), mi, _p(act), _p(po), pi,
                      _p(in_set), ctypes.byref(cnt), ctypes.byref(its), _p(st), _p(T), _p(M))
    if rc not in (OK, ENOTCONVERGED) or (rc == ENOTCONVERGED and not allow_partial):
        raise OracleError(rc, "mis2")
    return Mis2Result(in_set[:n].astype(bool), int(cnt.value), int(its.value), rc,
                      None if st is None else st[: its.value].copy(),
                      None if T is None else T[:n], None if M is None else M[:n])


# --- Alg. 3 / Alg. 2 ------------------------------------------------------
@dataclass
class AggResult:
    labels: np.ndarray
    num_aggs: int
    roots: np.ndarray
    stats: dict = field(default_factory=dict)


def aggregate(rowptr, colinds, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0,
              word_bits: int = 64) -> AggResult:
    """Alg. 3."""
    lib = _load()
    rowptr, colinds = _csr(rowptr, colinds)
    n = rowptr.shape[0] - 1
    labels = np.zeros(max(n, 1), dtype=np.int32)
    roots = np.zeros(max(n, 1), dtype=np.int32)
    na = ctypes.c_int64(0)
    st = np.zeros(8, dtype=np.int64)
    rc = lib.orc_aggregate(n, _p(rowptr), _p(colinds), seed, _scheme(scheme, word_bits), max_iters, _p(labels),
                           ctypes.byref(na), _p(roots), _p(st))
    if rc != OK:
        raise OracleError(rc, "aggregate")
    keys = ["mis1", "iters1", "mis2", "iters2", "accepted2", "leftovers", "n1", "num_aggs"]
    return AggResult(labels[:n], int(na.value), roots[: na.value].copy(), dict(zip(keys, map(int, st))))


def coarsen_basic(rowptr, colinds, seed: int = 0, scheme: str = "xorstar", max_iters: int = 0):
    """Alg. 2 -> (labels, num_aggs)."""
    lib = _load()
    rowptr, colinds = _csr(rowptr, colinds)
    n = rowptr.shape[0] - 1
    labels = np.zeros(max(n, 1), dtype=np.int32)
    na = ctypes.c_int64(0)
    rc = lib.orc_coarsen_basic(n, _p(rowptr), _p(colinds), seed, SCHEMES[scheme], max_iters,
                               _p(labels), ctypes.byref(na))
    if rc != OK:
        raise OracleError(rc, "coarsen_basic")
    return labels[:n], int(na.value)


def coarsen(rowptr, colinds, labels, num_aggs: int):
    """Coarse graph: returns (c_rowptr int64[na+1], c_colinds int32)."""
    lib = _load()
    rowptr, colinds = _csr(rowptr, colinds)
    n = rowptr.shape[0] - 1
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    crow = np.zeros(num_aggs + 1, dtype=np.int64)
    nnz = ctypes.c_int64(0)
    rc = lib.orc_coarsen(n, _p(rowptr), _p(colinds), _p(labels if n else np.zeros(1, np.int32)),
                         num_aggs, _p(crow), None, 0, ctypes.byref(nnz))
    if rc not in (OK, ERANGE):
        raise OracleError(rc, "coarsen count")
    ccol = np.zeros(max(nnz.value, 1), dtype=np.int32)
    rc = lib.orc_coarsen(n, _p(rowptr), _p(colinds), _p(labels if n else np.zeros(1, np.int32)),
                         num_aggs, _p(crow), _p(ccol), ccol.shape[0], ctypes.byref(nnz))
    if rc != OK:
        raise OracleError(rc, "coarsen")
    return crow, ccol[: nnz.value]


def multilevel(rowptr, colinds, threshold: int = 1000, max_levels: int = 32, seed: int = 0):
    """Repeated Alg. 3 + coarsen until n < threshold or no reduction
    (reading Q22).  Returns the list of (n, nnz, num_aggs)."""
    levels = []
    rp, ci = np.asarray(rowptr, np.int64), np.asarray(colinds, np.int32)
    for _ in range(max_levels):
        n = rp.shape[0] - 1
        if n < threshold:
            break
        agg = aggregate(rp, ci, seed=seed)
        levels.append((n, int(rp[-1]), agg.num_aggs))
        if agg.num_aggs == n:
            break
        rp, ci = coarsen(rp, ci, agg.labels, agg.num_aggs)
    return levels, (rp, ci)


# --- Alg. 4 -----------------------------------------------------
def color_jp(rowptr, colinds, seed: int = 0):
    """Deterministic greedy colouring (reading Q30): (colour int32[n], ncolors)."""
    lib = _load()
    rowptr, colinds = _csr(rowptr, colinds)
    n = rowptr.shape[0] - 1
    color = np.zeros(max(n, 1), dtype=np.int32)
    nc = ctypes.c_int32(0)
    rc = lib.orc_color_jp(n, _p(rowptr), _p(colinds), seed & ((1 << 64) - 1), _p(color), ctypes.byref(nc))
    if rc != OK:
        raise OracleError(rc, "color_jp")
    return color[:n], int(nc.value)


def cluster_sgs(rowptr, colinds, vals, labels, num_aggs, ccolor, ncolors, b, x0=None, sweeps: int = 1,
                direction: str = "symmetric"):
    """Alg. 4 apply / SGS (reading Q31) in fp64 from x0
    (default 0): returns x."""
    lib = _load()
    rowptr, colinds = _csr(rowptr, colinds)
    n = rowptr.shape[0] - 1
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    if vals.shape[0] == 0:
        vals = np.zeros(1)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    ccolor = np.ascontiguousarray(ccolor, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(max(n, 1)) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    d = {"symmetric": 0, "forward": 1, "backward": 2}[direction]
    rc = lib.orc_cluster_sgs(n, _p(rowptr), _p(colinds), _p(vals), _p(labels if n else np.zeros(1, np.int32)),
                             num_aggs, _p(ccolor if len(ccolor) else np.zeros(1, np.int32)), ncolors, _p(b), _p(x),
                             sweeps, d)
    if rc != OK:
        raise OracleError(rc, "cluster_sgs")
    return x[:n]


def cgs_setup(rowptr, colinds, seed: int = 0, point: bool = False):
    """Alg. 4 setup: clusters = Alg. 3 aggregates (or single rows when
    point=True, point multicolor GS), coloured on the coarse graph.
    Returns (labels, num_aggs, ccolor, ncolors)."""
    n = len(rowptr) - 1
    if point:
        labels, na = np.arange(n, dtype=np.int32), n
    else:
        a = aggregate(rowptr, colinds, seed=seed)
        labels, na = a.labels, a.num_aggs
    crow, ccol = coarsen(rowptr, colinds, labels, na)
    ccolor, nc = color_jp(crow, ccol, seed=seed)
    return labels, na, ccolor, nc
