"""Seeded synthetic graph generators shared by the oracle tests, the CUDA
parity tests and bench.py.

This module holds none of the method's arithmetic (no priorities, no status
words, no reductions): it only produces CSR graphs (rowptr int64[n+1], colinds
int32[nnz], rows sorted, symmetric, duplicate free) shaped like the paper's
workloads (§VI "Laplace3D_100 ... 7-point stencil",
"Elasticity3D_60 ... 27-point stencil and 3 degrees of freedom") and the
BASELINE.json configs.  The heavy generators are C (gen.c, OpenMP); small
random graphs for property tests are numpy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libmis2gen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into libmis2gen.so (gcc -O3 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, i32, u64, p = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p
        lib.gen_stencil_nnz.argtypes = [i64, i64, i64, i32, i32]
        lib.gen_stencil_nnz.restype = i64
        lib.gen_stencil.argtypes = [i64, i64, i64, i32, i32, p, p]
        lib.gen_stencil.restype = i64
        lib.gen_kronecker.argtypes = [i32, i32, u64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, p, p, p, p]
        lib.gen_kronecker.restype = i64
        lib.gen_checksum.argtypes = [i64, p, p]
        lib.gen_checksum.restype = u64
        lib.gen_num_threads.restype = i32
        _lib = lib
    return _lib


@dataclass
class Graph:
    """Host CSR graph: rowptr int64[n+1], colinds int32[nnz]."""
    rowptr: np.ndarray
    colinds: np.ndarray
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.rowptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def checksum(self) -> int:
        return int(_load().gen_checksum(self.n, self.rowptr.ctypes.data, self.colinds.ctypes.data))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def stencil(nx: int, ny: int, nz: int = 1, points: int = 7, dof: int = 1, name: str = "") -> Graph:
    """Laplacian-pattern graph with diagonal: points=7 (5-pt when nz == 1) or 27.

    dof > 1 gives the Elasticity3D pattern (stencil (x) dense dof x dof block)."""
    lib = _load()
    nnz = lib.gen_stencil_nnz(nx, ny, nz, points, dof)
    if nnz < 0:
        raise ValueError("bad stencil arguments")
    n = nx * ny * nz * dof
    rowptr = np.empty(n + 1, dtype=np.int64)
    colinds = np.empty(max(nnz, 1), dtype=np.int32)[:nnz]
    got = lib.gen_stencil(nx, ny, nz, points, dof, _ptr(rowptr), _ptr(colinds) if nnz else None)
    assert got == nnz
    return Graph(rowptr, colinds, name or f"{points}pt_{nx}x{ny}x{nz}" + (f"_dof{dof}" if dof > 1 else ""))


def grid2d_5pt(nx: int, ny: int) -> Graph:
    return stencil(nx, ny, 1, 7, 1, name=f"5pt_{nx}x{ny}")


def laplace3d_7pt(nx: int, ny: int | None = None, nz: int | None = None) -> Graph:
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    return stencil(nx, ny, nz, 7, 1, name=f"7pt_{nx}x{ny}x{nz}")


def laplace3d_27pt(nx: int, ny: int | None = None, nz: int | None = None) -> Graph:
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    return stencil(nx, ny, nz, 27, 1, name=f"27pt_{nx}x{ny}x{nz}")


def elasticity3d(nx: int, ny: int | None = None, nz: int | None = None, dof: int = 3) -> Graph:
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    return stencil(nx, ny, nz, 27, dof, name=f"elast{dof}_{nx}x{ny}x{nz}")


def kronecker(scale: int, edgefactor: int = 16, seed: int = 1,
              A: float = 0.57, B: float = 0.19, C: float = 0.19) -> Graph:
    """Graph500-style Kronecker graph (reading Q27): symmetric, no self-loops,
    no duplicates, no diagonal; labels permuted by a seeded shuffle."""
    lib = _load()
    n = 1 << scale
    m = edgefactor * n
    rowptr = np.empty(n + 1, dtype=np.int64)
    colbuf = np.empty(2 * m, dtype=np.int32)
    eu = np.empty(m, dtype=np.int32)
    ev = np.empty(m, dtype=np.int32)
    nnz = lib.gen_kronecker(scale, edgefactor, seed, A, B, C, _ptr(rowptr), _ptr(colbuf), _ptr(eu), _ptr(ev))
    if nnz < 0:
        raise RuntimeError("gen_kronecker failed")
    del eu, ev
    colinds = colbuf[:nnz].copy() if nnz < colbuf.shape[0] // 2 else colbuf[:nnz]
    return Graph(rowptr, colinds, f"kron_s{scale}_ef{edgefactor}")


def from_edges(n: int, edges, diagonal: bool = False, name: str = "") -> Graph:
    """CSR from an undirected edge list (symmetrised, deduplicated, sorted)."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
    e = e[e[:, 0] != e[:, 1]]
    both = np.concatenate([e, e[:, ::-1]], axis=0)
    if diagonal:
        d = np.arange(n, dtype=np.int64)
        both = np.concatenate([both, np.stack([d, d], axis=1)], axis=0)
    if both.shape[0]:
        key = np.unique(both[:, 0] * n + both[:, 1])
        rows, cols = key // n, key % n
    else:
        rows = cols = np.zeros(0, dtype=np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int64)
    return Graph(rowptr, cols.astype(np.int32), name)


def random_graph(n: int, density: float, seed: int, diagonal: bool = False) -> Graph:
    """Erdos-Renyi G(n, p) (numpy Generator(seed)); symmetric, sorted rows."""
    rng = np.random.default_rng(seed)
    if n < 2:
        return from_edges(n, [], diagonal, f"er_{n}_{density}_{seed}")
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.shape[0]) < density
    return from_edges(n, np.stack([iu[keep], ju[keep]], axis=1), diagonal, f"er_{n}_{density}_{seed}")


def random_powerlaw_graph(n: int, avg_deg: float, seed: int, gamma: float = 2.1) -> Graph:
    """Chung-Lu style skewed-degree graph for small parity cases (numpy)."""
    rng = np.random.default_rng(seed)
    w = (np.arange(1, n + 1, dtype=np.float64)) ** (-1.0 / (gamma - 1.0))
    w *= avg_deg * n / w.sum()
    m = int(avg_deg * n / 2)
    p = w / w.sum()
    u = rng.choice(n, size=m, p=p)
    v = rng.choice(n, size=m, p=p)
    perm = rng.permutation(n)
    return from_edges(n, np.stack([perm[u], perm[v]], axis=1), False, f"pl_{n}_{avg_deg}_{seed}")


def fig1_graph() -> Graph:
    """The 6-vertex graph of PAPER.md fig:example (edges 1-2, 2-3,
    3-4, 4-6, 5-4 in the figure's 1-based ids; here 0-based, reading Q14)."""
    return from_edges(6, [(0, 1), (1, 2), (2, 3), (3, 5), (4, 3)], False, "fig1")


def strip_diagonal(g: Graph) -> Graph:
    n = g.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.rowptr))
    keep = g.colinds.astype(np.int64) != rows
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, rows[keep] + 1, 1)
    return Graph(np.cumsum(rowptr).astype(np.int64), g.colinds[keep].copy(), g.name + "_nodiag")


def add_diagonal(g: Graph) -> Graph:
    n = g.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.rowptr))
    e = np.stack([rows, g.colinds.astype(np.int64)], axis=1)
    return from_edges(n, e, True, g.name + "_diag")


# BASELINE.json configs (index 0..4) -- the concrete synthetic inputs
# (DESIGN.md "Input recipe").
def config_graph(i: int) -> Graph:
    if i == 0:
        return grid2d_5pt(10, 10)
    if i == 1:
        return laplace3d_27pt(100)
    if i == 2:
        return laplace3d_7pt(300)
    if i == 3:
        return kronecker(24, 16, seed=1)
    if i == 4:
        return elasticity3d(150)
    raise ValueError(i)


def num_threads() -> int:
    return int(_load().gen_num_threads())


def spd_values(g: Graph, seed: int = 0):
    """Seeded symmetric, strictly diagonally dominant (hence SPD) values on
    the pattern of g, diagonal inserted where missing: the synthetic matrices
    of the Alg. 4 (cluster Gauss-Seidel) tests and bench.  Off-diagonal
    a_ij = a_ji = -(0.5 + 0.5 u(min(i,j), max(i,j))), u a splitmix64 hash in
    [0, 1); a_ii = 1 + sum_j |a_ij|.  Returns (Graph with diagonal, vals f64).
    Input generation only (no method arithmetic)."""
    gd = add_diagonal(g)
    n = gd.n
    rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(gd.rowptr).astype(np.int64))
    cols = gd.colinds.astype(np.uint64)
    lo, hi = np.minimum(rows, cols), np.maximum(rows, cols)
    with np.errstate(over="ignore"):
        z = lo * np.uint64(0x9E3779B97F4A7C15) + hi + np.uint64(seed & ((1 << 64) - 1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) / float(1 << 53)
    vals = -(0.5 + 0.5 * u)
    diag = rows == cols
    vals[diag] = 0.0
    rowsum = np.zeros(n)
    np.add.at(rowsum, rows.astype(np.int64), np.abs(vals))
    vals[diag] = 1.0 + rowsum[rows[diag].astype(np.int64)]
    return gd, vals
