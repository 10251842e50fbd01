"""Independent checks that pin the oracle to something other than itself.

Nothing here imports oracle/ or the CUDA package.  Each helper is a different
formulation of what the paper fixes (PAPER.md = P:n):

* ``py_f`` / ``py_word``: Python big-int restatement of reading Q3-Q5, used
  only as a cross-implementation vector check of the hash (P6) and to feed the
  Luby formulation below.
* ``is_d2_independent`` / ``is_d2_maximal``: BFS brute force of the MIS-2
  definition (§I "no path u<->v of length <= k"; "no additional vertex
  ... can be added").
* ``luby_g2``: Luby's Monte Carlo Algorithm A (distance-1) on the explicit
  square graph G^2 with self-loops (Lemma 1/2), using the same
  priorities per iteration -- P:381 "Luby's algorithm run on G^2 will terminate
  in the same number of iterations as Algorithm 1 run on G".
* ``bell_sweep``: worklist-free vectorised sweep (every vertex every
  iteration, as in Bell et al.), with numpy minimum.reduceat.
* ``check_aggregation``: the Alg. 3 invariants.
* ``coarse_ptap``: pattern(P^T A P) - diag with scipy.sparse.
"""
from __future__ import annotations

from collections import deque

import numpy as np
import scipy.sparse as sp

MASK64 = (1 << 64) - 1
IN, OUT = 0, MASK64


def py_xorshift(x: int) -> int:
    x &= MASK64
    x ^= (x << 13) & MASK64
    x ^= x >> 7
    x ^= (x << 17) & MASK64
    return x


def py_f(x: int) -> int:
    return (py_xorshift(x) * 0x2545F4914F6CDD1D) & MASK64


def py_bits(n: int) -> int:
    return (n + 1).bit_length()


def py_word(it: int, v: int, n: int, seed: int = 0, word_bits: int = 64) -> int:
    """Eq. 1 with word width W = word_bits: the priority field is the
    top W - b bits of the W-bit hash, and a W = 32 hash is the high half of
    the 64-bit one (readings Q5, Q32)."""
    b = py_bits(n)
    h = py_f(py_f(it ^ seed) ^ py_f(v)) >> (64 - word_bits)
    return (h >> b << b) | (v + 1)


def adjacency_sets(rowptr, colinds):
    n = len(rowptr) - 1
    return [set(int(c) for c in colinds[rowptr[v]:rowptr[v + 1]]) - {v} for v in range(n)]


def within2(adj, v):
    """Vertices at distance 1 or 2 from v (excluding v)."""
    seen = {v}
    out = set()
    dq = deque([(v, 0)])
    while dq:
        u, d = dq.popleft()
        if d == 2:
            continue
        for w in adj[u]:
            if w not in seen:
                seen.add(w)
                out.add(w)
                dq.append((w, d + 1))
    return out


def is_d2_independent(rowptr, colinds, in_set) -> bool:
    adj = adjacency_sets(rowptr, colinds)
    S = set(np.nonzero(np.asarray(in_set))[0].tolist())
    return all(not (within2(adj, v) & S) for v in S)


def is_d2_maximal(rowptr, colinds, in_set) -> bool:
    adj = adjacency_sets(rowptr, colinds)
    S = set(np.nonzero(np.asarray(in_set))[0].tolist())
    n = len(rowptr) - 1
    return all(v in S or (within2(adj, v) & S) for v in range(n))


def square_pattern(rowptr, colinds):
    """Pattern of (A + I)^2 as a CSR bool matrix (Lemma 1 with self-loops)."""
    n = len(rowptr) - 1
    A = sp.csr_matrix((np.ones(len(colinds), dtype=np.int64), np.asarray(colinds), np.asarray(rowptr)),
                      shape=(n, n))
    A = ((A + sp.identity(n, dtype=np.int64, format="csr")) > 0).astype(np.int64)
    return ((A @ A) > 0).tocsr()


def luby_g2(rowptr, colinds, seed=0, active=None, prio=None, max_iters=500, word_bits=64):
    """Luby (distance-1) on explicit G^2 (closed), priorities word(k, v).

    Iteration k, U = undecided at its start:
      OUT_k = {v in U : an IN vertex (decided before k) is a G^2-neighbour}
      IN_k  = {v in U - OUT_k : word(k,v) < word(k,u) for all u in N_G2(v) & U}
    Returns (in_set bool array, iterations)."""
    n = len(rowptr) - 1
    if n == 0:
        return np.zeros(0, dtype=bool), 0
    S2 = square_pattern(rowptr, colinds)
    act = np.ones(n, dtype=bool) if active is None else np.asarray(active, dtype=bool)
    if active is not None:  # induced subgraph: restrict G before squaring
        rp, ci = induced(rowptr, colinds, act)
        S2 = square_pattern(rp, ci)
    status = np.where(act, 1, 2)  # 1 undecided, 0 IN, 2 OUT (inactive = OUT, never seen)
    it = 0
    while (status == 1).any():
        assert it < max_iters
        U = np.nonzero(status == 1)[0]
        if prio is not None and it < len(prio):
            w = {int(v): (int(prio[it][v]) << py_bits(n)) | (int(v) + 1) for v in U}
        else:
            w = {int(v): py_word(it, int(v), n, seed, word_bits) for v in U}
        new_status = status.copy()
        for v in U:
            nb = S2.indices[S2.indptr[v]:S2.indptr[v + 1]]
            nb = nb[act[nb]]
            if (status[nb] == 0).any():
                new_status[v] = 2
                continue
            if all(w[v] <= w[int(u)] for u in nb if status[u] == 1):
                new_status[v] = 0
        status = new_status
        it += 1
    return status == 0, it


def induced(rowptr, colinds, mask):
    """Induced subgraph on mask, KEEPING the original ids (inactive rows empty)."""
    n = len(rowptr) - 1
    mask = np.asarray(mask, dtype=bool)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    keep = mask[rows] & mask[np.asarray(colinds)]
    cnt = np.bincount(rows[keep], minlength=n)
    rp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return rp, np.asarray(colinds)[keep].astype(np.int32)


def bell_sweep(rowptr, colinds, seed=0, active=None, max_iters=500):
    """Worklist-free Alg. 1 (every vertex every iteration), vectorised.

    Column: M_v = min over N[v] of T for every active v (IN -> OUT) -- but a
    vertex that once had M = OUT keeps it, which is exactly what
    recomputing gives, since IN persists.  Decide: every undecided v."""
    n = len(rowptr) - 1
    if n == 0:
        return np.zeros(0, dtype=bool), 0
    act = np.ones(n, dtype=bool) if active is None else np.asarray(active, dtype=bool)
    rp, ci = induced(rowptr, colinds, act)
    # closed neighbourhoods: add v to every row
    rows = np.repeat(np.arange(n), np.diff(rp))
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([ci.astype(np.int64), np.arange(n)])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    starts = np.searchsorted(rows, np.arange(n))
    b = py_bits(n)
    f_v = np.array([py_f(v) for v in range(n)], dtype=np.uint64)
    T = np.full(n, np.uint64(OUT), dtype=np.uint64)
    undecided = act.copy()
    M = np.full(n, np.uint64(OUT), dtype=np.uint64)
    it = 0
    mask_hi = np.uint64(~((1 << b) - 1) & MASK64)
    while undecided.any():
        assert it < max_iters
        fi = np.uint64(py_f(it ^ seed))
        with np.errstate(over="ignore"):
            x = f_v ^ fi
            x ^= x << np.uint64(13)
            x ^= x >> np.uint64(7)
            x ^= x << np.uint64(17)
            hv = x * np.uint64(0x2545F4914F6CDD1D)
        words = (hv & mask_hi) | (np.arange(n, dtype=np.uint64) + np.uint64(1))
        T = np.where(undecided, words, T)
        M = np.minimum.reduceat(T[cols], starts)
        M = np.where(M == np.uint64(IN), np.uint64(OUT), M)
        M = np.where(act, M, np.uint64(OUT))
        any_out = np.maximum.reduceat((M[cols] == np.uint64(OUT)).astype(np.int8), starts) > 0
        all_eq = np.minimum.reduceat((M[cols] == T[rows]).astype(np.int8), starts) > 0
        newT = T.copy()
        newT[undecided & any_out] = np.uint64(OUT)
        newT[undecided & ~any_out & all_eq] = np.uint64(IN)
        T = newT
        undecided = act & (T != np.uint64(IN)) & (T != np.uint64(OUT))
        it += 1
    return (T == np.uint64(IN)) & act, it


def check_aggregation(rowptr, colinds, labels, num_aggs, roots, mis1=None):
    """Alg. 3 invariants.  Returns a list of violated properties (empty = ok)."""
    bad = []
    n = len(rowptr) - 1
    labels = np.asarray(labels)
    if n == 0:
        return bad
    if labels.min() < 0 or labels.max() >= num_aggs:
        bad.append("label range")
        return bad
    if len(np.unique(labels)) != num_aggs:
        bad.append("empty aggregate")
    adj = adjacency_sets(rowptr, colinds)
    roots = np.asarray(roots)
    if len(roots) != num_aggs or (labels[roots] != np.arange(num_aggs)).any():
        bad.append("root label")
    # every aggregate connected (BFS inside the aggregate from its root)
    for a in range(num_aggs):
        members = set(np.nonzero(labels == a)[0].tolist())
        seen = {int(roots[a])}
        dq = deque([int(roots[a])])
        while dq:
            u = dq.popleft()
            for w in adj[u]:
                if w in members and w not in seen:
                    seen.add(w)
                    dq.append(w)
        if seen != members:
            bad.append(f"aggregate {a} disconnected")
            break
    if mis1 is not None:
        r1 = np.nonzero(mis1)[0]
        if not np.array_equal(np.sort(roots[: len(r1)]), r1):
            bad.append("phase-1 roots != MIS-2")
        for k, r in enumerate(r1):
            for w in adj[r]:
                if labels[w] != labels[r]:
                    bad.append("root neighbour not in root aggregate")
                    break
    return bad


def coarse_ptap(rowptr, colinds, labels, num_aggs):
    """pattern(P^T A P) minus the diagonal, P the 0/1 aggregate matrix."""
    n = len(rowptr) - 1
    A = sp.csr_matrix((np.ones(len(colinds), dtype=np.int64), np.asarray(colinds), np.asarray(rowptr)),
                      shape=(n, n))
    P = sp.csr_matrix((np.ones(n, dtype=np.int64), (np.arange(n), np.asarray(labels))), shape=(n, num_aggs))
    C = (P.T @ A @ P).tocsr()
    C.setdiag(0)
    C.eliminate_zeros()
    C.sort_indices()
    C = (C > 0).tocsr()
    C.sort_indices()
    return C.indptr.astype(np.int64), C.indices.astype(np.int32)


def np_words(it: int, gids: np.ndarray, n: int, seed: int = 0) -> np.ndarray:
    """Vectorised word(it, v) for global ids (same reading Q3-Q5 as py_word)."""
    b = py_bits(n)
    mask_hi = np.uint64(~((1 << b) - 1) & MASK64)
    g = np.asarray(gids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = g.copy()
        x ^= x << np.uint64(13)
        x ^= x >> np.uint64(7)
        x ^= x << np.uint64(17)
        fv = x * np.uint64(0x2545F4914F6CDD1D)
        y = fv ^ np.uint64(py_f(it ^ seed))
        y ^= y << np.uint64(13)
        y ^= y >> np.uint64(7)
        y ^= y << np.uint64(17)
        h = y * np.uint64(0x2545F4914F6CDD1D)
    return (h & mask_hi) | (g + np.uint64(1))
