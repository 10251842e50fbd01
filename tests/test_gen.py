"""Input generators (mis2gen): closed-form sizes and CSR well-formedness."""
import numpy as np
import pytest

import mis2gen as G


def _wellformed(g, diag):
    n = g.n
    assert g.rowptr[0] == 0 and (np.diff(g.rowptr) >= 0).all()
    assert g.colinds.dtype == np.int32 and g.rowptr.dtype == np.int64
    rows = np.repeat(np.arange(n), np.diff(g.rowptr))
    c = g.colinds.astype(np.int64)
    assert ((c >= 0) & (c < n)).all()
    key = rows * n + c
    assert (np.diff(key) > 0).all()  # sorted rows, no duplicates
    rev = np.sort(c * n + rows)
    assert np.array_equal(np.sort(key), rev)  # symmetric
    assert ((c == rows).sum() == n) if diag else ((c == rows).sum() == 0)


def test_closed_form_sizes():
    # 7-pt nx^3: n + 2*3*n^2*(n-1) (SPEC graph-core invariant); Laplace3D_100
    # |E| = 6.94M incl. diagonal (P:491 tab:matrices-times)
    assert G.laplace3d_7pt(100).nnz == 10**6 + 6 * 100 * 100 * 99 == 6_940_000
    assert G.laplace3d_27pt(100).nnz == 298**3 == 26_463_592
    g = G.elasticity3d(60)  # Elasticity3D_60: |V| 648,000, |E| 50,757,768, max deg 81
    assert g.n == 648_000 and g.nnz == 50_757_768 and np.diff(g.rowptr).max() == 81
    assert G.grid2d_5pt(10, 10).nnz == 460


@pytest.mark.parametrize("mk,diag", [
    (lambda: G.grid2d_5pt(10, 10), True), (lambda: G.laplace3d_7pt(7, 5, 3), True),
    (lambda: G.laplace3d_27pt(6, 4, 5), True), (lambda: G.elasticity3d(4, 3, 2), True),
    (lambda: G.kronecker(12), False), (lambda: G.random_graph(100, 0.1, 1), False),
    (lambda: G.random_powerlaw_graph(500, 6, 2), False), (lambda: G.fig1_graph(), False)])
def test_wellformed(mk, diag):
    _wellformed(mk(), diag)


def test_grid_ids_lexicographic():
    g = G.grid2d_5pt(10, 10)  # vertex id = 10*y + x (reading Q26)
    assert g.colinds[g.rowptr[11]:g.rowptr[12]].tolist() == [1, 10, 11, 12, 21]


def test_kronecker_shape_deterministic():
    a, b = G.kronecker(14, seed=1), G.kronecker(14, seed=1)
    assert np.array_equal(a.rowptr, b.rowptr) and np.array_equal(a.colinds, b.colinds)
    deg = np.diff(a.rowptr)
    assert 0.2 < (deg == 0).mean() < 0.4  # many isolated vertices (skew)
    assert deg.max() > 50 * deg.mean()
    assert G.kronecker(14, seed=2).checksum() != a.checksum()
