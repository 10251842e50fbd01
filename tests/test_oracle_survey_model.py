"""Agreement of the oracle with an INDEPENDENT implementation of the same
readings: the Python model recorded in SURVEY.md §8(c).5 (values are that
model's, not the paper's; the paper cannot fix them because its hash
constants are unpublished)."""
import numpy as np

import mis2gen as G
import oracle as O

C1_MIS = [0, 4, 9, 12, 16, 30, 33, 37, 45, 49, 52, 60, 67, 75, 89, 91, 94, 97]
C1_PHASE2 = [7, 18, 21, 25, 41, 54, 56, 58, 69, 71, 78, 80, 83, 86]
C1_LABELS = """
 0  0  3  1  1  1  4  4  2  2
 0  3  3  3  1  4  4  4  2  2
 5  5  3  6  6  4  4  7  7  2
 5  5  6  6  6  8  7  7  7  9
 5  5 10  6  8  8  8  7  9  9
11 10 10 10  8  8  8 12  9  9
11 11 10 10 13 13 12 12 12  9
11 11 18 18 13 13 13 12 14 14
15 15 18 18 16 13 17 17 14 14
15 15 15 16 16 16 17 17 17 14"""


def test_c1_full_golden():
    g = G.grid2d_5pt(10, 10)
    r = O.mis2(g.rowptr, g.colinds)
    assert np.nonzero(r.in_set)[0].tolist() == C1_MIS and r.iterations == 5
    a = O.aggregate(g.rowptr, g.colinds)
    assert a.labels.tolist() == [int(x) for x in C1_LABELS.split()]
    assert a.num_aggs == 19 and a.stats["iters2"] == 4 and a.stats["mis2"] == 14
    labels = np.array(a.labels)
    unagg1 = np.ones(100, bool)
    for v in C1_MIS:
        unagg1[v] = False
        unagg1[g.colinds[g.rowptr[v]:g.rowptr[v + 1]]] = False
    p2 = O.mis2(g.rowptr, g.colinds, active=unagg1)
    assert np.nonzero(p2.in_set)[0].tolist() == C1_PHASE2
    crow, ccol = O.coarsen(g.rowptr, g.colinds, labels, 19)
    assert len(ccol) == 84


def test_c2_profile():
    g = G.laplace3d_27pt(100)
    r = O.mis2(g.rowptr, g.colinds, stats=True)
    assert (r.count, r.iterations) == (21587, 10)
    assert r.stats[:, 0].tolist() == [1000000, 991562, 266531, 158664, 55073, 22621, 6070, 1485, 150, 12]
    assert r.stats[:, 3].tolist()[:3] == [26463592, 26463592, 20614595]
    a = O.aggregate(g.rowptr, g.colinds)
    assert a.num_aggs == 42261 and a.stats["accepted2"] == 20674 and a.stats["leftovers"] == 162369
