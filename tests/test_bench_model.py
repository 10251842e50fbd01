"""The bench's algorithmic-byte model (the roofline numerator) on the headline
workload, from the CPU oracle only: the per-iteration worklist statistics of
C2 (27-point 100^3) equal SURVEY.md §8(a)'s table (an independent scratch
model of the same readings), and bench.survey_bytes turns them into the
§8(d).3 per-iteration column / Decide bytes that table lists and the 0.990 GB
per call the roofline divides by."""
import os
import sys

import numpy as np

import mis2gen as G
import oracle as O

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

# SURVEY.md §8(a) "[scratch] per-iteration profile, C2": |wl1| |wl2| E1 E2,
# column MB, decide MB
SURVEY_C2 = [
    (1000000, 1000000, 26463592, 26463592, 137.9, 145.8),
    (991562, 1000000, 26242803, 26463592, 137.0, 141.8),
    (266531, 779211, 7001919, 20614595, 108.5, 41.7),
    (158664, 642315, 4162204, 17027967, 90.6, 26.0),
    (55073, 478192, 1440329, 12694987, 68.9, 10.1),
    (22621, 283901, 592757, 7550924, 42.3, 4.6),
    (6070, 143516, 159783, 3825474, 22.3, 1.4),
    (1485, 51009, 39105, 1363296, 8.2, 0.4),
    (150, 13017, 3915, 348111, 2.2, 0.0),
    (12, 1576, 306, 42147, 0.3, 0.0),
]


def test_c2_worklist_statistics_and_bytes():
    g = G.laplace3d_27pt(100)
    o = O.mis2(g.rowptr, g.colinds, stats=True)
    st = o.stats
    assert (o.count, o.iterations) == (21587, 10)
    assert st.shape[0] == len(SURVEY_C2)
    for i, (w1, w2, e1, e2, col_mb, dec_mb) in enumerate(SURVEY_C2):
        assert tuple(int(x) for x in st[i, :4]) == (w1, w2, e1, e2), i
        w1n = int(st[i + 1, 0]) if i + 1 < st.shape[0] else 0
        w2n = int(st[i + 1, 1]) if i + 1 < st.shape[0] else 0
        col = 4 * e2 + 8 * int(st[i, 5]) + 20 * w2 + 4 * w2n
        dec = 4 * e1 + 8 * int(st[i, 4]) + 28 * w1 + 4 * w1n
        assert abs(col / 1e6 - col_mb) <= 0.051 and abs(dec / 1e6 - dec_mb) <= 0.051, (i, col, dec)
    total = bench.survey_bytes(st)
    assert abs(total / 1e9 - 0.990) < 0.0005, total  # 0.990 GB per call
    # the roofline at the measured HBM copy bandwidth: 50% <=> <= 0.303 ms per call
    assert 0.300 < total / (0.5 * 6538e9) * 1e3 < 0.305
