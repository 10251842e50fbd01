"""Measurement aid: the workload compute-sanitizer runs (memcheck / racecheck /
synccheck / initcheck): MIS-2 (both Decide forms, keys on/off), aggregation
(Alg. 3 and Alg. 2), the coarse graph, multilevel, the partitioned driver
(local transport, 3 parts), colouring and one cluster Gauss-Seidel sweep, on
configs[0] (2-D 5-pt 10x10) and a 7-pt 30^3 graph.  Results are checked
against the oracle so a sanitizer run also proves the path it watched ran."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mis2gen as G
import oracle as O
import paper_2204_02934_b200 as m

for g in [G.config_graph(0), G.laplace3d_7pt(30)]:
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colinds).cuda()
    o = O.mis2(g.rowptr, g.colinds)
    for decide in ("pull", "push"):
        for keys in ("off", "on"):
            r = m.mis2(rp, ci, decide=decide, keys=keys)
            assert r.count == o.count and np.array_equal(r.in_set.cpu().numpy().astype(bool), o.in_set)
    oa = O.aggregate(g.rowptr, g.colinds)
    a = m.aggregate(rp, ci)
    assert a.num_aggs == oa.num_aggs and np.array_equal(a.labels.cpu().numpy(), oa.labels)
    m.aggregate(rp, ci, basic=True)
    crow, ccol = m.coarsen(rp, ci, a.labels, a.num_aggs)
    orow, ocol = O.coarsen(g.rowptr, g.colinds, oa.labels, oa.num_aggs)
    assert np.array_equal(ccol.cpu().numpy(), ocol)
    m.multilevel(rp, ci, threshold=50)
    m.validate_graph(rp, ci)
    c = m.Comm.local_parts(3).set_graph(g.n, g.rowptr, g.colinds)
    out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    cnt, its = c.mis2(out)
    assert cnt == o.count
    lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
    na, _ = c.aggregate(lab)
    assert na == oa.num_aggs
    c.coarsen(lab, na)
    c.close()
    m.color(rp, ci)
    gv, vals = G.spd_values(g, seed=1)
    rpv, civ = torch.from_numpy(gv.rowptr).cuda(), torch.from_numpy(gv.colinds).cuda()
    av = m.aggregate(rpv, civ)
    cg = m.ClusterSGS(rpv, civ, torch.from_numpy(vals).cuda(), labels=av.labels, num_aggs=av.num_aggs)
    cg.apply(torch.ones(gv.n, dtype=torch.float64, device="cuda"), sweeps=1)
    cg.close()
torch.cuda.synchronize()
print("sanitize workload ok")
