"""Measurement aid: Alg. 4 setup and symmetric-sweep time on a config
(point and MIS-2-aggregate clusters), CUDA events, inputs resident.
usage: python tools/cgs_probe.py CFG"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g, vals = G.spd_values(G.config_graph(cfg), seed=1)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda(); vd = torch.from_numpy(vals).cuda()
b = torch.ones(g.n, dtype=torch.float64, device="cuda")


def ev(fn, reps=3):
    ts = []
    r = None
    for k in range(reps):
        if r is not None and hasattr(r, "close"):
            r.close()  # release the previous handle outside the timed region
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); r = fn(); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
    return min(ts), r


for kind in ("point", "cluster"):
    extra = {}
    if kind == "point":
        ms_setup, cg = ev(lambda: m.ClusterSGS(rp, ci, vd))
    else:
        def setup():
            a = m.aggregate(rp, ci)
            return m.ClusterSGS(rp, ci, vd, labels=a.labels, num_aggs=a.num_aggs)
        ms_setup, cg = ev(setup)
        a = m.aggregate(rp, ci)
        co = m.coarsen(rp, ci, a.labels, a.num_aggs)
        extra["agg_ms"], _ = ev(lambda: m.aggregate(rp, ci))
        extra["coarsen_ms"], _ = ev(lambda: m.coarsen(rp, ci, a.labels, a.num_aggs))
        extra["cgs_setup_only_ms"], h2 = ev(lambda: m.ClusterSGS(rp, ci, vd, labels=a.labels, num_aggs=a.num_aggs,
                                                                 coarse=co))
        h2.close()
    x = torch.zeros(g.n, dtype=torch.float64, device="cuda")
    cg.apply(b, x, sweeps=1)
    ms_sweep, _ = ev(lambda: cg.apply(b, x, sweeps=1))
    # compulsory bytes of one symmetric sweep: 2 passes x (vals 8 + colinds 4 per nnz + rowptr, b, x, diag per row)
    byt = 2 * (12 * g.nnz + (8 + 8 + 8 + 8 + 8) * g.n)
    print(json.dumps({"config": cfg, "kind": kind, "n": g.n, "nnz": g.nnz, "ncolors": cg.ncolors,
                      "setup_ms": ms_setup, **extra, "sym_sweep_ms": ms_sweep, "sweep_GBps": byt / ms_sweep / 1e6}), flush=True)
    cg.close()
