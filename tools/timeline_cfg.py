import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
cfg = int(sys.argv[1]); grp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci, group=grp)
r = m.mis2(rp, ci, timeline=True, group=grp)
st = m.mis2(rp, ci, stats=True, group=grp).stats
print("phase us:", np.round(r.stats, 1).tolist(), "sum", round(float(r.stats.sum()), 1), "init/final us", r.extra)
print("wl1:", st[:, 0].tolist()); print("wl2:", st[:, 1].tolist())
d = np.diff(g.rowptr); print("deg max", d.max(), "rows>256", (d > 256).sum(), "entries in rows>256", d[d > 256].sum())
