"""Measurement aid: per-block timing of one push-form Decide phase
(MIS2_DBG_IT, phase 1).  usage: python tools/decide_dbg.py CFG IT"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
cfg, it = int(sys.argv[1]), int(sys.argv[2])
os.environ["MIS2_DBG_IT"], os.environ["MIS2_DBG_PH"] = str(it), "1"
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci)
L = m.lib(); L.mis2_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
r = m.mis2(rp, ci, timeline=True)
ws, wsb = m.workspace(m.OP_MIS2, g.n, g.nnz)
buf = np.zeros(1184 * 64, dtype=np.int64)
L.mis2_debug_read(ws.data_ptr(), wsb, g.n, buf.ctypes.data, buf.size)
d = buf.reshape(1184, 64)
nb = int((d[:, 0] > 0).sum()); d = d[:nb]
t0 = d[:, 0].min()
f = lambda c: (d[:, c] - t0) / 1e3
print(f"phase us {r.stats[2*it+1]:.1f}  blocks {nb}  rows/block median {np.median(d[:,1])}")
for nm, c in [("start", 0), ("loop end", 2), ("after sync", 5), ("cands end", 3)]:
    x = f(c); print(f"  {nm:10s} median {np.median(x):6.2f}  p90 {np.percentile(x,90):6.2f}  max {x.max():6.2f}")
print("  candidates per block: median", np.median(d[:, 4]), "max", d[:, 4].max())
