"""Measurement aid: per-block timing of the push-form Decide (decide_push's
MIS2_DBG_IT / MIS2_DBG_PH=1 records): main loop, candidate resolution."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
it = int(sys.argv[1]) if len(sys.argv) > 1 else 0
os.environ["MIS2_DBG_IT"], os.environ["MIS2_DBG_PH"] = str(it), "1"
g = G.config_graph(int(os.environ.get("CFG", "1")))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci)
r = m.mis2(rp, ci, timeline=True)
ws, wsb = m.workspace(m.OP_MIS2, g.n, g.nnz)
buf = np.zeros(1184 * 64, dtype=np.int64)
L = m.lib(); L.mis2_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
L.mis2_debug_read(ws.data_ptr(), wsb, g.n, buf.ctypes.data, buf.size)
d = buf.reshape(1184, 64)
d = d[d[:, 0] > 0]
t0 = d[:, 0].min()
q = lambda a: f"median {np.median(a):.2f} max {a.max():.2f}"
print("phase us:", np.round(r.stats, 1).tolist())
print(f"blocks {len(d)} rows {q(d[:,1])} cands {q(d[:,4])}")
print(f"start  {q((d[:,0]-t0)/1e3)}")
print(f"loop   {q((d[:,2]-d[:,0])/1e3)}")
print(f"sync   {q((d[:,5]-d[:,2])/1e3)}")
print(f"cands  {q((d[:,3]-d[:,5])/1e3)}")
print(f"end    {q((d[:,3]-t0)/1e3)}")
