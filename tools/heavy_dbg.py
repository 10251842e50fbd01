import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
cfg, it, ph = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
os.environ["MIS2_DBG_IT"], os.environ["MIS2_DBG_PH"] = str(it), str(ph)
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci)
r = m.mis2(rp, ci, timeline=True)
ws, wsb = m.workspace(m.OP_MIS2, g.n, g.nnz)
buf = np.zeros(1184 * 64, dtype=np.int64)
L = m.lib(); L.mis2_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
L.mis2_debug_read(ws.data_ptr(), wsb, g.n, buf.ctypes.data, buf.size)
d = buf.reshape(1184, 64)[:592]
t0 = d[:, 0].min()
steps_end = (d[:, 3] - t0) / 1e3
h_start = (d[:, 60] - t0) / 1e3
h_end = (d[:, 62] - t0) / 1e3
nh = d[:, 61]; he = d[:, 63]
print("phase us", np.round(r.stats[:6], 1).tolist())
print(f"steps end: median {np.median(steps_end):.1f} max {steps_end.max():.1f} us")
print(f"heavy: rows/block median {np.median(nh):.0f} max {nh.max()} entries/block median {np.median(he):.0f} max {he.max()}")
print(f"heavy time: median {np.median(h_end-h_start):.1f} max {(h_end-h_start).max():.1f} us ; end max {h_end.max():.1f}")
k = np.argmax(h_end - h_start); print("slowest block", k, "rows", nh[k], "entries", he[k], "time", (h_end-h_start)[k])
