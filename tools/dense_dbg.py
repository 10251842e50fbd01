import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
cfg, it, ph = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
os.environ["MIS2_DBG_IT"], os.environ["MIS2_DBG_PH"] = str(it), str(ph)
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci)
L = m.lib(); L.mis2_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
ends = []
for rep in range(3):
    r = m.mis2(rp, ci, timeline=True)
    ws, wsb = m.workspace(m.OP_MIS2, g.n, g.nnz)
    buf = np.zeros(1184 * 64, dtype=np.int64)
    L.mis2_debug_read(ws.data_ptr(), wsb, g.n, buf.ctypes.data, buf.size)
    d = buf.reshape(1184, 64)[:592]
    t0 = d[:, 0].min()
    ends.append((d[:, 3] - t0) / 1e3)
    sm = d[:, 59]
    st = (d[:, 0] - t0) / 1e3
e = np.array(ends)
print("phase us", np.round(r.stats[:4], 1).tolist())
print("end per rep: median", np.median(e, 1).round(1), "max", e.max(1).round(1))
print("start spread", st.max().round(2), "corr(end rep0, rep1)", np.corrcoef(e[0], e[1])[0, 1].round(2))
slow = np.argsort(-e.mean(0))[:15]
print("slowest blocks", slow.tolist(), "sm", sm[slow].tolist(), "end", e.mean(0)[slow].round(1).tolist())
per_sm = {}
for b in range(592): per_sm.setdefault(int(sm[b]), []).append(e.mean(0)[b])
sm_mean = {k: np.mean(v) for k, v in per_sm.items()}
ks = sorted(sm_mean, key=lambda k: -sm_mean[k])
print("slowest SMs", [(k, round(sm_mean[k], 1), len(per_sm[k])) for k in ks[:8]], "fastest", [(k, round(sm_mean[k], 1)) for k in ks[-4:]])
print("end by block quartile", [round(float(np.median(e.mean(0)[q*148:(q+1)*148])), 1) for q in range(4)])
