"""Measurement aid: per-step timestamps of one instrumented phase
(MIS2_DBG_IT / MIS2_DBG_PH), medians over blocks.
usage: python tools/dense_steps.py CFG IT PH"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
cfg, it, ph = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
os.environ["MIS2_DBG_IT"], os.environ["MIS2_DBG_PH"] = str(it), str(ph)
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci)
L = m.lib(); L.mis2_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda"); flush.fill_(3); torch.cuda.synchronize()
r = m.mis2(rp, ci, timeline=True)
ws, wsb = m.workspace(m.OP_MIS2, g.n, g.nnz)
buf = np.zeros(1184 * 64, dtype=np.int64)
L.mis2_debug_read(ws.data_ptr(), wsb, g.n, buf.ctypes.data, buf.size)
nb = int((buf.reshape(1184, 64)[:, 0] > 0).sum())
d = buf.reshape(1184, 64)[:nb]
t0 = d[:, 0].min()
print("blocks", nb, "phase us", np.round(r.stats[2 * it + ph], 1), "nsteps median", np.median(d[:, 1]))
print("start spread us", ((d[:, 0] - t0) / 1e3).max().round(2), "loop end median/max", np.median((d[:, 3] - t0) / 1e3).round(1), ((d[:, 3] - t0) / 1e3).max().round(1),
      "finish end median/max", np.median((d[:, 62] - t0) / 1e3).round(1), ((d[:, 62] - t0) / 1e3).max().round(1))
names = ["sync", "prefetch", "mbar_wait", "process"]
for k in range(11):
    s = d[:, 4 + 5 * k: 9 + 5 * k]
    ok = s[:, 4] > 0
    if ok.sum() == 0: break
    dd = np.diff(s[ok], axis=1) / 1e3
    st = (s[ok, 0] - t0) / 1e3
    print(f"step {k:2d} n={ok.sum():4d} start {np.median(st):6.2f}  " + "  ".join(f"{nm} {np.median(dd[:, i]):5.2f}/{np.percentile(dd[:, i], 90):5.2f}" for i, nm in enumerate(names)))
