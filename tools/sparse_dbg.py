"""Per-block timing of one sparse phase (MIS2_FLAG_TIMELINE + MIS2_DBG_IT/PH)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
it, ph = int(sys.argv[1]), int(sys.argv[2])
os.environ["MIS2_DBG_IT"], os.environ["MIS2_DBG_PH"] = str(it), str(ph)
g = G.config_graph(int(os.environ.get("CFG", "1")))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.mis2(rp, ci)
r = m.mis2(rp, ci, timeline=True)
ws, wsb = m.workspace(m.OP_MIS2, g.n, g.nnz)
buf = np.zeros(1184 * 64, dtype=np.int64)
L = m.lib(); L.mis2_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
L.mis2_debug_read(ws.data_ptr(), wsb, g.n, buf.ctypes.data, buf.size)
d = buf.reshape(1184, 64)
act = d[:, 0] > 0
d = d[act]
t0 = d[:, 0].min()
print("phase us per iteration:", np.round(r.stats, 1).tolist())
print(f"blocks {act.sum()}  nsteps mean {d[:,1].mean():.1f} max {d[:,1].max()}  rows mean {d[:,2].mean():.0f} max {d[:,2].max()}")
print(f"start spread {(d[:,0].max()-t0)/1e3:.2f} us; end: median {np.median(d[:,3]-t0)/1e3:.2f} max {(d[:,3].max()-t0)/1e3:.2f} us")
for k in range(min(8, int(d[:, 1].max()))):
    sel = d[:, 1] > k
    st = d[sel, 4 + 5 * k: 9 + 5 * k].astype(np.float64)
    dt = np.diff(st, axis=1) / 1e3
    print(f"step {k}: n={sel.sum():4d} sync {np.median(dt[:,0]):6.2f} plan {np.median(dt[:,1]):6.2f} wait {np.median(dt[:,2]):6.2f} process {np.median(dt[:,3]):6.2f}   (max {dt.max(0).round(2).tolist()})  start@{np.median(st[:,0]-t0)/1e3:.2f}")
# per-SM view: blocks grouped by SM id (dbuf[59], dense phases only), end times
if (d[:, 59] > 0).any():
    ends = (d[:, 3] - t0) / 1e3
    sm = d[:, 59]
    per_sm_last = np.array([ends[sm == s].max() for s in np.unique(sm)])
    per_sm_first = np.array([ends[sm == s].min() for s in np.unique(sm)])
    print(f"SMs {len(per_sm_last)}: last block end median {np.median(per_sm_last):.2f} max {per_sm_last.max():.2f}; "
          f"first block end median {np.median(per_sm_first):.2f}")
# deferred (long) rows of the phase, per block (finish_phase: dbuf[60] start, [61] rows, [62] end, [63] entries)
hv = d[:, 60] > 0
if hv.any():
    dur = (d[hv, 62] - d[hv, 60]) / 1e3
    endh = (d[hv, 62] - t0) / 1e3
    print(f"deferred rows: blocks {hv.sum()}  rows/block median {np.median(d[hv,61]):.0f} max {d[hv,61].max()}  "
          f"entries/block median {np.median(d[hv,63]):.0f} max {d[hv,63].max()}  "
          f"time median {np.median(dur):.1f} max {dur.max():.1f} us  end median {np.median(endh):.1f} max {endh.max():.1f} us")
