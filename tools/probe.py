"""Quick timing probe of MIS-2 on the bench config for several group widths."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mis2gen as G
import paper_2204_02934_b200 as m

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
sc = torch.zeros(2, dtype=torch.int64, device="cuda")
for grp in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "4", "8", "16", "32"])]:
    r = m.mis2(rp, ci, group=grp)
    ts = []
    for k in range(12):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); m.mis2_async(rp, ci, out, sc, group=grp); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts = sorted(ts[2:])
    warm = []
    for k in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); m.mis2_async(rp, ci, out, sc, group=grp); e.record(); torch.cuda.synchronize()
        warm.append(s.elapsed_time(e))
    print(f"cfg{cfg} n={g.n} nnz={g.nnz} G={grp} count={r.count} it={r.iterations} cold(L2 flushed) med {ts[len(ts)//2]:.4f} ms min {ts[0]:.4f}  warm med {sorted(warm)[5]:.4f} ms  GTEPS(cold) {g.nnz/ts[len(ts)//2]/1e6:.1f}", flush=True)

if os.environ.get("TIMELINE"):
    for grp in [1, 2]:
        m.mis2(rp, ci, group=grp)
        r = m.mis2(rp, ci, group=grp, timeline=True)
        print(f"G={grp} phase us (col,dec per iteration):", np.round(r.stats, 1).tolist(), "sum", round(float(r.stats.sum()), 1))
