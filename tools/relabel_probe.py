"""Measurement aid: MIS-2 time on a degree-ordered relabelling of a config graph
(hubs first) against the original ids -- the locality the internal relabelling
would buy (results differ: the ids are different)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = G.config_graph(cfg)
deg = np.diff(g.rowptr)
t = time.time()
perm = np.argsort(-deg, kind="stable").astype(np.int64)          # new -> old
inv = np.empty(g.n, dtype=np.int64); inv[perm] = np.arange(g.n)  # old -> new
nd = deg[perm]
rp2 = np.zeros(g.n + 1, dtype=np.int64); np.cumsum(nd, out=rp2[1:])
src = np.repeat(g.rowptr[perm], nd) + (np.arange(rp2[-1]) - np.repeat(rp2[:-1], nd))
ci2 = inv[g.colinds[src]].astype(np.int32)
print(f"host relabel {time.time()-t:.1f} s; top-1% rows hold {nd[:g.n//100].sum()/g.nnz:.2f} of nnz")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, rp, ci in (("original", g.rowptr, g.colinds), ("degree-ordered", rp2, ci2)):
    rp_d, ci_d = torch.from_numpy(rp).cuda(), torch.from_numpy(np.ascontiguousarray(ci)).cuda()
    for keys in ("auto", "off", "on"):
        m.mis2(rp_d, ci_d, keys=keys)
        ts = []
        for _ in range(3):
            flush.zero_(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); r = m.mis2(rp_d, ci_d, keys=keys); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
        print(f"{name:15s} keys={keys:4s} {min(ts):8.2f} ms  |S|={r.count} iters={r.iterations}", flush=True)
    del rp_d, ci_d
