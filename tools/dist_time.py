"""Measurement aid: the partitioned MIS-2 (mis2_dist_mis2, local transport:
P partitions in one cooperative launch on this GPU) against mis2() on a
config graph; CUDA events, L2 flushed before each call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
parts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
g = G.config_graph(cfg)
rp, ci = torch.from_numpy(g.rowptr).cuda(), torch.from_numpy(g.colinds).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

def timeit(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts), min(ts)

ref = m.mis2(rp, ci)
med, mn = timeit(lambda: m.mis2(rp, ci))
print(f"cfg{cfg} mis2(): {med*1e3:.1f} us (min {mn*1e3:.1f})", flush=True)
for P in parts:
    c = m.Comm.local_parts(P).set_graph(g.n, g.rowptr, g.colinds)
    out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    cnt, its = c.mis2(out)
    ok = cnt == ref.count and its == ref.iterations and torch.equal(out, ref.in_set)
    med, mn = timeit(lambda: c.mis2(out))
    print(f"cfg{cfg} local {P} parts: {med*1e3:.1f} us (min {mn*1e3:.1f}) ok={ok}", flush=True)
    c.close()
