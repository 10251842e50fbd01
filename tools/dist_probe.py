"""Measurement aid: the partitioned driver (local transport: P partitions on
this GPU) on a config -- time per mis2 / aggregate call vs the single-GPU
call.  usage: python tools/dist_probe.py CFG P1,P2,..."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mis2gen as G, paper_2204_02934_b200 as m

cfg = int(sys.argv[1]); parts = [int(x) for x in sys.argv[2].split(",")]
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()


def ev(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - a))
    return min(ts)


print(json.dumps({"cfg": cfg, "single_gpu_mis2_ms": ev(lambda: m.mis2(rp, ci))}), flush=True)
for P in parts:
    c = m.Comm.local_parts(P).set_graph(g.n, g.rowptr, g.colinds)
    out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    ms = ev(lambda: c.mis2(out))
    print(json.dumps({"cfg": cfg, "parts": P, "dist_mis2_ms_wall": ms, "launches": int(m.lib().mis2_last_launch_count())}),
          flush=True)
    c.close()
