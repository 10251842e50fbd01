"""One warm MIS-2 call on a config for ncu (kernel regex mis2_persistent)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mis2gen as G, paper_2204_02934_b200 as m
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
grp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
for _ in range(3):
    r = m.mis2(rp, ci, group=grp)
torch.cuda.synchronize()
print("count", r.count, "iters", r.iterations)
