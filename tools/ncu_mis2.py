"""MIS-2 calls on a config for ncu (kernel regex mis2_persistent).
usage: ncu_mis2.py [config] [group] [max_iters]  (max_iters > 0: partial run)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mis2gen as G, paper_2204_02934_b200 as m
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
grp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mi = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
for _ in range(3):
    r = m.mis2(rp, ci, group=grp, max_iters=mi, allow_partial=True)
torch.cuda.synchronize()
print("count", r.count, "iters", r.iterations)
