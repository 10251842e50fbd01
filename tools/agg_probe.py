"""Measurement aid: one aggregate + coarsen call on a config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mis2gen as G, paper_2204_02934_b200 as m
g = G.config_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
for _ in range(2):
    a = m.aggregate(rp, ci)
    c = m.coarsen(rp, ci, a.labels, a.num_aggs)
torch.cuda.synchronize()
print("aggs", a.num_aggs, a.stats)
