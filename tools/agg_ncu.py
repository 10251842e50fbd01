"""Measurement aid: two aggregate() calls on a config (run under ncu for the
launch list of the second; tools/launch_list.py keeps the second half).
usage: python tools/agg_ncu.py CFG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mis2gen as G, paper_2204_02934_b200 as m
g = G.config_graph(int(sys.argv[1]))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
for _ in range(2):
    a = m.aggregate(rp, ci)
torch.cuda.synchronize()
print("num_aggs", a.num_aggs)
