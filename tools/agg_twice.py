import sys, os
sys.path.insert(0, os.getcwd())
import torch, mis2gen as G, paper_2204_02934_b200 as m
g = G.config_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
m.aggregate(rp, ci); torch.cuda.synchronize()
m.aggregate(rp, ci); torch.cuda.synchronize()
