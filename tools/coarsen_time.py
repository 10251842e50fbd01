"""Measurement aid: coarse-graph time (CUDA events, median of 5) on a config.
usage: [MIS2_LIB_PATH=alt.so] python tools/coarsen_time.py CFG"""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, mis2gen as G, paper_2204_02934_b200 as m
g = G.config_graph(int(sys.argv[1]))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
a = m.aggregate(rp, ci)
c0 = m.coarsen(rp, ci, a.labels, a.num_aggs)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = m.coarsen(rp, ci, a.labels, a.num_aggs); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print(os.environ.get("MIS2_LIB_PATH", "default"), sys.argv[1], sorted(ts)[2], int(c[1].numel()),
      torch.equal(c[0], c0[0]) and torch.equal(c[1], c0[1]))
