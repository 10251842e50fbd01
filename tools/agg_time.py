"""Measurement aid: aggregation time (CUDA events, median of 5) and stats on a config.
usage: [MIS2_LIB_PATH=alt.so] python tools/agg_time.py CFG"""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, mis2gen as G, paper_2204_02934_b200 as m
g = G.config_graph(int(sys.argv[1]))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
a = m.aggregate(rp, ci)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); a2 = m.aggregate(rp, ci); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print(os.environ.get("MIS2_LIB_PATH", "default"), sorted(ts)[2], a.num_aggs, a.stats, torch.equal(a.labels, a2.labels))
