"""Measurement aid: aggregate() through the C ABI with fixed output / workspace
buffers (CUDA-graph replay eligible), CUDA events around each call, L2 flushed
between calls; MIS2_AGG_GRAPH read per call.  usage: python tools/agg_graph_probe.py CFG"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m
g = G.config_graph(int(sys.argv[1]))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
gg, n, nnz = m._graph(rp, ci)
o = m._opts(0, "xorstar", 0, 0)
ws, wsb = m.workspace(m.OP_AGGREGATE, n, nnz)
labels = torch.empty(n, dtype=torch.int32, device="cuda"); roots = torch.empty(n, dtype=torch.int32, device="cuda")
na = ctypes.c_int64(0); st = np.zeros(8, dtype=np.int64)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = m.aggregate(rp, ci)
for mode in ("0", "1"):
    os.environ["MIS2_AGG_GRAPH"] = mode
    ts = []
    for r in range(25):
        flush.fill_(r & 0xff)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = m.lib().mis2_aggregate(ctypes.byref(gg), ctypes.byref(o), labels.data_ptr(), ctypes.byref(na),
                                    roots.data_ptr(), st.ctypes.data, ws.data_ptr(), wsb, m._stream())
        b.record(); b.synchronize()
        assert rc == 0
        if r >= 5: ts.append(a.elapsed_time(b) * 1e3)
    ok = na.value == ref.num_aggs and torch.equal(labels, ref.labels)
    print(f"graph={mode}: median {np.median(ts):.1f} us min {min(ts):.1f} us ok={ok} launches={m.lib().mis2_last_launch_count()}", flush=True)
