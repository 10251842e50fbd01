"""Measurement aid: C-config MIS-2 time (CUDA events, L2 flushed) per lane-group
width G and tile mode (MIS2_SMALL_TILES read per call).
usage: python tools/probe_group.py CFG G1,G2,... MODE1,MODE2,..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as Gen, paper_2204_02934_b200 as m
g = Gen.config_graph(int(sys.argv[1]))
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
out = torch.empty(g.n, dtype=torch.uint8, device="cuda"); sc = torch.zeros(2, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = m.mis2(rp, ci)
for mode in sys.argv[3].split(","):
    os.environ["MIS2_SMALL_TILES"] = mode
    for grp in [int(x) for x in sys.argv[2].split(",")]:
        ts = []
        for r in range(25):
            flush.fill_(r & 0xff)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); m.mis2_async(rp, ci, out, sc, group=grp); b.record(); b.synchronize()
            if r >= 5: ts.append(a.elapsed_time(b) * 1e3)
        r2 = m.mis2(rp, ci, group=grp)
        ok = r2.count == ref.count and torch.equal(r2.in_set, ref.in_set)
        tl = m.mis2(rp, ci, group=grp, timeline=True)
        print(f"small={mode} G={grp}: median {np.median(ts):.1f} us ok={ok} | " + " ".join(f"{x:.1f}" for x in tl.stats), flush=True)
