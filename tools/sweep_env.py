"""Measurement aid: time mis2_async on a config under several values of one
tuning environment variable (read by libmis2 per call).  L2 flushed before
each timed call, CUDA events on the current stream.
usage: python tools/sweep_env.py CFG VAR v1,v2,... [--timeline]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m

cfg, var = int(sys.argv[1]), sys.argv[2]
vals = sys.argv[3].split(";") if ";" in sys.argv[3] else sys.argv[3].split(",")
g = G.config_graph(cfg)
rp = torch.from_numpy(g.rowptr).cuda(); ci = torch.from_numpy(g.colinds).cuda()
out = torch.empty(g.n, dtype=torch.uint8, device="cuda"); sc = torch.zeros(2, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = m.mis2(rp, ci)
for v in vals:
    os.environ[var] = v
    ts = []
    for r in range(25):
        flush.fill_(r & 0xff)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); m.mis2_async(rp, ci, out, sc); b.record(); b.synchronize()
        if r >= 5: ts.append(a.elapsed_time(b) * 1e3)
    try:
        r2 = m.mis2(rp, ci)
        ok = r2.count == ref.count and torch.equal(r2.in_set, ref.in_set)
    except Exception as e:  # measurement-only knobs may break the result
        ok = f"error {e}"[:40]
    line = f"{var}={v}: median {np.median(ts):.1f} us min {min(ts):.1f} us ok={ok}"
    if "--timeline" in sys.argv:
        flush.fill_(1); torch.cuda.synchronize()
        try:
            tl = m.mis2(rp, ci, timeline=True).stats
            line += " | phases " + " ".join(f"{x:.1f}" for x in tl)
        except Exception:
            pass
    print(line, flush=True)
