"""Timing of every §8 row on the BASELINE configs (device-resident inputs,
CUDA events, L2 flushed before each timed call).  Prints one JSON line per
measurement; used to fill profiles/ and BASELINE.md."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mis2gen as G, paper_2204_02934_b200 as m

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); r = fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2], r


cfgs = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "1", "2", "3", "4"])]
for ci in cfgs:
    t0 = time.time(); g = G.config_graph(ci); gen_s = time.time() - t0
    rp = torch.from_numpy(g.rowptr).cuda(); cl = torch.from_numpy(g.colinds).cuda()
    out = torch.empty(max(g.n, 1), dtype=torch.uint8, device="cuda")
    sc = torch.zeros(2, dtype=torch.int64, device="cuda")
    ms, _ = timed(lambda: m.mis2_async(rp, cl, out, sc))
    r = m.mis2(rp, cl)
    row = {"config": ci, "n": g.n, "nnz": g.nnz, "gen_s": round(gen_s, 1), "mis2_ms": ms, "mis2_gteps": g.nnz / ms / 1e6,
           "mis2_size": r.count, "iters": r.iterations}
    if ci != 3:
        ms_a, a = timed(lambda: m.aggregate(rp, cl), reps=3)
        row.update(agg_ms=ms_a, num_aggs=a.num_aggs)
        ms_c, cc = timed(lambda: m.coarsen(rp, cl, a.labels, a.num_aggs), reps=3)
        row.update(coarsen_ms=ms_c, coarse_nnz=int(cc[1].numel()))
    if ci == 4 or ci == 1:
        ms_ml, ml = timed(lambda: m.multilevel(rp, cl, threshold=1000), reps=2)
        row.update(multilevel_ms=ms_ml, levels=[l[0] for l in ml[0]] + [int(ml[1][0].numel() - 1)])
    print(json.dumps(row), flush=True)
    del rp, cl, out
    torch.cuda.empty_cache()
