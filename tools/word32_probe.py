import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, mis2gen as G, paper_2204_02934_b200 as m
for ci in (1, 2, 4):
    g = G.config_graph(ci)
    rp = torch.from_numpy(g.rowptr).cuda(); cl = torch.from_numpy(g.colinds).cuda()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    row = {"config": ci}
    for wb in (64, 32):
        for s in ("xorstar", "fixed", "xor"):
            r = m.mis2(rp, cl, word_bits=wb, scheme=s)
            ts = []
            for _ in range(7):
                flush.zero_(); torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); m.mis2(rp, cl, word_bits=wb, scheme=s); b.record(); b.synchronize()
                ts.append(a.elapsed_time(b))
            row[f"w{wb}_{s}"] = dict(size=r.count, iters=r.iterations, ms=round(sorted(ts)[3], 4))
    print(json.dumps(row), flush=True)
