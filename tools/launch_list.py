"""Measurement aid: per-kernel durations (ncu launch list CSV, metric
gpu__time_duration.sum) of the second half of the launches in a file."""
import csv, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
out = [(r[ki][:60], float(r[vi].replace(",", "")), r[ui]) for r in rows[1:]]
out = out[len(out) // 2:]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = 0.0
for k, v, u in out:
    us = v * scale.get(u, 1e-3)
    tot += us
    print("%-60s %10.1f us" % (k, us))
print("total %.1f us" % tot)
