"""Measurement aid: per-kernel durations of the last of two repeated calls in
an ncu launch list (`--metrics gpu__time_duration.sum --csv`)."""
import csv, sys
for f in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(f) if not l.startswith('==')))
    h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
    out = [(r[ki][:44], int(r[vi].replace(',', ''))) for r in rows[1:]]
    out = out[len(out) // 2:]
    print(f, 'total us', sum(v for _, v in out) / 1e3)
    for k, v in out:
        if v > 8000: print('  %-44s %9.1f' % (k, v / 1e3))
