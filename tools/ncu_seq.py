"""Per-launch sequence (kernel, grid, duration us) of an ncu --metrics gpu__time_duration.sum CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
gi = h.index('Grid Size') if 'Grid Size' in h else None
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', '')) * {'nsecond': 1e-3, 'usecond': 1, 'msecond': 1e3}.get(r[ui], 1)
    print(f"{r[ki].split('(')[0][-32:]:34s} {r[gi] if gi else '':16s} {v:9.1f}")
