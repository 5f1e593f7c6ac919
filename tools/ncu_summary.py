"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch) by kernel."""
import collections, csv, sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    idi = hdr.index('ID')
    launches = collections.defaultdict(dict)
    for r in data:
        if len(r) <= vi:
            continue
        launches[r[idi]][r[mi]] = (r[vi], r[ui])
        launches[r[idi]]['name'] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for lid, m in launches.items():
        v, u = m['gpu__time_duration.sum']
        v = float(v.replace(',', ''))
        v *= {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3}.get(u, 1.0)
        name = m['name'].split('(')[0]
        if 'launch__grid_size' in m:
            name += f" grid={m['launch__grid_size'][0]}"
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':90s} {'n':>5s} {'total us':>10s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k[:90]:90s} {n:5d} {t:10.1f} {100 * t / tot:5.1f}%")
    print(f"launches {len(launches)}, total {tot / 1e3:.3f} ms")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
