"""Per-step kernel-class totals from an ncu launch list (CSV of gpu__time_duration.sum [+ DRAM bytes,
IMMA-pipe %]): steps are delimited by the perturb kernel that starts every Lanczos step / HVP.
Durations are ncu's (serialised, cold cache), so the SHARES are what compare with a timed step.
usage: python tools/ncu_classes.py launches.csv"""
import collections
import csv
import sys

CLASSES = [("gemm_i8", ("k_oz_gemm",)), ("oz_slice", ("k_oz_slice", "k_oz_colexp", "k_att_rows", "k_att_cols")),
           ("gemm", ("gemm_dmma_kernel", "splitk_reduce", "gemm_kernel", "k_tc_")),
           ("attention", ("softmax", "k_att_sm")), ("norm", ("layernorm", "rmsnorm", "colreduce")),
           ("cross_entropy", ("cross_entropy",)), ("embedding", ("embed", "pos_bwd")),
           ("perturb", ("perturb",)), ("fd_lanczos", ("k_fd",)), ("reorth", ("reorth", "gram")),
           ("elementwise", ("rope", "swiglu", "k_add", "convert", "gelu", "k_oz_act"))]


def cls_of(name):
    for c, keys in CLASSES:
        if any(k in name for k in keys):
            return c
    return "vector"


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    L = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        d = L.setdefault(int(r[idi]), {"name": r[ki]})
        d[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    launches = [L[k] for k in sorted(L)]
    steps, cur = [], None
    for d in launches:
        if "k_perturb" in d["name"]:
            cur = collections.defaultdict(lambda: [0, 0.0, 0.0])
            steps.append(cur)
        if cur is None:
            continue
        v, u = d["gpu__time_duration.sum"]
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
        byt = sum(d.get(m, (0, ""))[0] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        c = cur[cls_of(d["name"])]
        c[0] += 1
        c[1] += us
        c[2] += byt
    for i, st in enumerate(steps):
        tot = sum(c[1] for c in st.values())
        print(f"step {i}: {sum(c[0] for c in st.values())} launches, {tot / 1e3:.2f} ms (ncu, serialised)")
        for k, (n, us, byt) in sorted(st.items(), key=lambda x: -x[1][1]):
            print(f"  {k:14s} {n:5d} launches {us / 1e3:9.3f} ms {100 * us / tot:5.1f}%  DRAM {byt / 1e9:7.2f} GB "
                  f"({byt / n / 1e6 if n else 0:8.1f} MB/launch)")


if __name__ == "__main__":
    main(sys.argv[1])
