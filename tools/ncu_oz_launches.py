"""k_oz_gemm launches of one Lanczos step from an ncu launch list: duration, DRAM bytes and INT8
(IMMA) pipe activity per launch, grouped by identical (read, write) byte counts (= GEMM shape)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    L = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        d = L.setdefault(int(r[idi]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(L)
    starts = [k for k in ids if "k_perturb" in L[k]["name"]]
    step = [k for k in ids if starts[0] <= k < starts[1]]
    groups = collections.OrderedDict()
    for k in step:
        d = L[k]
        if "k_oz_gemm" not in d["name"]:
            continue
        key = (round(d["dram__bytes_read.sum"] / 1e7), round(d["dram__bytes_write.sum"] / 1e7))
        g = groups.setdefault(key, [d["name"].split("(")[0].replace("void ", ""), 0, 0.0, 0.0, 0.0, 0.0])
        g[1] += 1
        g[2] += d["gpu__time_duration.sum"] / 1e3
        g[3] += d["dram__bytes_read.sum"] / 1e6
        g[4] += d["dram__bytes_write.sum"] / 1e6
        g[5] += d.get("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
    tot = sum(g[2] for g in groups.values())
    print(f"k_oz_gemm launches of one step: {sum(g[1] for g in groups.values())}, {tot / 1e3:.2f} ms (ncu, serialised)")
    print(f"{'kernel':28s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'read MB':>8s} {'write MB':>8s} {'IMMA %':>7s}")
    for name, n, us, rd, wr, imma in sorted(groups.values(), key=lambda g: -g[2]):
        print(f"{name[:28]:28s} {n:4d} {us / n:10.1f} {100 * us / tot:5.1f}% {rd / n:8.0f} {wr / n:8.0f} {imma / n:7.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
