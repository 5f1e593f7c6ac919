"""Summaries of the round-1 final evidence run (tools/prof_r01b.sh) into profiles/ (diagnostic)."""
import collections, csv, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    K, M, V, I = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = {}
    for r in rows[hi + 1:]:
        if len(r) > V:
            d.setdefault((int(r[I]), r[K].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")),
                         {})[r[M]] = float(r[V].replace(",", ""))
    return d


d = launches(os.path.join(G, "fb_launches_c2.csv"))
shutil.copy(os.path.join(G, "fb_launches_c2.csv"), os.path.join(P, "launches_r01_c2_final.csv"))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, k), m in d.items():
    a = agg[k]
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"]
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
with open(os.path.join(P, "launches_r01_c2_final_summary.txt"), "w") as f:
    f.write("# c2 launch list (bench.py --steps 2 --warmup 1, launches 600..1099): ncu --metrics gpu__time_duration.sum,"
            "launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (cold cache, serialised)\n")
    f.write("kernel launches total_us mean_us share_% mean_dram_MB\n")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{k} {a[0]} {a[1] / 1e3:.1f} {a[1] / a[0] / 1e3:.1f} {100 * a[1] / tot:.1f} {a[2] / a[0] / 1e6:.2f}\n")
gm = [(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) for (i, k), m in d.items()
      if "gemm_dmma" in k or "splitk_reduce" in k]
traffic = {"gemm": {"dram_bytes_per_launch": sum(gm) / len(gm), "launches_captured": len(gm),
                    "note": "mean dram__bytes_read.sum + dram__bytes_write.sum over the DMMA GEMM (+ split-K reduce) "
                            "launches of profiles/launches_r01_c2_final.csv (ncu launch list of bench.py --steps 2, "
                            "cold cache)"}}
o = launches(os.path.join(G, "fb_oz_c3.csv"))
ob = [(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) for m in o.values()]
with open(os.path.join(P, "ncu_r01_c3_oz_launches.txt"), "w") as f:
    f.write("# k_oz_gemm launches of one c3 step (FP64_OZ): ncu --metrics gpu__time_duration.sum,launch__grid_size,"
            "dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg."
            "pct_of_peak_sustained_active --clock-control none -k regex:k_oz_gemm -c 40\n")
    f.write("id kernel duration_us dram_read_MB dram_write_MB imma_pipe_active_%\n")
    for (i, k), m in sorted(o.items()):
        f.write(f"{i} {k} {m['gpu__time_duration.sum'] / 1e3:.1f} {m.get('dram__bytes_read.sum', 0) / 1e6:.1f} "
                f"{m.get('dram__bytes_write.sum', 0) / 1e6:.1f} "
                f"{m.get('sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f}\n")
traffic["gemm_i8"] = {"dram_bytes_per_launch": sum(ob) / len(ob), "launches_captured": len(ob),
                      "note": "mean DRAM bytes of the k_oz_gemm launches of one c3 step "
                              "(profiles/ncu_r01_c3_oz_launches.txt, cold cache)"}
json.dump(traffic, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
rep = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_report.py"), os.path.join(G, "fb_oz_c5g.ncu-rep")],
                     capture_output=True, text=True).stdout
with open(os.path.join(P, "ncu_r01_c5gemm_oz_full.txt"), "w") as f:
    f.write("# ncu --set full --clock-control none -k regex:k_oz_gemm -s 8 -c 1, bench.py --config c5_gemm "
            "(Llama-3-8B layer shapes), summarised with tools/ncu_report.py\n" + rep)
for n, src in (("bench_r01_c2_final.json", "fb_c2.json"), ("bench_r01_c3_oz.json", "fb_c3.json"),
               ("bench_r01_c5gemm_oz.json", "fb_c5g.json")):
    shutil.copy(os.path.join(G, src), os.path.join(P, n))
print("ok", traffic)
