"""Key metrics per captured launch from an ncu report (diagnostic; needs the ncu CLI)."""
import csv, io, subprocess, sys

KEYS = [
    ("Kernel Name", "kernel"), ("Grid Size", "grid"), ("Block Size", "block"),
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_%"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_inst_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc_pipe_%"),
    ("sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "uma_inst_%"),
    ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    tensor_cols = [h for h in hdr if "pipe_tensor" in h and "pct_of_peak_sustained_active" in h and h.startswith("sm__")]
    for r in data:
        parts = []
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                parts.append(f"{label}={r[i]}{(' ' + units[i]) if units[i] and label not in ('kernel', 'grid', 'block') else ''}")
        for h in tensor_cols:
            if not any(h == k for k, _ in KEYS):
                parts.append(f"{h.replace('.avg.pct_of_peak_sustained_active', '')}={r[hdr.index(h)]}%")
        print(" | ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
