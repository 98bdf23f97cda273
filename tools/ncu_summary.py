"""Key metrics of ncu --set full reports (one kernel launch each) as a
markdown table: time, DRAM bytes and throughput, L2 hit rate, occupancy,
FP64 / DMMA pipe activity, registers.

    python tools/ncu_summary.py profiles/*.ncu-rep > profiles/r1_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("dram_TBps", "dram__bytes.sum.per_second"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("dmma_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Kbyte": 1e-3, "byte": 1e-6,
         "Tbyte/s": 1.0, "Gbyte/s": 1e-3}


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:48]}
        for name, key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                try:
                    v = float(vals[i].replace(",", ""))
                    v *= SCALE.get(units[i], 1.0)
                    d[name] = round(v, 3)
                except ValueError:
                    d[name] = vals[i]
        res.append(d)
    return res


def main():
    print("| report | kernel | " + " | ".join(n for n, _ in KEYS) + " |")
    print("|" + "---|" * (len(KEYS) + 2))
    for p in sys.argv[1:]:
        for d in summarize(p):
            print(f"| {p.split('/')[-1]} | `{d['kernel']}` | " + " | ".join(str(d.get(n, "")) for n, _ in KEYS) + " |")


if __name__ == "__main__":
    main()
