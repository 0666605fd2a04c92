"""Key metrics of the first kernel in an ncu report, and a per-kernel table of a launch list.

    python probes/ncu_summary.py report.ncu-rep      # --set full capture
    python probes/ncu_summary.py launches.csv        # --metrics gpu__time_duration.sum list
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]

path = sys.argv[1]
if path.endswith(".ncu-rep"):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    print(v[h.index("Kernel Name")][:90])
    for k in KEYS:
        if k in h:
            print(f"  {k:70s} {v[h.index(k)]:>14s} {units[h.index(k)]}")
else:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[-1])
    tot = sum(v[1] for v in agg.values())
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name[:60]:60s} {n:4d} {t / 1e6:8.3f} ms {100 * t / tot:5.1f}%")
    print(f"total {tot / 1e6:.3f} ms")
