"""Measured dense INT8 tensor peak of this B200 through cuBLASLt (torch._int_mm,
int8 x int8 -> int32), the INT8 counterpart of MEASURED_PEAKS.json's bf16 rows:
burst = best of 10 single 8192^3 products; sustained = back to back for 4 s.
Writes profiles/int8_peak_r01.json."""
import json
import subprocess
import sys
import time
from pathlib import Path

import torch

n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()  # column-major B (cuBLASLt TN)
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
ops = 2.0 * n ** 3
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = max(best, ops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                        "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
count = 0
while time.perf_counter() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    count += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = ops * count / (e0.elapsed_time(e1) * 1e-3) / 1e12
smi.terminate()
lines = [l.split(",") for l in smi.stdout.read().strip().splitlines() if l.count(",") == 2]
clk = sorted(float(l[0]) for l in lines) if lines else [0]
res = {"probe": "torch._int_mm (cuBLASLt int8 GEMM, int32 out)", "n": n, "int8_tops_burst": best,
       "int8_tops_sustained": sustained, "sm_mhz_median_sustained": clk[len(clk) // 2],
       "power_w_max": max((float(l[1]) for l in lines), default=0.0),
       "sw_power_cap_seen": any("Active" in l[2] for l in lines)}
print(json.dumps(res))
out = Path(__file__).resolve().parents[1] / "profiles" / "int8_peak_r01.json"
if len(sys.argv) > 1:
    out = Path(sys.argv[1])
out.write_text(json.dumps(res, indent=1) + "\n")
