"""Time the matching-coefficient kernel (HBM-write bound) at the BASELINE shapes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json  # noqa: E402

import torch  # noqa: E402

from paper_1611_00606_b200.physics import match_coeffs_device, synthetic_system  # noqa: E402

SHAPES = {"C1": (2, 1, 6, 500), "C2": (8, 2, 8, 3000), "C3": (32, 4, 10, 8000), "C4": (128, 4, 10, 20000)}
names = sys.argv[1:] or list(SHAPES)
peak = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json")).get("hbm_gbs", 6535.4) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6535.4
for name in names:
    na, nt, lmax, ng = SHAPES[name]
    system, k, kmax, g = synthetic_system(na, nt, lmax, ng, seed=0, kpt_frac=(0.1, 0.2, 0.3))
    for _ in range(3):
        a, b = match_coeffs_device(system, k, g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        match_coeffs_device(system, k, g)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nbytes = 2 * a.numel() * 16
    print(json.dumps({"config": name, "n_g": len(g), "rows": a.shape[1], "ms_per_call": ms,
                      "write_GB": nbytes / 1e9, "GBps": nbytes / ms / 1e6, "frac_of_hbm": nbytes / ms / 1e6 / peak}))
