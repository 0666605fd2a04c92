"""CUDA-event section times of the host-buffer build_hs path (C3) vs the device path."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, DeviceProblem, ProblemSpec, build_hs, build_hs_device, generate, pin_instance  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = pin_instance(generate(ProblemSpec(CONFIGS[cfg], seed=0)))
for _ in range(3):
    o = build_hs(p)
t = o.timings
print("host path:", {k: round(v * 1e3, 2) for k, v in t.items() if isinstance(v, float)})
dp = DeviceProblem.from_instance(p)
for _ in range(3):
    h, s, split, td, info = build_hs_device(dp)
torch.cuda.synchronize()
print("device path:", {k: round(v * 1e3, 2) for k, v in td.items() if isinstance(v, float)})
