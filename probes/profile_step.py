"""One device-resident H/S build (for ncu launch lists and --set full captures).

    python probes/profile_step.py [C2|C3|C4] [repeats]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, DeviceProblem, ProblemSpec, build_hs_device, generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = generate(ProblemSpec(CONFIGS[cfg], seed=0))
dp = DeviceProblem.from_instance(p)
for _ in range(reps):
    h, s, split, t, info = build_hs_device(dp)
torch.cuda.synchronize()
print(cfg, split, {k: round(v * 1e3, 3) for k, v in t.items() if isinstance(v, float)})
