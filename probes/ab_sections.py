"""Device-resident build sections at a config, many reps (A/B of env toggles:
run once per setting in separate processes).

    python probes/ab_sections.py [C3] [reps]
"""
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, DeviceProblem, ProblemSpec, build_hs_device, generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dp = DeviceProblem.from_instance(generate(ProblemSpec(CONFIGS[cfg], seed=0)))
for _ in range(3):
    build_hs_device(dp)
ts = [build_hs_device(dp)[3] for _ in range(reps)]
keys = ("loop1", "s1", "h1", "h3", "total", "h_core", "s_core")
env = {k: v for k, v in os.environ.items() if k.startswith("HSB_NO")}
print(cfg, env, {k: round(statistics.median(t[k] for t in ts) * 1e3, 3) for k in keys}, flush=True)
