"""Per-k-point wall time of iter_hs_kpoints vs serial build_hs (C3 by default).

    python probes/kpoint_pipeline.py [C2|C3] [n] [depth]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, ProblemSpec, build_hs, generate, iter_hs_kpoints, pin_instance  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 2
p = pin_instance(generate(ProblemSpec(CONFIGS[cfg], seed=0)))
for _ in range(3):
    o = build_hs(p)
del o
t0 = time.perf_counter()
for _ in range(n):
    o = build_hs(p)
    del o
t_serial = (time.perf_counter() - t0) / n
for o in iter_hs_kpoints([p] * (depth + 2), depth=depth):  # warm contexts + pinned cache
    del o
t0 = time.perf_counter()
stamps = []
for o in iter_hs_kpoints([p] * n, depth=depth):
    stamps.append(time.perf_counter() - t0)
    del o
t_pipe = stamps[-1] / n
print(f"{cfg}: serial {t_serial*1e3:.1f} ms/k-point, pipelined depth {depth}: {t_pipe*1e3:.1f} ms/k-point")
print("completion stamps (ms):", [round(s * 1e3, 1) for s in stamps])
