"""Host overhead of one device-resident build at small sizes (C2): wall time per call
vs the CUDA-event span of the build (timings['total'])."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, DeviceProblem, GpuPolicy, ProblemSpec, build_hs_device, generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
dp = DeviceProblem.from_instance(generate(ProblemSpec(CONFIGS[cfg], seed=0)))
for eng in ("int8", "dmma"):
    pol = GpuPolicy(engine=eng)
    for _ in range(5):
        build_hs_device(dp, policy=pol)
    torch.cuda.synchronize()
    n = 20
    t0 = time.perf_counter()
    spans = []
    for _ in range(n):
        _, _, _, t, _ = build_hs_device(dp, policy=pol)
        spans.append(t["total"])
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n
    print(f"{cfg} {eng}: wall {wall*1e3:.3f} ms/call, GPU span {sum(spans)/n*1e3:.3f} ms, launches {t['launches']}")
