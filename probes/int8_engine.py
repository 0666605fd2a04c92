"""INT8 (CRT) engine vs FP64 DMMA on one build: accuracy and device time.

    python probes/int8_engine.py [C2|C3|C4] [bits]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import (CONFIGS, DeviceProblem, GpuPolicy, ProblemSpec, build_hs_device,  # noqa: E402
                                   generate, rel_frob_error)

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = generate(ProblemSpec(CONFIGS[cfg], seed=0))
dp = DeviceProblem.from_instance(p)
res = {}
for name, pol in (("dmma", GpuPolicy(engine="dmma")), ("int8", GpuPolicy(engine="int8", int8_bits=bits))):
    for _ in range(2):
        h, s, split, t, info = build_hs_device(dp, policy=pol)
    torch.cuda.synchronize()
    reps = 3
    t0 = time.perf_counter()
    ts = []
    for _ in range(reps):
        h, s, split, t, info = build_hs_device(dp, policy=pol)
        ts.append(t)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    res[name] = (h.clone(), s.clone())
    print(name, f"wall {wall*1e3:.2f} ms", {k: round(v * 1e3, 3) for k, v in ts[-1].items() if isinstance(v, float)},
          flush=True)
hd, sd = res["dmma"]
hi, si = res["int8"]
eh = (torch.linalg.norm(hi - hd) / (1 + torch.linalg.norm(hd))).item()
es = (torch.linalg.norm(si - sd) / (1 + torch.linalg.norm(sd))).item()
print(f"{cfg} int8 vs dmma: rel frob H {eh:.3e}  S {es:.3e}")
