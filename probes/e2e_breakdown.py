"""Where does the end-to-end (host numpy in/out) build time go?"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, ProblemSpec, build_hs, generate, validate_instance  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = generate(ProblemSpec(CONFIGS[cfg], seed=0))
t0 = time.perf_counter(); validate_instance(p); t1 = time.perf_counter()
print(f"validate_instance {1e3*(t1-t0):.1f} ms")
for i in range(4):
    t0 = time.perf_counter()
    out = build_hs(p)
    t1 = time.perf_counter()
    t = out.timings
    print(f"iter {i}: wall {1e3*(t1-t0):.1f} ms | C total {1e3*t['total']:.1f} h2d {1e3*t['h2d']:.1f} "
          f"d2h(after H) {1e3*t['d2h']:.1f} compute {1e3*(t['total']-t['h2d']-t['d2h']):.1f}")
a = np.asarray(p.a_blocks[0])
t0 = time.perf_counter(); np.isfinite(a).all(); t1 = time.perf_counter()
print(f"isfinite one block ({a.nbytes/1e6:.1f} MB) {1e3*(t1-t0):.2f} ms")
x = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for d in ("h2d", "d2h"):
    t0 = time.perf_counter()
    (y.copy_(x, non_blocking=True) if d == "h2d" else x.copy_(y, non_blocking=True))
    torch.cuda.synchronize()
    print(f"pinned {d} 1 GiB: {(1<<30)/(time.perf_counter()-t0)/1e9:.1f} GB/s")
src = np.ones(1 << 27)  # 1 GiB pageable
dst = x.numpy().view(np.float64)
t0 = time.perf_counter(); np.copyto(dst, src); t1 = time.perf_counter()
print(f"single-thread host memcpy 1 GiB: {(1<<30)/(t1-t0)/1e9:.1f} GB/s")
