"""Host<->device bandwidth: H2D alone, D2H alone, and both at once (pinned, 1 GiB)."""
import time

import torch

n = 1 << 30
h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_src, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_dst.copy_(d_b, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


for name, a, b in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
    t = run(a, b)
    print(f"{name}: {t*1e3:.1f} ms, {(a + b) * n / t / 1e9:.1f} GB/s aggregate")
