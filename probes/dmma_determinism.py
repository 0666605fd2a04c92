"""Repeat one DMMA triangle launch (hsb_zherk, 3M with sum planes: the S/H
kernel of the DMMA engine) on fixed device data from process start and
compare every result bit for bit with the first: does the kernel alone
produce the early-run disagreements?"""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import _lib  # noqa: E402

n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 2100, int(sys.argv[2]) if len(sys.argv) > 2 else 968
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
lib = _lib.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn((n, k), dtype=torch.complex128, device=dev, generator=g)  # column-major k x n
outs = []
t0 = time.time()
with _lib.using(0, "3m", "dmma") as ctx:
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ref = None
    bad = 0
    for r in range(reps):
        c = torch.zeros((n, n), dtype=torch.complex128, device=dev)
        _lib.check(lib.hsb_zherk(ctx, st, n, k, 1.0, ctypes.c_void_p(a.data_ptr()), k, 0.0,
                                 ctypes.c_void_p(c.data_ptr()), n, 0), ctx)
        torch.cuda.synchronize()
        if ref is None:
            ref = c.clone()
            continue
        if not torch.equal(c, ref):
            d = (c != ref).nonzero()
            bad += 1
            print(f"rep {r} t={time.time() - t0:.1f}s: {d.shape[0]} entries differ, first {d[:3].tolist()}", flush=True)
print(f"n {n} k {k}: {bad} of {reps - 1} launches differ from the first")
