"""One rank's partial build of a P-way atom shard (for an ncu launch list):
    python probes/shard_launches.py C4 8"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, DeviceProblem, Dims, GpuPolicy, ProblemSpec, build_hs_device, generate  # noqa: E402

name, P = sys.argv[1], int(sys.argv[2])
dims = CONFIGS[name]
p = generate(ProblemSpec(Dims(dims.n_atoms // P, dims.n_l, dims.n_g), seed=0))
dp = DeviceProblem.from_instance(p)
h = torch.empty((dims.n_g, dims.n_g), dtype=torch.complex128, device="cuda")
s = torch.empty_like(h)
for _ in range(2):
    t = build_hs_device(dp, h, s, GpuPolicy())[3]
torch.cuda.synchronize()
print({k: round(v * 1e3, 3) for k, v in t.items() if isinstance(v, float) and k not in ("h2d_bytes", "d2h_bytes")})
