"""Multi-process check of the fused scatter (CUDA-IPC receive slots): each rank
builds its atoms' partial H/S into the owners' slots; every rank's column block
is compared with the single-process build.  Run under torchrun (ranks may
share one GPU: HSB_DIST_BACKEND=gloo)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1611_00606_b200 import DeviceProblem, Dims, GpuPolicy, ProblemSpec, build_hs_device, generate  # noqa: E402
from paper_1611_00606_b200 import distributed as hd  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
torch.cuda.set_device(dev)
dist.init_process_group(os.environ.get("HSB_DIST_BACKEND", "nccl"))
p = generate(ProblemSpec(Dims(6, 121, 1500), seed=77, nonhpd_fraction=0.3))
pol = GpuPolicy(engine="int8")
slots = hd.PeerSlots.group(p.dims.n_g, dev)
lo, hi = hd.atom_ranges(p.dims.n_atoms, world)[rank]
dp = DeviceProblem.from_instance(hd.shard_instance(p, range(lo, hi)))
hb, sb = hd.build_hs_sharded_fused(dp, slots, pol)
h, s, _, _, _ = build_hs_device(DeviceProblem.from_instance(p), policy=pol)
torch.cuda.synchronize()
c0, c1 = rank * slots.cols, min((rank + 1) * slots.cols, p.dims.n_g)
scale = 1 + torch.linalg.norm(h).item()
eh = torch.linalg.norm(hb[: c1 - c0] - h[c0:c1]).item() / scale
es = torch.linalg.norm(sb[: c1 - c0] - s[c0:c1]).item() / scale
print(f"rank {rank}: columns [{c0}, {c1}) rel err H {eh:.2e} S {es:.2e}", flush=True)
ok = torch.tensor([int(eh < 1e-10 and es < 1e-10)])
dist.all_reduce(ok)
dist.barrier()
slots.close()
dist.destroy_process_group()
if rank == 0:
    print("fused scatter", "OK" if ok.item() == world else "MISMATCH")
