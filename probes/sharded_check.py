"""Run under torchrun: the sharded build's column blocks must equal the
single-GPU build of the whole instance (rank 0 compares after a gather)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1611_00606_b200 import Dims, ProblemSpec, build_hs, generate, rel_frob_error  # noqa: E402
from paper_1611_00606_b200.distributed import build_hs_sharded  # noqa: E402

backend = os.environ.get("HSB_DIST_BACKEND", "nccl")
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local % torch.cuda.device_count())
dist.init_process_group(backend)
p = generate(ProblemSpec(Dims(7, 40, 523), seed=5, nonhpd_fraction=0.3))
res = build_hs_sharded(p)
blocks = [None] * dist.get_world_size()
dist.all_gather_object(blocks, (res.col0, res.columns("h"), res.columns("s")))
if dist.get_rank() == 0:
    full = build_hs(p)
    h = np.concatenate([b[1] for b in sorted(blocks, key=lambda x: x[0])], axis=1)
    s = np.concatenate([b[2] for b in sorted(blocks, key=lambda x: x[0])], axis=1)
    eh, es = rel_frob_error(h, full.h.matrix), rel_frob_error(s, full.s.matrix)
    print(f"sharded world={dist.get_world_size()} backend={backend}: rel err H {eh:.2e} S {es:.2e} "
          f"split {res.hpd}/{res.nonhpd} vs {full.split}")
    assert eh < 1e-12 and es < 1e-12 and (res.hpd, res.nonhpd) == (full.split.hpd, full.split.nonhpd)
dist.destroy_process_group()
