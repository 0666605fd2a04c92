"""Repeat test_physical_build_host_outputs_match_device and report where the
host-output build differs from the device-output build (flake hunt)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1611_00606_b200 import GpuPolicy  # noqa: E402
from paper_1611_00606_b200.physics import build_hs_physical, synthetic_system, synthetic_t_matrices  # noqa: E402

engine = sys.argv[1] if len(sys.argv) > 1 else "dmma"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sync_between = len(sys.argv) > 3 and sys.argv[3] == "sync"
system, k, kmax, g = synthetic_system(5, 2, 8, 1300, seed=5)
t_aa, t_ab, t_bb = synthetic_t_matrices(system, seed=5, nonhpd_fraction=0.2)
pol = GpuPolicy(engine=engine)
bad = 0
for r in range(reps):
    h, s, split, _, _ = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=pol)
    if sync_between:
        torch.cuda.synchronize()
    hh, sh, split_h, t, _ = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=pol, host_outputs=True)
    torch.cuda.synchronize()
    hd, sd = h.cpu().numpy().T, s.cpu().numpy().T
    for name, a, b in (("H", hh, hd), ("S", sh, sd)):
        if not np.array_equal(a, b):
            bad += 1
            diff = np.argwhere(a != b)
            upper = int(np.sum(diff[:, 0] < diff[:, 1]))
            print(f"rep {r} {name}: {len(diff)} differing entries ({upper} upper), max |d| "
                  f"{np.max(np.abs(a - b)):.3e}, first {diff[:3].tolist()}, rel {np.linalg.norm(a-b)/np.linalg.norm(b):.2e}",
                  flush=True)
print(f"{engine}: {bad} mismatches in {reps} reps (sync between calls: {sync_between})")
