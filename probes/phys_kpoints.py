"""Per-k-point wall time of physics.iter_hs_physical_kpoints (physical inputs,
H/S to pinned host memory) vs serial build_hs_physical(host_outputs=True).

    python probes/phys_kpoints.py [C3|C4] [n] [depth ...]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS  # noqa: E402
from paper_1611_00606_b200 import physics  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
depths = [int(x) for x in sys.argv[3:]] or [1, 2, 3]
d = CONFIGS[cfg]
system, k0, kmax, _ = physics.synthetic_system(d.n_atoms, 4, int(round(d.n_l ** 0.5)) - 1, d.n_g, seed=0)
t = physics.synthetic_t_matrices(system, seed=0)
rng = np.random.default_rng(17)
kpts = [k0] + [rng.uniform(-0.5, 0.5, 3) for _ in range(n - 1)]
gsets = [physics.gvector_set(system.lattice, k, kmax) for k in kpts]
imax = int(np.argmax([g.shape[0] for g in gsets]))
for depth in depths:
    for o in physics.iter_hs_physical_kpoints(system, [kpts[imax]] * (depth + 2), [gsets[imax]] * (depth + 2), *t,
                                              depth=depth):
        del o
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stamps = []
    for o in physics.iter_hs_physical_kpoints(system, kpts, gsets, *t, depth=depth):
        stamps.append(time.perf_counter() - t0)
        del o
    print(f"{cfg} depth {depth}: {stamps[-1] / n * 1e3:.1f} ms/k-point; stamps (ms):",
          [round(s * 1e3, 1) for s in stamps], "device GB in use:",
          round(torch.cuda.memory_allocated() / 1e9, 1), "reserved:", round(torch.cuda.memory_reserved() / 1e9, 1),
          flush=True)
