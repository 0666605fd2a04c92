"""C5 end-to-end pieces: per-call wall time of iter_hs_physical_kpoints over the
16 k-points, repeated, to see whether repeated calls pay a setup cost."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import c5_kpoints  # noqa: E402
from paper_1611_00606_b200 import CONFIGS, GpuPolicy, physics  # noqa: E402

c3 = CONFIGS["C3"]
system, _k0, kmax, _ = physics.synthetic_system(c3.n_atoms, 4, 10, c3.n_g, seed=0)
t_aa, t_ab, t_bb = physics.synthetic_t_matrices(system, seed=0)
kpts = c5_kpoints()
gsets = [physics.gvector_set(system.lattice, k, kmax) for k in kpts]
pol = GpuPolicy()
for n in (4, 16, 16, 16):
    t0 = time.perf_counter()
    stamps = []
    for hh, sh, _, tp, _ in physics.iter_hs_physical_kpoints(system, kpts[:n], gsets[:n], t_aa, t_ab, t_bb, pol,
                                                             depth=3):
        stamps.append(time.perf_counter() - t0)
        del hh, sh
    dt = time.perf_counter() - t0
    print(f"{n} k-points: {dt * 1e3:.1f} ms, {dt / n * 1e3:.1f} ms/k; arrivals "
          + " ".join(f"{x * 1e3:.0f}" for x in stamps), flush=True)
