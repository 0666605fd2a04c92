"""Locate INT8-engine deviations on a long her2k (k=40000, n=130): where are the
largest elementwise errors against the DMMA engine?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_1611_00606_b200 import GpuPolicy, KernelKind, run_partitioned  # noqa: E402

for k, n, bits in [(40000, 130, 0), (40000, 130, 53), (17000, 260, 0), (40000, 300, 0), (2000, 130, 55)]:
    rng = np.random.default_rng(k + n)
    z = np.asfortranarray(rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)))
    b = np.asfortranarray(rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)))
    c1 = np.zeros((n, n), complex, order="F")
    c2 = np.zeros((n, n), complex, order="F")
    run_partitioned(KernelKind.HER2K, (1.0, z, b, 0.0, c1), GpuPolicy(engine="int8", int8_bits=bits))
    run_partitioned(KernelKind.HER2K, (1.0, z, b, 0.0, c2), GpuPolicy(engine="dmma"))
    d = np.abs(np.tril(c1 - c2))
    i, j = np.unravel_index(np.argmax(d), d.shape)
    bad = np.argwhere(d > 1e-9 * np.abs(c2).max())
    print(f"k={k} n={n} bits={bits}: rel {np.linalg.norm(c1 - c2) / np.linalg.norm(c2):.2e} max at ({i},{j}) "
          f"{d[i, j]:.3e} vs |c| {abs(c2[i, j]):.3e}; bad elements {len(bad)} rows {sorted(set(bad[:, 0]))[:10]} "
          f"cols {sorted(set(bad[:, 1]))[:10]}", flush=True)
