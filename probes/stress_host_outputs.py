"""Stress: random sequences of builds (engines, entry points, sizes, host /
device outputs, k-point pipelines, kernel-level calls) in one process; every
host-output build is compared bit for bit with a device-output build of the
same input made right before it.  Hunting a one-off S mismatch."""
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1611_00606_b200 import (Dims, GpuPolicy, ProblemSpec, build_hs, build_hs_kpoints, generate,  # noqa: E402
                                   pin_instance)
from paper_1611_00606_b200.physics import build_hs_physical, synthetic_system, synthetic_t_matrices  # noqa: E402

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 240
rng = random.Random(7)
systems = {}
bad = n = 0
t_end = time.time() + seconds
while time.time() < t_end:
    engine = rng.choice(["int8", "dmma"])
    pol = GpuPolicy(engine=engine)
    kind = rng.choice(["phys", "phys", "inst", "kpts", "kphys", "lower"])
    if kind == "phys":
        key = rng.choice([(5, 2, 8, 1300, 5), (3, 2, 6, 700, 9), (4, 2, 10, 2100, 3)])
        if key not in systems:
            sysm, k, _, g = synthetic_system(*key[:4], seed=key[4])
            systems[key] = (sysm, k, g, synthetic_t_matrices(sysm, seed=key[4], nonhpd_fraction=0.2))
        sysm, k, g, t = systems[key]
        h, s, _, _, _ = build_hs_physical(sysm, k, g, *t, policy=pol)
        torch.cuda.synchronize()
        hd, sd = h.cpu().numpy().T, s.cpu().numpy().T
        hh, sh, _, _, _ = build_hs_physical(sysm, k, g, *t, policy=pol, host_outputs=True)
        pairs = (("H", hh, hd), ("S", sh, sd))
    elif kind == "inst":
        dims = rng.choice([Dims(4, 25, 900), Dims(3, 49, 1300), Dims(6, 16, 513)])
        p = generate(ProblemSpec(dims, seed=rng.randrange(1000), nonhpd_fraction=0.3))
        if rng.random() < 0.5:
            p = pin_instance(p)
        a = build_hs(p, pol)
        b = build_hs(p, GpuPolicy(engine=engine, pinned_outputs=False))
        pairs = (("H", a.h.matrix, b.h.matrix), ("S", a.s.matrix, b.s.matrix))
    elif kind == "kphys":
        from paper_1611_00606_b200.physics import gvector_set, iter_hs_physical_kpoints
        key = (3, 2, 6, 700, 9)
        if key not in systems:
            sysm, k, _, g = synthetic_system(*key[:4], seed=key[4])
            systems[key] = (sysm, k, g, synthetic_t_matrices(sysm, seed=key[4], nonhpd_fraction=0.2))
        sysm, k0, g0, t = systems[key]
        kpts = [np.array(x) for x in [(0.0, 0.0, 0.0), (0.5, 0.25, 0.0), (0.125, -0.375, 0.25)]]
        gsets = [g0] * len(kpts)
        got = list(iter_hs_physical_kpoints(sysm, kpts, gsets, *t, policy=pol, depth=rng.choice([2, 3])))
        pairs = []
        for i, (hh, sh, *_r) in enumerate(got):
            h, s, *_ = build_hs_physical(sysm, kpts[i], gsets[i], *t, policy=pol)
            torch.cuda.synchronize()
            pairs += [(f"kph{i}H", hh, h.cpu().numpy().T), (f"kph{i}S", sh, s.cpu().numpy().T)]
    elif kind == "lower":
        from paper_1611_00606_b200 import DeviceProblem, build_hs_device
        dims = rng.choice([Dims(4, 25, 900), Dims(3, 49, 1300)])
        p = generate(ProblemSpec(dims, seed=rng.randrange(1000), nonhpd_fraction=0.3))
        dp = DeviceProblem.from_instance(p)
        hf, sf, *_ = build_hs_device(dp, policy=pol)
        hl = torch.zeros((dims.n_g + 1, dims.n_g), dtype=torch.complex128, device="cuda")
        sl = torch.zeros_like(hl)
        build_hs_device(dp, hl, sl, policy=pol, lower_only=True)
        torch.cuda.synchronize()
        n_ = dims.n_g
        mask = np.tril(np.ones((n_, n_), dtype=bool))
        a1, b1 = hf.cpu().numpy().T, hl[:n_].cpu().numpy().T
        a2, b2 = sf.cpu().numpy().T, sl[:n_].cpu().numpy().T
        pairs = (("lowH", np.where(mask, a1, 0), np.where(mask, b1, 0)),
                 ("lowS", np.where(mask, a2, 0), np.where(mask, b2, 0)))
    else:
        dims = rng.choice([Dims(3, 25, 700), Dims(2, 36, 1000)])
        ps = [generate(ProblemSpec(dims, seed=rng.randrange(1000))) for _ in range(4)]
        outs = build_hs_kpoints(ps, pol, depth=rng.choice([2, 3]))
        ref = [build_hs(q, GpuPolicy(engine=engine, pinned_outputs=False)) for q in ps]
        pairs = [(f"kp{i}H", o.h.matrix, r.h.matrix) for i, (o, r) in enumerate(zip(outs, ref))] + \
                [(f"kp{i}S", o.s.matrix, r.s.matrix) for i, (o, r) in enumerate(zip(outs, ref))]
    n += 1
    for name, x, y in pairs:
        if not np.array_equal(x, y):
            bad += 1
            d = np.argwhere(x != y)
            print(f"MISMATCH #{n} {kind} {engine} {name}: {len(d)} entries, rows {d[:,0].min()}..{d[:,0].max()} "
                  f"cols {d[:,1].min()}..{d[:,1].max()} upper {int(np.sum(d[:,0] < d[:,1]))} "
                  f"max {np.max(np.abs(x - y)):.2e} first {d[:3].tolist()}", flush=True)
print(f"{n} cases, {bad} mismatches")
