"""Which of the DMMA physical builds is wrong when device- and host-output
builds of the same input differ?  Runs device / host(streamed) / host(staged)
/ device builds of one input in a loop, each compared with the oracle-free
majority."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1611_00606_b200 import GpuPolicy  # noqa: E402
from paper_1611_00606_b200.physics import build_hs_physical, synthetic_system, synthetic_t_matrices  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
import os as _os  # noqa: E402
cfgs = [(4, 2, 10, 2100, 3), (5, 2, 8, 1300, 5), (3, 2, 6, 700, 9)]
if _os.environ.get("STRESS_CFGS") == "lmax":  # lmax 10 at small N_G, lmax 6/8 at large N_G
    cfgs = [(4, 2, 10, 700, 3), (4, 2, 8, 2100, 5), (4, 2, 6, 2100, 9)]
data = {}
for c in cfgs:
    sysm, k, _, g = synthetic_system(*c[:4], seed=c[4])
    data[c] = (sysm, k, g, synthetic_t_matrices(sysm, seed=c[4], nonhpd_fraction=0.2))
pol = GpuPolicy(engine="dmma")
pol_staged = GpuPolicy(engine="dmma", pinned_outputs=False)
import os, time  # noqa: E401,E402
warm = os.environ.get("STRESS_WARM", "")
if warm == "sleep":
    time.sleep(10)
elif warm == "dmma700":  # 10 s of DMMA builds of another config first
    t_end = time.time() + 10
    c = cfgs[2]
    while time.time() < t_end:
        build_hs_physical(data[c][0], data[c][1], data[c][2], *data[c][3], policy=pol)
elif warm == "gemm":  # 10 s of cuBLAS-free GPU load (torch elementwise)
    x = torch.randn(1 << 26, device="cuda", dtype=torch.float64)
    t_end = time.time() + 10
    while time.time() < t_end:
        x = x * 1.0000001 + 1e-9
    torch.cuda.synchronize()
elif warm == "fullpass":  # every build type at every config once (all allocations grown)
    for c in cfgs:
        sysm, k, g, t = data[c]
        build_hs_physical(sysm, k, g, *t, policy=pol)
        build_hs_physical(sysm, k, g, *t, policy=pol, host_outputs=True)
        build_hs_physical(sysm, k, g, *t, policy=pol_staged, host_outputs=True)
    torch.cuda.synchronize()
    time.sleep(2)
elif warm == "dmma2100once":
    c = cfgs[0]
    build_hs_physical(data[c][0], data[c][1], data[c][2], *data[c][3], policy=pol)
    torch.cuda.synchronize()
    time.sleep(5)
bad = 0
for r in range(reps):
    for c in cfgs:
        sysm, k, g, t = data[c]
        outs = []
        h, s, *_ = build_hs_physical(sysm, k, g, *t, policy=pol)
        torch.cuda.synchronize()
        outs.append(("dev1", h.cpu().numpy().T, s.cpu().numpy().T))
        hh, sh, *_ = build_hs_physical(sysm, k, g, *t, policy=pol, host_outputs=True)
        outs.append(("host", hh, sh))
        hh2, sh2, *_ = build_hs_physical(sysm, k, g, *t, policy=pol_staged, host_outputs=True)
        outs.append(("staged", hh2, sh2))
        h, s, *_ = build_hs_physical(sysm, k, g, *t, policy=pol)
        torch.cuda.synchronize()
        outs.append(("dev2", h.cpu().numpy().T, s.cpu().numpy().T))
        for mi, m in ((1, "H"), (2, "S")):
            ref = outs[0][mi]
            same = [np.array_equal(o[mi], ref) for o in outs]
            if not all(same):
                bad += 1
                # the odd one out: compare each with all others
                votes = [sum(np.array_equal(o[mi], p[mi]) for p in outs) for o in outs]
                odd = [o[0] for o, v in zip(outs, votes) if v == min(votes)]
                d = np.argwhere(outs[int(np.argmin(votes))][mi] != outs[int(np.argmax(votes))][mi])
                print(f"rep {r} cfg {c[3]} {m}: agreement {votes} odd {odd}; {len(d)} entries, first {d[:3].tolist()}",
                      flush=True)
                lo = d[d[:, 0] >= d[:, 1]]
                good, badm = outs[int(np.argmax(votes))][mi], outs[int(np.argmin(votes))][mi]
                for (i, j) in lo[:64]:
                    print(f"   ({i},{j}) tile ({i // 64},{j // 64}) in-tile ({i % 64},{j % 64}) good {good[i, j]:.6e} "
                          f"bad {badm[i, j]:.6e}", flush=True)
print(f"{reps} reps x {len(cfgs)} cfgs: {bad} disagreements")
