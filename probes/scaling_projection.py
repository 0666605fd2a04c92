"""Projected atom-sharded strong scaling from one GPU.

No multi-GPU box exists for this run, so the N > 1 curve is projected from
measured pieces: the rank-local build of a P-way atom shard (N_A / P atoms,
full N_G: every rank still produces partial N_G x N_G H and S, and the INT8
engine's CRT reconstructs all of them) is timed on this B200 with CUDA
events, and the reduce-scatter of H and S is modelled at the guide's measured
NVLink bus bandwidth (B200_PROFILING.md: 725 GB/s 8-rank all-reduce bus
bandwidth).  Per-rank bytes: (P-1)/P x N_G^2 x 16 per matrix (full), or half
that when the lower triangles are reduce-scattered (distributed.py
triangle-packed path).  S's reduce-scatter overlaps the H contraction
(distributed.build_hs_sharded_device), so only H's is exposed.

    python probes/scaling_projection.py [C3 C4] > profiles/scaling_projection_r02.jsonl
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1611_00606_b200 import CONFIGS, DeviceProblem, GpuPolicy, ProblemSpec, build_hs_device, generate  # noqa: E402
from paper_1611_00606_b200 import _lib, total_model_flops  # noqa: E402
from paper_1611_00606_b200.distributed import shard_instance  # noqa: E402

BUS_GBS = 725.0
cfgs = sys.argv[1:] or ["C3", "C4"]
for name in cfgs:
    dims = CONFIGS[name]
    p = generate(ProblemSpec(dims, seed=0))
    n_g = dims.n_g
    flops = total_model_flops(dims, 0)
    base = None
    for P in (1, 2, 4, 8):
        shard = shard_instance(p, range(dims.n_atoms // P))
        dp = DeviceProblem.from_instance(shard)
        h = torch.empty((n_g, n_g), dtype=torch.complex128, device="cuda")
        s = torch.empty_like(h)
        pol = GpuPolicy()
        reps = 10 if name == "C3" else 3
        for _ in range(2):
            build_hs_device(dp, h, s, pol)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            t = build_hs_device(dp, h, s, pol)[3]
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        rs_full = (P - 1) / P * n_g * n_g * 16 / (BUS_GBS * 1e9) * 1e3
        rs_tri = rs_full / 2
        t_full = ms + rs_full  # S's reduce-scatter hidden behind H; H's exposed
        t_tri = ms + rs_tri
        if P == 1:
            base = ms
        rec = {"config": name, "P": P, "atoms_per_rank": dims.n_atoms // P, "n_g": n_g,
               "rank_build_ms": ms, "h_core_ms": t["h_core"] * 1e3, "s_core_ms": t["s_core"] * 1e3,
               "rs_h_ms_full": rs_full, "rs_h_ms_triangle": rs_tri,
               "projected_ms_full_rs": t_full, "projected_ms_triangle_rs": t_tri,
               "speedup_full_rs": base / t_full, "speedup_triangle_rs": base / t_tri,
               "projected_tflops_triangle_rs": flops / (t_tri * 1e-3) / 1e12}
        print(json.dumps(rec), flush=True)
        del dp, h, s
        _lib.trim_all()
        torch.cuda.empty_cache()
