"""N > 1 host logic on CPU: world_size-2 gloo processes run the sharded
build with a CPU partial builder (the oracle) injected in place of the GPU
pipeline, and the reduce-scattered block columns must equal the columns of
the full single-process result.  Also: k-point replica assignment."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_00606_b200 import Dims, ProblemSpec, SplitCounts, generate, rel_frob_error
from paper_1611_00606_b200.distributed import (
    atom_ranges, balanced_atom_groups, build_hs_sharded, kpoint_assignment, padded_columns, shard_instance,
)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cpu_partial(shard, h, s):
    from oracle import alg1

    out = alg1.build_hs_cpu(shard)
    n = shard.dims.n_g
    # row-major (ncols, n_g) tensor row j == column j of the matrix
    h[:n] = torch.from_numpy(np.ascontiguousarray(out["h"].T))
    s[:n] = torch.from_numpy(np.ascontiguousarray(out["s"].T))
    return SplitCounts(out["hpd"], out["nonhpd"]), {}


def _worker(rank, world, port, dims, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = generate(ProblemSpec(Dims(*dims), seed=3, nonhpd_fraction=0.4))
    res = build_hs_sharded(p, partial=_cpu_partial)
    q.put((rank, res.col0, res.columns("h"), res.columns("s"), res.hpd, res.nonhpd))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, (5, 6, 37)), (3, (2, 4, 20))])
def test_sharded_reduce_scatter_matches_single_process(world, dims):
    from oracle import alg1

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = generate(ProblemSpec(Dims(*dims), seed=3, nonhpd_fraction=0.4))
    full = alg1.build_hs_cpu(p)
    h_cols = np.concatenate([g[2] for g in sorted(got)], axis=1)
    s_cols = np.concatenate([g[3] for g in sorted(got)], axis=1)
    assert h_cols.shape == (dims[2], dims[2])
    assert rel_frob_error(h_cols, full["h"]) < 1e-13
    assert rel_frob_error(s_cols, full["s"]) < 1e-13
    for g in got:
        assert g[4] + g[5] == dims[0] and g[4] == full["hpd"]
    cb = padded_columns(dims[2], world) // world
    assert sorted(g[1] for g in got) == [r * cb for r in range(world)]


def test_partition_helpers():
    assert atom_ranges(32, 8) == [(4 * r, 4 * r + 4) for r in range(8)]
    assert atom_ranges(5, 2) == [(0, 3), (3, 5)]
    assert atom_ranges(1, 3) == [(0, 1), (1, 1), (1, 1)]
    assert padded_columns(8000, 8) == 8000 and padded_columns(3001, 4) == 3004
    groups = balanced_atom_groups([16, 12, 12, 12, 16, 12], 2)
    assert sorted(sum(groups, [])) == list(range(6))
    assert abs(sum([16, 12, 12, 12, 16, 12][a] for a in groups[0]) - 40) <= 4
    assert kpoint_assignment(16, 8, 3) == [3, 11]
    p = generate(ProblemSpec(Dims(4, 3, 5), seed=1))
    q = shard_instance(p, [1, 3])
    assert q.dims.n_atoms == 2 and q.a_blocks[1] is p.a_blocks[3]


def _cpu_partial_lower(shard, h, s):
    from oracle import alg1

    out = alg1.build_hs_cpu(shard)
    n = shard.dims.n_g
    # lower triangles only (the HSB_OPT_LOWER_ONLY contract); garbage above
    # the diagonal must not leak into the result
    junk = np.triu(np.full((n, n), 7.0 + 3.0j), 1)
    h[:n] = torch.from_numpy(np.ascontiguousarray((np.tril(out["h"]) + junk).T))
    s[:n] = torch.from_numpy(np.ascontiguousarray((np.tril(out["s"]) + junk).T))
    return SplitCounts(out["hpd"], out["nonhpd"]), {}


def _worker_tri(rank, world, port, dims, nb, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1611_00606_b200.distributed import build_hs_sharded_tri

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = generate(ProblemSpec(Dims(*dims), seed=4, nonhpd_fraction=0.3))
    hc, sc, cols, hpd, nonhpd = build_hs_sharded_tri(p, partial=_cpu_partial_lower, nb=nb)
    q.put((rank, hc.numpy(), sc.numpy(), cols.numpy(), hpd, nonhpd))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,nb", [(2, (5, 6, 37), 4), (3, (4, 5, 50), 8), (4, (3, 4, 23), 16)])
def test_triangle_packed_exchange_matches_single_process(world, dims, nb):
    from oracle import alg1
    from paper_1611_00606_b200.distributed import TrianglePlan

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tri, args=(r, world, port, dims, nb, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = generate(ProblemSpec(Dims(*dims), seed=4, nonhpd_fraction=0.4 - 0.1))
    full = alg1.build_hs_cpu(p)
    seen = []
    for rank, hc, sc, cols, hpd, nonhpd in got:
        assert hpd + nonhpd == dims[0]
        # row-major (local column, row) -> columns cols of the matrices
        assert rel_frob_error(hc.T, full["h"][:, cols]) < 1e-13
        assert rel_frob_error(sc.T, full["s"][:, cols]) < 1e-13
        seen += cols.tolist()
    assert sorted(seen) == list(range(dims[2]))


@pytest.mark.parametrize("n_g,world,nb", [(2000, 4, 32), (1500, 8, 16), (1200, 2, 64)])
def test_triangle_plan_moves_about_half_the_bytes(n_g, world, nb):
    # per-rank bytes of the triangle-packed exchange against a full-matrix
    # reduce-scatter ((P-1)/P N^2 complex128): (P-1)/(2P) N^2 + the tiles
    from paper_1611_00606_b200.distributed import TrianglePlan

    plan = TrianglePlan(n_g, world, nb)
    full = (world - 1) / world * n_g * n_g * 16
    worst = max(plan.bytes_per_rank(r) for r in range(world))
    model = full / 2 * (1 + 1 / world)  # RS of the triangle + upper tiles from the other ranks
    assert worst < 1.15 * model and worst < 0.85 * full
    # lower-only columns (what uplo='L' eigensolvers read): the reduce-scatter alone
    assert (world - 1) * plan.chunk * 16 < 0.6 * full
    assert sorted(torch.cat(plan.cols).tolist()) == list(range(n_g))


def _kpoint_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import alg1
    from paper_1611_00606_b200.distributed import build_kpoints

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kpts = [generate(ProblemSpec(Dims(2, 4, 15 + 3 * i), seed=100 + i)) for i in range(7)]  # ragged N_G
    mine = build_kpoints(kpts, builder=lambda p, _pol: alg1.build_hs_cpu(p))
    gathered = [None] * world
    dist.all_gather_object(gathered, sorted(mine))
    q.put((rank, {k: (v["h"], v["s"]) for k, v in mine.items()}, gathered))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_kpoint_replicas_cover_every_kpoint_once(world):
    # config C5's distribution: round-robin k-points, no
    # communication on the data path; every k-point built exactly once and
    # equal to the serial build
    from oracle import alg1

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kpoint_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    owned = sorted(k for _, res, _ in got for k in res)
    assert owned == list(range(7))
    for rank, res, gathered in got:
        assert sorted(res) == kpoint_assignment(7, world, rank)
        assert sorted(k for g in gathered for k in g) == list(range(7))
        for k, (h, s) in res.items():
            ref = alg1.build_hs_cpu(generate(ProblemSpec(Dims(2, 4, 15 + 3 * k), seed=100 + k)))
            assert np.array_equal(h, ref["h"]) and np.array_equal(s, ref["s"])
