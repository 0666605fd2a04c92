"""The N > 1 paths with real per-rank GPU builds (world sizes 2 and 3).

One GPU is available, so the ranks are processes sharing cuda:0, joined by a
gloo process group (host-side collectives: no rank's kernel ever waits on
another's).  Each rank builds the partial H/S of its atom shard on the GPU
(the single-GPU pipeline) and

* ``nccl`` path: ``build_hs_sharded`` -- partial into padded (ncols, N_G)
  buffers, ``reduce_scatter_block_columns`` (gloo here, NCCL on a box);
* ``tri`` path: ``build_hs_sharded_tri`` -- lower-triangle partials
  (HSB_OPT_LOWER_ONLY), the triangle-packed reduce-scatter and the tile
  all-to-all into block-cyclic columns;
* ``fused`` path: ``build_hs_sharded_fused`` -- the INT8 engine's CRT epilogue
  stores every element into its owner's receive slot (CUDA-IPC peer memory),
  owners sum their slots; run for 2 steps so the slot reuse is exercised;

and the column blocks are compared with the CPU oracle (oracle/alg1.py) of
the whole instance.  Basis: linearity over atoms (PAPER.md:303-313,
pkg/tests/test_reference.py:141-152).
"""

import os
import socket

import numpy as np
import pytest

from paper_1611_00606_b200 import Dims, ProblemSpec, generate, rel_frob_error

pytestmark = pytest.mark.gpu

DIMS = (6, 49, 1100)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_1611_00606_b200 import DeviceProblem, GpuPolicy
    from paper_1611_00606_b200 import distributed as hd

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p = generate(ProblemSpec(Dims(*DIMS), seed=9, nonhpd_fraction=0.3))
        pol = GpuPolicy()
        if mode == "nccl":
            res = hd.build_hs_sharded(p, pol)
            blocks = (res.col0, res.columns("h"), res.columns("s"), res.hpd, res.nonhpd)
        elif mode == "tri":  # lower-triangle partials, triangle-packed exchange, block-cyclic columns
            hc, sc, cols, hpd, nonhpd = hd.build_hs_sharded_tri(p, pol, nb=64)
            blocks = (cols.cpu().numpy(), np.asfortranarray(hc.cpu().numpy().T),
                      np.asfortranarray(sc.cpu().numpy().T), hpd, nonhpd)
        else:
            slots = hd.PeerSlots.group(p.dims.n_g, dev)
            lo, hi = hd.atom_ranges(p.dims.n_atoms, world)[rank]
            dp = hd_dp = DeviceProblem.from_instance(hd.shard_instance(p, range(lo, hi)))
            for _ in range(2):  # the second step rewrites the slots after the owners summed them
                hb, sb = hd.build_hs_sharded_fused(hd_dp, slots, pol)
            torch.cuda.synchronize()
            c0 = rank * slots.cols
            c1 = min(c0 + slots.cols, p.dims.n_g)
            h = np.asfortranarray(hb[: c1 - c0].cpu().numpy().T)
            s = np.asfortranarray(sb[: c1 - c0].cpu().numpy().T)
            del dp
            slots.close()
            blocks = (c0, h, s, -1, -1)
        q.put((rank, *blocks))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # noqa: BLE001 -- report to the parent
        q.put((rank, "error", repr(exc)))
        raise


def _kpoint_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_1611_00606_b200 import GpuPolicy
    from paper_1611_00606_b200 import distributed as hd

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        kpts = [generate(ProblemSpec(Dims(3, 25, 300 + 37 * i), seed=40 + i, nonhpd_fraction=0.3)) for i in range(5)]
        mine = hd.build_kpoints(kpts, GpuPolicy())
        q.put((rank, {k: (o.h.matrix, o.s.matrix) for k, o in mine.items()}))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # noqa: BLE001 -- report to the parent
        q.put((rank, "error", repr(exc)))
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_kpoint_replicas_on_gpu_match_oracle(world):
    # config C5's k-point replicas: each rank builds its round-robin share on
    # the GPU, no communication; every k-point once, each against the oracle
    import torch.multiprocessing as mp

    from oracle import alg1

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kpoint_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    errors = [g for g in got if isinstance(g[1], str) and g[1] == "error"]
    assert not errors, errors
    assert all(pr.exitcode == 0 for pr in procs)
    assert sorted(k for _, res in got for k in res) == list(range(5))
    for _, res in got:
        for k, (h, s) in res.items():
            ref = alg1.build_hs_cpu(generate(ProblemSpec(Dims(3, 25, 300 + 37 * k), seed=40 + k, nonhpd_fraction=0.3)))
            assert rel_frob_error(h, ref["h"]) < 1e-14 and rel_frob_error(s, ref["s"]) < 1e-14


@pytest.mark.parametrize("mode", ["nccl", "fused", "tri"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gpu_ranks_match_oracle(world, mode):
    import torch.multiprocessing as mp

    from oracle import alg1

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    errors = [g for g in got if isinstance(g[1], str) and g[1] == "error"]
    assert not errors, errors
    assert all(pr.exitcode == 0 for pr in procs)
    p = generate(ProblemSpec(Dims(*DIMS), seed=9, nonhpd_fraction=0.3))
    full = alg1.build_hs_cpu(p)
    got.sort(key=lambda g: g[0])
    h_cols = np.concatenate([g[2] for g in got], axis=1)
    s_cols = np.concatenate([g[3] for g in got], axis=1)
    assert h_cols.shape == (DIMS[2], DIMS[2])
    if mode == "tri":  # block-cyclic ownership: put the columns back in order
        order = np.argsort(np.concatenate([g[1] for g in got]))
        h_cols, s_cols = h_cols[:, order], s_cols[:, order]
    eh, es = rel_frob_error(h_cols, full["h"]), rel_frob_error(s_cols, full["s"])
    print(f"world {world} {mode}: rel err H {eh:.2e} S {es:.2e}")
    assert eh < 1e-14 and es < 1e-14
    if mode in ("nccl", "tri"):
        assert all(g[4] == full["hpd"] and g[4] + g[5] == DIMS[0] for g in got)
