"""Fused reduce-scatter: each rank's reconstruction epilogue
writes its partial H and S straight into the owners' receive slots
(hsb_peer_out), and each owner sums its slots.  Emulated here with several
"ranks" in one process on one GPU (the slots are local allocations; on a
multi-GPU box they are CUDA-IPC-mapped peer memory, distributed.PeerSlots.group).
The owners' column blocks must equal the single-GPU build's columns."""

import numpy as np
import pytest
import torch

from paper_1611_00606_b200 import DeviceProblem, Dims, GpuPolicy, ProblemSpec, build_hs_device, generate
from paper_1611_00606_b200 import distributed as hd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_atoms,n_ranks,n_g,frac", [(6, 3, 700, 0.0), (5, 2, 513, 0.4), (4, 4, 300, 0.5)])
def test_fused_scatter_matches_single_gpu_build(n_atoms, n_ranks, n_g, frac):
    p = generate(ProblemSpec(Dims(n_atoms, 49, n_g), seed=n_atoms * 10 + n_ranks, nonhpd_fraction=frac))
    pol = GpuPolicy(engine="int8")
    full = DeviceProblem.from_instance(p)
    h, s, split, _, _ = build_hs_device(full, policy=pol)
    torch.cuda.synchronize()
    dev = full.a_stack.device
    slots = hd.PeerSlots.emulated(n_ranks, n_g, dev)
    for r, (lo, hi) in enumerate(hd.atom_ranges(n_atoms, n_ranks)):
        shard = DeviceProblem.from_instance(hd.shard_instance(p, range(lo, hi)))
        build_hs_device(shard, policy=pol, peer=slots[r], wait=False)
    torch.cuda.synchronize()
    for r in range(n_ranks):
        hb, sb = slots[r].finish()
        c0 = r * slots[r].cols
        c1 = min(c0 + slots[r].cols, n_g)
        # blocks are (cols, n_g) row-major = column-major n_g x cols
        want_h, want_s = h[c0:c1].cpu().numpy(), s[c0:c1].cpu().numpy()
        got_h, got_s = hb[: c1 - c0].cpu().numpy(), sb[: c1 - c0].cpu().numpy()
        scale = 1 + np.linalg.norm(h.cpu().numpy())
        assert np.linalg.norm(got_h - want_h) / scale < 1e-10
        assert np.linalg.norm(got_s - want_s) / scale < 1e-10
        if c1 - c0 < slots[r].cols:  # padding columns stay zero
            assert torch.count_nonzero(hb[c1 - c0:]).item() == 0


def test_peer_output_needs_the_int8_engine():
    from paper_1611_00606_b200 import InputError  # noqa: F401

    p = generate(ProblemSpec(Dims(2, 9, 77), seed=3))
    dp = DeviceProblem.from_instance(p)
    slots = hd.PeerSlots.emulated(2, 77, dp.a_stack.device)
    with pytest.raises(RuntimeError, match="INT8"):
        build_hs_device(dp, policy=GpuPolicy(engine="dmma"), peer=slots[0])


@pytest.mark.parametrize("n_slots,cols,n_g", [(1, 5, 33), (3, 17, 257), (8, 64, 1000)])
def test_sum_slots_kernel_is_rank_ordered_sum(n_slots, cols, n_g):
    # hsb_sum_slots (the owner's reduction of the fused scatter) against the
    # same rank-ordered sum in torch: bitwise
    g = torch.Generator(device="cuda").manual_seed(n_slots * 1000 + cols)
    recv = torch.randn((n_slots, cols, n_g), dtype=torch.complex128, device="cuda", generator=g)
    slots = hd.PeerSlots(n_slots, 0, cols, n_g, recv, recv.clone(), [], [])
    hb, sb = slots.finish()
    want = recv[0].clone()
    for r in range(1, n_slots):
        want += recv[r]
    torch.cuda.synchronize()
    assert torch.equal(hb, want) and torch.equal(sb, want)


def test_sum_slots_rejects_bad_dimensions():
    import ctypes

    from paper_1611_00606_b200 import DimensionError, _lib

    lib = _lib.load()
    ctx = _lib.context(0)
    buf = torch.zeros(8, dtype=torch.complex128, device="cuda")
    for n_slots, stride, count in ((0, 4, 4), (2, 3, 4), (2, 4, -1)):
        with pytest.raises(DimensionError):
            _lib.check(lib.hsb_sum_slots(ctx, None, ctypes.c_void_p(buf.data_ptr()), n_slots, stride, count,
                                         ctypes.c_void_p(buf.data_ptr())), ctx)
