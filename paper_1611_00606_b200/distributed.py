"""Multi-GPU H/S generation: atom sharding + reduce-scatter, and k-point replicas.

No reference counterpart (the reference is single-process);
this is the north star's part (3) and SURVEY.md section 8(e):

* H and S are sums over atoms (Eqs. 6-7; linearity is tested in
  the reference at pkg/tests/test_reference.py:141-152), so each rank builds
  the partial H/S of its own atoms on its own GPU — the full single-GPU
  pipeline (Loop 1, Cholesky routing, Loop 2, fused H and S contractions) —
  and one reduce-scatter per matrix sums the partials and leaves every rank
  the 1-D block of columns an eigensolver consumes.  Columns are padded to a
  multiple of the world size so each rank's block is one contiguous chunk of
  the column-major matrix (a row-major (ncols, n_g) tensor).
* Independent k-points are replicas: rank r builds k-points r, r+P, ... with
  no communication.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on the GPU
box; gloo in the CPU tests, which inject a CPU partial builder).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .hs_types import Dims
from .instances import ProblemInstance


def atom_ranges(n_atoms: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, size-balanced atom ranges (equal-cost atoms for nonhpd = 0)."""
    base, extra = divmod(n_atoms, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def balanced_atom_groups(costs, world: int) -> list[list[int]]:
    """LPT partition of atoms by cost (HPD rows ~12 N_G^2, non-HPD ~16 N_G^2
    per row in the model of SURVEY.md 8e); groups keep ascending atom order."""
    bins = [[] for _ in range(world)]
    load = [0.0] * world
    for a in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda j: (load[j], j))
        bins[r].append(a)
        load[r] += costs[a]
    return [sorted(b) for b in bins]


def shard_instance(p, atoms) -> ProblemInstance:
    """View of ``p`` restricted to the given atoms (no copies of the blocks)."""
    atoms = list(atoms)
    q = ProblemInstance(Dims(max(1, len(atoms)), p.dims.n_l, p.dims.n_g))
    for name in ("a_blocks", "b_blocks", "t_aa", "t_ab", "t_bb", "u_norms"):
        setattr(q, name, [getattr(p, name)[a] for a in atoms])
    return q


def padded_columns(n_g: int, world: int) -> int:
    return -(-n_g // world) * world


def reduce_scatter_block_columns(full, block, group=None) -> None:
    """block <- this rank's column block of sum_ranks(full).

    ``full`` is a row-major (ncols, n_g) complex128 tensor = column-major
    n_g x ncols matrix; ``block`` is (ncols / world, n_g).  Complex sums are
    float64 sums over interleaved (re, im), so the real view is reduced.
    """
    import torch
    import torch.distributed as dist

    if full.is_cuda and dist.get_backend(group) == "gloo":
        # debugging path (several ranks sharing one GPU): gloo reduces host copies
        host = torch.empty_like(block, device="cpu")
        dist.reduce_scatter_tensor(torch.view_as_real(host), torch.view_as_real(full.cpu()), op=dist.ReduceOp.SUM,
                                   group=group)
        block.copy_(host)
        return
    dist.reduce_scatter_tensor(torch.view_as_real(block), torch.view_as_real(full), op=dist.ReduceOp.SUM,
                               group=group)


@dataclass
class ShardedResult:
    h_block: object      # torch (cols_per_rank, n_g): columns [col0, col0 + cols) of H
    s_block: object
    col0: int
    n_g: int
    hpd: int             # summed over ranks
    nonhpd: int
    timings: dict

    def columns(self, which: str = "h") -> np.ndarray:
        """Host copy of the block as an n_g x cols column-major numpy array
        (padding columns beyond n_g removed)."""
        t = self.h_block if which == "h" else self.s_block
        cols = max(0, min(t.shape[0], self.n_g - self.col0))
        return np.asfortranarray(t[:cols].cpu().numpy().T)


def build_hs_sharded(p, policy=None, group=None, partial=None) -> ShardedResult:
    """Atom-sharded H/S build across the ranks of ``group``.

    Every rank passes the same full instance ``p`` (or at least the blocks of
    its own atoms).  ``partial(shard, h, s)`` fills the rank's partial H/S
    (row-major (ncols, n_g) tensors, pad columns zero) and returns
    (SplitCounts, timings); by default it is the GPU pipeline
    (``pipeline.build_hs_into``).  Returns this rank's block of columns.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_g = int(p.dims.n_g)
    ncols = padded_columns(n_g, world)
    lo, hi = atom_ranges(int(p.dims.n_atoms), world)[rank]
    if partial is None:
        from .pipeline import build_hs_into

        dev = torch.device("cuda", torch.cuda.current_device())

        def partial(shard, h, s):
            split, t, _ = build_hs_into(shard, h, s, policy)
            return split, t
    else:
        dev = torch.device("cpu")
    h = torch.zeros((ncols, n_g), dtype=torch.complex128, device=dev)
    s = torch.zeros_like(h)
    t0 = time.perf_counter()
    if hi > lo:
        split, timings = partial(shard_instance(p, range(lo, hi)), h, s)
        counts = [split.hpd, split.nonhpd]
    else:  # more ranks than atoms: contribute zeros
        timings, counts = {}, [0, 0]
    hb = torch.empty((ncols // world, n_g), dtype=torch.complex128, device=dev)
    sb = torch.empty_like(hb)
    reduce_scatter_block_columns(h, hb, group)
    reduce_scatter_block_columns(s, sb, group)
    c = torch.tensor(counts, dtype=torch.int64,
                     device=dev if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    dist.all_reduce(c, group=group)
    timings = dict(timings)
    timings["sharded_wall"] = time.perf_counter() - t0
    return ShardedResult(hb, sb, rank * (ncols // world), n_g, int(c[0]), int(c[1]), timings)


def build_hs_sharded_device(dp, h, s, hb, sb, policy=None, group=None, comm_stream=None):
    """One atom-sharded step on device-resident inputs with S's reduce-scatter
    overlapping the H contraction: the library records an event when S is
    final, a communication stream waits on it and reduce-scatters S while the
    compute stream runs Loop 2 and H; H's reduce-scatter follows on the
    compute stream.  ``dp`` holds this rank's atoms; h, s are (ncols, n_g)
    partial buffers, hb, sb this rank's (ncols / world, n_g) column blocks."""
    import torch

    from .pipeline import build_hs_device

    dev = h.device
    compute = torch.cuda.current_stream(dev)
    comm = comm_stream if comm_stream is not None else torch.cuda.Stream(device=dev)
    s_ready = torch.cuda.Event()
    build_hs_device(dp, h, s, policy, s_ready=s_ready, wait=False)
    with torch.cuda.stream(comm):
        comm.wait_event(s_ready)
        reduce_scatter_block_columns(s, sb, group)
    reduce_scatter_block_columns(h, hb, group)
    compute.wait_stream(comm)
    return hb, sb


class TrianglePlan:
    """Index maps of the triangle-packed exchange ("triangle-packed
    reduce-scatter halves the bytes").

    Columns are distributed 1-D block-cyclically -- blocks of ``nb`` columns,
    block j owned by rank j mod P, the layout ScaLAPACK-style eigensolvers
    consume -- which balances the lower triangle across owners.  Each rank's
    partial H / S is built as a lower triangle only (HSB_OPT_LOWER_ONLY: the
    epilogue writes no mirror), and then

    1. reduce-scatter: every owner receives the summed lower trapezoid of each
       of its blocks (rows from the block's first column down), packed in
       owner order and padded to the largest owner's share;
    2. all-to-all: the strict upper part of an owner's columns is the
       conjugate transpose of lower-trapezoid rows held by the owners of
       earlier blocks: each sends the nb x nb tiles its owners need;
    3. the upper halves of the diagonal blocks are mirrored locally.

    Bytes per rank: (P-1)/P * N^2/2 (reduce-scatter, half the full-matrix
    form) + about N^2 / (2P) * (P-1)/P (tiles), complex128.

    Index tensors are built once per (n_g, P, nb) on ``device``; element (r, c)
    of a partial buffer (a row-major (>= n_g + 1, n_g) tensor whose row n_g is
    zero, the padding target) is at c * n_g + r; of the local result (a
    row-major (len(cols), n_g) tensor) at lc * n_g + r, lc the local column.
    """

    def __init__(self, n_g: int, world: int, nb: int = 64, device="cpu"):
        import torch

        self.n_g, self.world, self.nb = n_g, world, nb
        nblk = -(-n_g // nb)
        self.blocks = [list(range(q, nblk, world)) for q in range(world)]
        rng = lambda j: (j * nb, min((j + 1) * nb, n_g))  # noqa: E731
        self.cols = [torch.cat([torch.arange(*rng(j)) for j in bl]) if bl else torch.zeros(0, dtype=torch.long)
                     for bl in self.blocks]
        local_of = torch.empty(n_g, dtype=torch.long)  # local column of a global column on its owner
        for q in range(world):
            local_of[self.cols[q]] = torch.arange(len(self.cols[q]))

        def trapezoid(j):  # (r, c) of block j's lower trapezoid, column by column
            c0, c1 = rng(j)
            c = torch.arange(c0, c1).repeat_interleave(n_g - c0)
            r = torch.arange(c0, n_g).repeat(c1 - c0)
            return r, c

        send, recv, lens = [], [], []
        for q in range(world):
            rs, cs = zip(*[trapezoid(j) for j in self.blocks[q]]) if self.blocks[q] else ((), ())
            r = torch.cat(rs) if rs else torch.zeros(0, dtype=torch.long)
            c = torch.cat(cs) if cs else torch.zeros(0, dtype=torch.long)
            send.append(c * n_g + r)
            recv.append(local_of[c] * n_g + r)
            lens.append(len(r))
        self.chunk = max(lens) if lens else 0
        pad = n_g * n_g  # row n_g of the partial buffer (zeros)
        self.send_idx = torch.cat([torch.cat([x, torch.full((self.chunk - len(x),), pad, dtype=torch.long)])
                                   for x in send]).to(device)
        self.recv_pos = [x.to(device) for x in recv]
        # tiles: owner q2 of block j2 sends rows of block j (j > j2, owned by q) of its
        # block j2's columns; q writes their conjugates at (column r, row c)
        self.tile_send, self.tile_split_out = [], []
        self.tile_recv, self.tile_split_in = [], []
        for me in range(world):
            out_idx, out_split = [], []
            for q in range(world):
                idx = []
                for j2 in self.blocks[me]:
                    c0, c1 = rng(j2)
                    for j in self.blocks[q]:
                        if j <= j2:
                            continue
                        r0, r1 = rng(j)
                        c = torch.arange(c0, c1).repeat_interleave(r1 - r0)
                        r = torch.arange(r0, r1).repeat(c1 - c0)
                        idx.append(local_of[c] * n_g + r)
                flat = torch.cat(idx) if idx else torch.zeros(0, dtype=torch.long)
                out_idx.append(flat)
                out_split.append(len(flat))
            self.tile_send.append(torch.cat(out_idx).to(device))
            self.tile_split_out.append(out_split)
        for me in range(world):
            in_pos, in_split = [], []
            for q2 in range(world):
                pos = []
                for j2 in self.blocks[q2]:
                    c0, c1 = rng(j2)
                    for j in self.blocks[me]:
                        if j <= j2:
                            continue
                        r0, r1 = rng(j)
                        c = torch.arange(c0, c1).repeat_interleave(r1 - r0)
                        r = torch.arange(r0, r1).repeat(c1 - c0)
                        pos.append(local_of[r] * n_g + c)  # element (c, r) of column r
                flat = torch.cat(pos) if pos else torch.zeros(0, dtype=torch.long)
                in_pos.append(flat)
                in_split.append(len(flat))
            self.tile_recv.append(torch.cat(in_pos).to(device))
            self.tile_split_in.append(in_split)
        # diagonal blocks: (r < c) of column c = conj of (c, r), both local
        self.diag_dst, self.diag_src = [], []
        for q in range(world):
            dst, src = [], []
            for j in self.blocks[q]:
                c0, c1 = rng(j)
                c, r = torch.meshgrid(torch.arange(c0, c1), torch.arange(c0, c1), indexing="ij")
                m = r < c
                dst.append(local_of[c[m]] * n_g + r[m])
                src.append(local_of[r[m]] * n_g + c[m])
            self.diag_dst.append((torch.cat(dst) if dst else torch.zeros(0, dtype=torch.long)).to(device))
            self.diag_src.append((torch.cat(src) if src else torch.zeros(0, dtype=torch.long)).to(device))

    def bytes_per_rank(self, rank: int) -> int:
        """complex128 bytes that reach this rank over the links: its
        reduce-scatter share plus the tiles received from other ranks."""
        tiles = sum(x for q, x in enumerate(self.tile_split_in[rank]) if q != rank)
        return 16 * ((self.world - 1) * self.chunk + tiles)


def triangle_reduce_scatter(partial, plan: TrianglePlan, group=None, upper: bool = True):
    """This rank's columns (plan.cols[rank], block-cyclic) of sum_ranks(partial),
    FULL Hermitian, as a row-major (len(cols), n_g) complex128 tensor
    (``upper=False``: the lower trapezoids only -- all an uplo='L' Hermitian
    eigensolver reads -- skipping the tile exchange: half a full reduce-scatter's bytes).

    ``partial`` is a row-major (>= n_g + 1, n_g) complex128 tensor holding this
    rank's partial matrix as a lower triangle (rows >= column of each column;
    the upper triangle is never read) and zeros in row n_g."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n_g = plan.n_g
    flat = partial.reshape(-1)
    send = flat[plan.send_idx.to(flat.device)]
    stage = partial.is_cuda and dist.get_backend(group) == "gloo"  # ranks sharing a GPU in tests
    if stage:
        send = send.cpu()
    recv = torch.empty(plan.chunk, dtype=send.dtype, device=send.device)
    dist.reduce_scatter_tensor(torch.view_as_real(recv), torch.view_as_real(send), op=dist.ReduceOp.SUM, group=group)
    dev = partial.device
    local = torch.zeros((len(plan.cols[rank]), n_g), dtype=partial.dtype, device=dev)
    lf = local.view(-1)
    pos = plan.recv_pos[rank].to(dev)
    lf[pos] = recv[: len(pos)].to(dev)
    if not upper:
        return local
    tsend = lf[plan.tile_send[rank].to(dev)]
    if stage:
        tsend = tsend.cpu()
    trecv = torch.empty(sum(plan.tile_split_in[rank]), dtype=local.dtype, device=tsend.device)
    dist.all_to_all_single(torch.view_as_real(trecv), torch.view_as_real(tsend),
                           output_split_sizes=plan.tile_split_in[rank], input_split_sizes=plan.tile_split_out[rank],
                           group=group)
    lf[plan.tile_recv[rank].to(dev)] = trecv.to(dev).conj()
    lf[plan.diag_dst[rank].to(dev)] = lf[plan.diag_src[rank].to(dev)].conj()
    return local


def build_hs_sharded_tri(p, policy=None, group=None, partial=None, nb: int = 64, plan=None):
    """Atom-sharded H/S build with the triangle-packed exchange: this rank's
    block-cyclic columns (``plan.cols[rank]``) of H and S.  ``partial(shard,
    h, s)`` fills lower-triangle partial sums (default: the GPU pipeline with
    HSB_OPT_LOWER_ONLY).  Returns (ShardedResult-like tuple) h_cols, s_cols,
    global column indices, split counts summed over ranks."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n_g = int(p.dims.n_g)
    lo, hi = atom_ranges(int(p.dims.n_atoms), world)[rank]
    if partial is None:
        from .pipeline import build_hs_into

        dev = torch.device("cuda", torch.cuda.current_device())

        def partial(shard, h, s):
            split, t, _ = build_hs_into(shard, h, s, policy, lower_only=True)
            return split, t
    else:
        dev = torch.device("cpu")
    if plan is None:
        plan = TrianglePlan(n_g, world, nb, device=dev)
    h = torch.zeros((n_g + 1, n_g), dtype=torch.complex128, device=dev)
    s = torch.zeros_like(h)
    counts = [0, 0]
    if hi > lo:
        split, _t = partial(shard_instance(p, range(lo, hi)), h, s)
        counts = [split.hpd, split.nonhpd]
    hc = triangle_reduce_scatter(h, plan, group)
    sc = triangle_reduce_scatter(s, plan, group)
    c = torch.tensor(counts, dtype=torch.int64,
                     device=dev if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    dist.all_reduce(c, group=group)
    return hc, sc, plan.cols[rank], int(c[0]), int(c[1])


class PeerSlots:
    """Receive slots for the fused reduce-scatter (hsb_peer_out).

    Rank q owns columns [q * cols, (q + 1) * cols) and holds ``h_recv`` and
    ``s_recv``: (n_ranks, cols, n_g) complex128 tensors; slot r receives rank
    r's partial H / S for those columns, written over NVLink by rank r's
    reconstruction epilogue (the INT8 engine's CRT kernel stores each
    element straight into its owner's slot).  After every rank's build has
    completed, the owner's block is the sum of its slots (``finish``).

    ``PeerSlots.group(...)`` wires real ranks (one process per GPU: CUDA IPC
    handles exchanged through torch.distributed); ``PeerSlots.emulated(...)``
    wires several "ranks" inside one process on one device (tests).
    """

    def __init__(self, n_ranks, rank, cols, n_g, h_recv, s_recv, h_ptrs, s_ptrs, opened=()):
        import torch

        self.n_ranks, self.rank, self.cols, self.n_g = n_ranks, rank, cols, n_g
        self.h_recv, self.s_recv = h_recv, s_recv
        dev = h_recv.device
        self._h_tab = torch.tensor(h_ptrs, dtype=torch.int64, device=dev)
        self._s_tab = torch.tensor(s_ptrs, dtype=torch.int64, device=dev)
        self._opened = list(opened)

    @staticmethod
    def alloc(n_ranks, n_g, device):
        import torch

        cols = -(-n_g // n_ranks)
        shape = (n_ranks, cols, n_g)
        return (torch.zeros(shape, dtype=torch.complex128, device=device),
                torch.zeros(shape, dtype=torch.complex128, device=device), cols)

    @classmethod
    def emulated(cls, n_ranks, n_g, device):
        """All ranks in this process: returns one PeerSlots per rank."""
        bufs = [cls.alloc(n_ranks, n_g, device) for _ in range(n_ranks)]
        hp = [b[0].data_ptr() for b in bufs]
        sp = [b[1].data_ptr() for b in bufs]
        return [cls(n_ranks, r, bufs[r][2], n_g, bufs[r][0], bufs[r][1], hp, sp) for r in range(n_ranks)]

    @classmethod
    def group(cls, n_g, device, group=None):
        """One process per GPU: allocate this rank's slots, exchange CUDA IPC
        handles with every rank of ``group`` and open the peers' slots."""
        import ctypes

        import torch.distributed as dist

        from . import _lib

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        h_recv, s_recv, cols = cls.alloc(world, n_g, device)
        lib = _lib.load()
        ctx = _lib.context(device.index if device.index is not None else 0)

        def handle(t):
            buf = ctypes.create_string_buffer(64)
            _lib.check(lib.hsb_ipc_handle(ctx, ctypes.c_void_p(t.data_ptr()), buf), ctx)
            return buf.raw

        mine = (handle(h_recv), handle(s_recv))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        hp, sp, opened = [], [], []
        for q, (hh, sh) in enumerate(allh):
            if q == rank:
                hp.append(h_recv.data_ptr())
                sp.append(s_recv.data_ptr())
                continue
            for raw, lst in ((hh, hp), (sh, sp)):
                ptr = ctypes.c_void_p()
                _lib.check(lib.hsb_ipc_open(ctx, raw, ctypes.byref(ptr)), ctx)
                lst.append(ptr.value)
                opened.append(ptr.value)
        return cls(world, rank, cols, n_g, h_recv, s_recv, hp, sp, opened)

    def struct(self):
        from . import _lib

        st = _lib.HsbPeerOut()
        st.n_ranks, st.rank, st.cols_per_rank, st.ld = self.n_ranks, self.rank, self.cols, self.n_g
        st.h_slots, st.s_slots = self._h_tab.data_ptr(), self._s_tab.data_ptr()
        return st

    def finish(self, hb=None, sb=None):
        """This rank's column blocks (cols, n_g) = sums of its receive slots
        (``hsb_sum_slots``, on the current stream).  Call once every rank's
        build has completed (e.g. after a barrier)."""
        import ctypes

        import torch

        from . import _lib

        lib = _lib.load()
        dev = self.h_recv.device
        ctx = _lib.context(dev.index or 0)
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        out = []
        for recv, o in ((self.h_recv, hb), (self.s_recv, sb)):
            if o is None:
                o = torch.empty(recv.shape[1:], dtype=recv.dtype, device=dev)
            assert recv.is_contiguous() and o.is_contiguous() and o.shape == recv.shape[1:]
            per_slot = recv[0].numel()
            _lib.check(lib.hsb_sum_slots(ctx, stream, ctypes.c_void_p(recv.data_ptr()), recv.shape[0], per_slot,
                                         per_slot, ctypes.c_void_p(o.data_ptr())), ctx)
            out.append(o)
        return out[0], out[1]

    def close(self):
        import ctypes

        from . import _lib

        if not self._opened:
            return
        lib = _lib.load()
        ctx = _lib.context(self.h_recv.device.index or 0)
        for ptr in self._opened:
            lib.hsb_ipc_close(ctx, ctypes.c_void_p(ptr))
        self._opened = []


def build_hs_sharded_fused(dp, slots: "PeerSlots", policy=None, group=None):
    """Atom-sharded step with the fused reduce-scatter: this rank's partial H
    and S go straight from the reconstruction epilogue into the owners' slots
    (no NCCL collective on the data path); a barrier, then each owner sums
    its slots, and a second barrier before the slots can be written again.
    Returns this rank's (cols, n_g) blocks of H and S."""
    import torch
    import torch.distributed as dist

    from .pipeline import build_hs_device

    stream = torch.cuda.current_stream(slots.h_recv.device)
    build_hs_device(dp, policy=policy, peer=slots, wait=False)
    stream.synchronize()
    if dist.is_initialized():
        dist.barrier(group=group)  # every rank's partial has landed in the owners' slots
    hb, sb = slots.finish()
    stream.synchronize()
    if dist.is_initialized():
        # the slots are reused: no rank may start its next build (whose epilogue
        # writes into the owners' slots over NVLink) before every owner has
        # finished summing this step's
        dist.barrier(group=group)
    return hb, sb


def kpoint_assignment(n_kpoints: int, world: int, rank: int) -> list[int]:
    """k-points handled by ``rank`` (round robin, no communication)."""
    return list(range(rank, n_kpoints, world))


def build_kpoints(instances, policy=None, group=None, builder=None):
    """Replica-parallel builds of independent k-points: returns
    {k-index: BuildOutput} for the k-points owned by this rank."""
    import torch.distributed as dist

    if builder is None:
        from .pipeline import build_hs as builder
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return {k: builder(instances[k], policy) for k in kpoint_assignment(len(instances), world, rank)}


def e2e_sharded_step_ms(p, policy, n_g: int, ncols: int, steps: int, dev):
    """End-to-end time per sharded step for bench.py: host blocks in (H2D in
    the timed region), partial build, reduce-scatter, D2H of this rank's
    H and S column blocks.  Returns (max-over-ranks ms, local wall s)."""
    import torch
    import torch.distributed as dist

    from .pipeline import build_hs_into

    world = dist.get_world_size()
    h = torch.zeros((ncols, n_g), dtype=torch.complex128, device=dev)
    s = torch.zeros_like(h)
    hb = torch.empty((ncols // world, n_g), dtype=torch.complex128, device=dev)
    sb = torch.empty_like(hb)
    hh = torch.empty(hb.shape, dtype=hb.dtype, pin_memory=True)
    sh = torch.empty_like(hh, pin_memory=True)

    def one():
        build_hs_into(p, h, s, policy)
        reduce_scatter_block_columns(h, hb)
        reduce_scatter_block_columns(s, sb)
        hh.copy_(hb, non_blocking=True)
        sh.copy_(sb, non_blocking=True)

    one()
    barrier(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize(dev)
    wall = (time.perf_counter() - t0) / steps
    ms = max(e0.elapsed_time(e1) / steps, wall * 1e3)
    return max_over_ranks(ms, dev), wall


def barrier(dev) -> None:
    """Barrier + device synchronize (NCCL barrier bound to the rank's device)."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[dev.index])
        else:
            dist.barrier()
    torch.cuda.synchronize(dev)


def max_over_ranks(value: float, dev) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return value
    on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
