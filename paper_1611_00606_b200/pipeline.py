"""``build_hs`` — the drop-in for ``hsgen.builder.build_hs`` on one B200.

Reference: /root/reference/pkg/src/hsgen/builder.py:211-224 (and the phases it
calls, builder.py:73-208).  Same signature, same contracts:

* validates the instance first and raises ``InvariantError`` (probgen.py:140);
* never mutates the instance's A/B blocks (restore contract);
* returns FULL Hermitian H and S (``Fill.FULL``);
* ``SplitCounts(hpd, nonhpd)`` with hpd + nonhpd = n_atoms;
* one ``FlopRecord`` per reference kernel call, in the reference's order,
  so ledger totals equal ``section_flops(dims, nonhpd)`` and the first-seen
  section order is Loop 1, H1, S1, U norm, S2, Loop 2, H2, H3;
* honours ``force_nonhpd`` (builder.py:138,146-147).

All arithmetic runs in libhsb200.so (hand-written sm_100a kernels, see
csrc/); this module only marshals pointers and builds the ledger.  Record
``seconds`` come from CUDA events: batched per-atom launches and fused
launches are split over their records in proportion to model flops.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hs_types import Dims, Fill, HermitianResult, InputError, InvariantError, SplitCounts, reference_module
from .instances import validate_instance
from .ledger import FlopLedger, KernelKind, flops_of


@dataclass(frozen=True)
class GpuPolicy:
    """Device selection and launch strategy for the B200 build.

    A separate type rather than a new ``ExecPolicy.mode`` value, because the
    reference rejects unknown modes (executor.py:38-39, test_executor.py:18-19).
    ``fused`` runs H and S as one launch each (mirror fused into the
    epilogue); ``fused=False`` runs one launch per reference section.
    ``pinned_outputs`` returns H and S in page-locked host memory (torch's
    caching pinned allocator), so the device-to-host copies run at full
    PCIe rate and overlap the H contraction.
    ``complex_mult`` is the real-product form of every complex contraction:
    "3m" (default; Gauss, 3 real DMMA products per complex product) or "4m"
    (4 real products).  Both agree with the reference to ~1e-15 relative
    Frobenius; the ledger charges the reference's model flops either way.

    ``engine`` selects the engine of the S and H contractions: "int8"
    emulates them on the INT8 tensor cores (Chinese-remainder / Ozaki-II
    scheme, see csrc/ozaki.cuh) with operands rounded to ``int8_bits`` bits
    per column -- by default 53, a full FP64 mantissa: the largest entries of
    every column are exact and the result is as accurate as the FP64 DMMA
    engine (~1e-16 relative Frobenius, measured against the oracle at C3 and
    C4); "dmma" runs them on the FP64 DMMA tensor cores; "auto" (default)
    is "int8" here and "dmma" for the kernel-level ``run_partitioned``, whose
    general operands get elementwise FP64 rounding.  ``int8_bits`` in
    [30, 55] (0 = 53); fewer bits need fewer moduli (~2^-bits of each
    column's max; e.g. 39 bits -> ~2e-12 with 13 instead of 17 moduli).

    ``lower_d2h`` (pinned outputs, INT8 engine): H and S cross PCIe as lower
    triangles and host threads fill the upper triangles (conjugate mirror)
    as column ranges land -- half the download bytes; identical results.
    """

    device: int = 0
    fused: bool = True
    pinned_outputs: bool = True
    complex_mult: str = "3m"
    engine: str = "auto"
    int8_bits: int = 0
    lower_d2h: bool = True

    def __post_init__(self):
        if int(self.device) != self.device or self.device < 0:
            raise InputError(f"device must be a nonnegative integer, got {self.device!r}")
        if self.complex_mult not in ("3m", "4m"):
            raise InputError(f"complex_mult must be '3m' or '4m', got {self.complex_mult!r}")
        if self.engine not in ("auto", "dmma", "int8"):
            raise InputError(f"engine must be 'auto', 'dmma' or 'int8', got {self.engine!r}")
        if self.int8_bits != 0 and not 30 <= int(self.int8_bits) <= 55:
            raise InputError(f"int8_bits must be 0 (default 53) or in [30, 55], got {self.int8_bits!r}")


@dataclass
class BuildOutput:
    h: HermitianResult
    s: HermitianResult
    split: SplitCounts
    ledger: FlopLedger
    timings: dict | None = None


def _policy(policy) -> GpuPolicy:
    # Accept the reference's ExecPolicy (or None) for signature compatibility.
    return policy if isinstance(policy, GpuPolicy) else GpuPolicy()


def _f_c16(m) -> np.ndarray:
    a = np.asarray(m)
    if a.dtype != np.complex128 or not a.flags.f_contiguous:
        a = np.asfortranarray(a, dtype=np.complex128)
    return a


def _ptr_array(arrays) -> ctypes.Array:
    return (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])


def _timings_dict(t: _lib.HsbTimings) -> dict:
    return {name: getattr(t, name) for name, _ in _lib.HsbTimings._fields_ if name != "reserved"}


def ledger_from_timings(dims: Dims, info, t: dict, force_nonhpd: bool) -> FlopLedger:
    """Reference-ordered ledger (builder.py:73-208) from section timings."""
    n_a, n_l, n_g = dims.n_atoms, dims.n_l, dims.n_g
    k = n_a * n_l
    hpd = [int(i) == 0 for i in info]
    led = FlopLedger()
    loop1 = []
    for _ in range(n_a):
        loop1 += [(KernelKind.GEMM, (n_l, n_g, n_l)), (KernelKind.HEMM, (n_l, n_g))]
    _emit_named(led, t["loop1"], "Loop 1", loop1)
    _emit_named(led, t["h1"], "H1", [(KernelKind.HER2K, (n_g, k))])
    _emit_named(led, t["s1"], "S1", [(KernelKind.HERK, (n_g, k))])
    _emit_named(led, t["unorm"], "U norm", [(KernelKind.DIAG_SCALE, (k, n_g))])
    _emit_named(led, t["s2"], "S2", [(KernelKind.HERK, (n_g, k))])
    loop2 = []
    for ok in hpd:
        if ok:
            loop2 += [(KernelKind.POTRF, (n_l,)), (KernelKind.TRMM, (n_l, n_g))]
        else:
            loop2 += [(KernelKind.HEMM, (n_l, n_g))]
    _emit_named(led, t["loop2"], "Loop 2", loop2)
    n_hpd = sum(hpd)
    if n_hpd < n_a:
        _emit_named(led, t["h2"], "H2", [(KernelKind.GEMM, (n_g, n_g, (n_a - n_hpd) * n_l))])
    if n_hpd:
        _emit_named(led, t["h3"], "H3", [(KernelKind.HERK, (n_g, n_hpd * n_l))])
    return led


def _emit_named(led: FlopLedger, seconds: float, section: str, records) -> None:
    total = sum(flops_of(kind, d) for kind, d in records) or 1
    for kind, d in records:
        led.add(kind, d, max(0.0, seconds) * flops_of(kind, d) / total, section)


def _host_matrix(n: int, pinned: bool) -> np.ndarray:
    """n x n complex128 F-order host array, optionally page-locked."""
    if pinned:
        import torch

        return torch.empty((n, n), dtype=torch.complex128, pin_memory=True).numpy().T
    return np.empty((n, n), dtype=np.complex128, order="F")


def pin_instance(p):
    """Copy an instance's blocks into page-locked host memory.

    The drop-in accepts ordinary numpy blocks (they are staged through pinned
    slots by host threads); blocks that already live in pinned memory are
    DMA'd directly, which is the fastest way to feed repeated builds.
    Returns a new ``ProblemInstance`` whose blocks are F-order numpy views of
    torch pinned tensors.
    """
    import torch

    from .instances import ProblemInstance

    def pin(m):
        m = np.asarray(m)
        if m.ndim == 1:
            out = torch.empty(m.shape, dtype=torch.float64, pin_memory=True).numpy()
        else:
            out = torch.empty(m.shape[::-1], dtype=torch.complex128, pin_memory=True).numpy().T
        out[...] = m
        return out

    q = ProblemInstance(Dims(p.dims.n_atoms, p.dims.n_l, p.dims.n_g))
    for name in ("a_blocks", "b_blocks", "t_aa", "t_ab", "t_bb", "u_norms"):
        setattr(q, name, [pin(m) for m in getattr(p, name)])
    return q


def _host_problem(p):
    """hsb_problem over the instance's own host blocks (no stacking copy)."""
    n_a, n_l, n_g = int(p.dims.n_atoms), int(p.dims.n_l), int(p.dims.n_g)
    blocks = {name: [_f_c16(m) for m in getattr(p, name)]
              for name in ("a_blocks", "b_blocks", "t_aa", "t_ab", "t_bb")}
    blocks["u_norms"] = [np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in p.u_norms]
    arrays = {name: _ptr_array(v) for name, v in blocks.items()}
    prob = _lib.HsbProblem()
    prob.n_atoms, prob.n_l, prob.n_g = n_a, n_l, n_g
    prob.location = _lib.HSB_LOC_HOST
    for name, arr in arrays.items():
        setattr(prob, name, ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)))
    return prob, (blocks, arrays)


def _call_build(pol, prob, out, stream, force_nonhpd, n_a, slot: int = 0, wait: bool = True, phys=None,
                lower_only: bool = False):
    lib = _lib.load()
    opts = (_lib.HSB_OPT_FORCE_NONHPD if force_nonhpd else 0) | (0 if pol.fused else _lib.HSB_OPT_UNFUSED)
    if not pol.lower_d2h:
        opts |= _lib.HSB_OPT_FULL_D2H
    if lower_only:
        opts |= _lib.HSB_OPT_LOWER_ONLY
    if prob.location == _lib.HSB_LOC_HOST:
        opts |= _lib.HSB_OPT_VALIDATE  # T / u values are checked natively, before any transfer
    tim = _lib.HsbTimings()
    info = (ctypes.c_int32 * n_a)()
    with _lib.using(pol.device, pol.complex_mult, pol.engine, pol.int8_bits, slot) as ctx:
        # no timings -> the library returns without waiting (device in/out only)
        if phys is not None:  # matching coefficients into prob's stacks, then the build (one call)
            _lib.check(lib.hsb_build_hs_physical(ctx, stream, ctypes.byref(phys), ctypes.byref(prob), opts,
                                                 ctypes.byref(out), ctypes.byref(tim) if wait else None,
                                                 info if wait else None), ctx)
        else:
            _lib.check(lib.hsb_build_hs(ctx, stream, ctypes.byref(prob), opts, ctypes.byref(out),
                                        ctypes.byref(tim) if wait else None, info if wait else None), ctx)
    return (tim, list(info)) if wait else (None, None)


def build_hs(p, policy=None, force_nonhpd: bool = False) -> BuildOutput:
    """Assemble H and S on the GPU from host-resident per-atom blocks.

    When the reference package is importable the result is the reference's
    own ``hsgen.builder.BuildOutput`` (with ``hsgen`` HermitianResult,
    SplitCounts and FlopLedger inside; ``timings`` attached), so code that
    consumes ``hsgen.build_hs`` results -- cli.cmd_run (cli.py:160-183),
    report.summarize -- takes the drop-in's unchanged."""
    return to_reference_output(_build_host(p, policy, force_nonhpd))


def to_reference_output(out: BuildOutput):
    """``out`` as ``hsgen.builder.BuildOutput`` when the reference is
    importable (builder.py:51-62), else unchanged."""
    builder, kernels, matcore = (reference_module(m) for m in ("builder", "kernels", "matcore"))
    if builder is None or kernels is None or matcore is None:
        return out
    led = kernels.FlopLedger()
    for r in out.ledger:
        led.add(kernels.KernelKind(r.kind.value), r.dims, r.seconds, r.section)
    ref = builder.BuildOutput(h=matcore.HermitianResult(out.h.matrix, matcore.Fill(out.h.fill.value)),
                              s=matcore.HermitianResult(out.s.matrix, matcore.Fill(out.s.fill.value)),
                              split=builder.SplitCounts(out.split.hpd, out.split.nonhpd), ledger=led)
    ref.timings = out.timings
    return ref


def _validate_shapes(p) -> None:
    """Shapes and block counts here; values natively (HSB_OPT_VALIDATE for T
    and u, staging for A and B).  On a shape error the full reference-order
    validation runs, so an earlier field's value error still wins."""
    try:
        validate_instance(p, check_stack_values=False, check_block_values=False)
    except InvariantError:
        validate_instance(p)
        raise


def _build_host(p, policy, force_nonhpd, slot: int = 0, stream=None, s_ready=None, order=None) -> BuildOutput:
    _validate_shapes(p)
    pol = _policy(policy)
    dims = Dims(p.dims.n_atoms, p.dims.n_l, p.dims.n_g)
    prob, _keep = _host_problem(p)
    h = _host_matrix(dims.n_g, pol.pinned_outputs)
    s = _host_matrix(dims.n_g, pol.pinned_outputs)
    out = _lib.HsbOutput()
    out.location = _lib.HSB_LOC_HOST
    out.ld = dims.n_g
    out.h, out.s = h.ctypes.data, s.ctypes.data
    if s_ready is not None:
        out.s_ready = s_ready
    if order is not None:  # (h2d_after, h2d_done, compute_after, compute_done, order_in, order_out)
        (out.h2d_after, out.h2d_done, out.compute_after, out.compute_done, out.order_in, out.order_out) = order
    try:
        tim, info = _call_build(pol, prob, out, stream, force_nonhpd, dims.n_atoms, slot)
    except InvariantError:
        # the native checks run T / u before the A / B scan; report the
        # failure the reference's validation order (probgen.py:140-168) finds first
        validate_instance(p)
        raise
    t = _timings_dict(tim)
    led = ledger_from_timings(dims, info, t, force_nonhpd)
    return BuildOutput(HermitianResult(h, Fill.FULL), HermitianResult(s, Fill.FULL),
                       SplitCounts(tim.n_hpd, tim.n_nonhpd), led, t)


def iter_hs_kpoints(instances, policy=None, force_nonhpd: bool = False, depth: int = 2):
    """Yield ``build_hs`` of each independent k-point (BASELINE config C5) in
    input order, pipelined on one GPU: ``depth`` host threads each drive their
    own context and CUDA stream, so one k-point's uploads and H/S downloads
    (PCIe) overlap another's kernels.  Consecutive k-points are chained by
    CUDA events (hsb_output.h2d_after / compute_after): uploads run back to
    back in k-point order on the host-to-device engine, kernels in k-point
    order on the SMs, and each k-point's downloads overlap the next one's
    kernels and the one after's uploads -- a three-stage pipeline at
    depth >= 3.  At most ``depth`` results are in flight beyond the one being
    consumed, so pinned output memory stays bounded when the caller drops each
    result after use."""
    pol = _policy(policy)
    if int(depth) != depth or depth < 1:
        raise InputError(f"depth must be a positive integer, got {depth!r}")
    instances = list(instances)
    if depth == 1 or len(instances) <= 1:
        for p in instances:
            yield _build_host(p, pol, force_nonhpd)
        return

    def run(i, slot, stream, order):
        return _build_host(instances[i], pol, force_nonhpd, slot=slot, stream=ctypes.c_void_p(stream.cuda_stream),
                           order=order)

    yield from _lane_pipeline(len(instances), depth, pol, max(int(p.dims.n_g) for p in instances), run)


def _lane_pipeline(count: int, depth: int, pol, n_max: int, run):
    """Run ``run(i, slot, stream, order)`` for i in 0..count-1 on ``depth``
    lanes (host threads, each with its own context slot and CUDA stream) and
    yield the results in order.  ``order`` is the hsb_output ordering tuple
    (h2d_after, h2d_done, compute_after, compute_done, order_in, order_out)
    that chains item i's uploads and kernels after item i-1's."""
    import threading

    import torch

    dev = torch.device("cuda", pol.device)
    streams = [torch.cuda.Stream(device=dev) for _ in range(depth)]
    if pol.pinned_outputs:
        # up to depth + 1 results (two matrices each) are alive at once: have the
        # caching pinned allocator hold that many blocks before the lanes start,
        # so no 1 GB cudaHostAlloc lands in the middle of the pipeline
        warm = [_host_matrix(n_max, True) for _ in range(2 * (depth + 1))]
        del warm
    results = [None] * count
    ready = [threading.Event() for _ in range(count)]
    # window: item i may start once fewer than depth results ahead of it are
    # unconsumed (i < consumed + depth), so a fast lane cannot use up the
    # window with later items while the consumer waits for an earlier one
    window = threading.Condition()
    consumed = [0]
    failure = []

    # ordering: item i's uploads wait for item i-1's (h2d events), its kernels
    # for item i-1's (compute events).  The library only waits on an event
    # once the previous call has recorded it (progress flags, one per item).
    # Events are recycled modulo depth + 2: item i + depth + 2 starts only
    # after result i + 1 was consumed, i.e. after item i + 1 finished waiting
    # on item i's events.
    n_ev = depth + 2
    h2d_ev = [torch.cuda.Event() for _ in range(n_ev)]
    cmp_ev = [torch.cuda.Event() for _ in range(n_ev)]
    for ev in h2d_ev + cmp_ev:
        ev.record(torch.cuda.current_stream(dev))  # materialise the CUDA events
    torch.cuda.current_stream(dev).synchronize()
    flags = (ctypes.c_int32 * count)()
    flag_ptr = ctypes.cast(flags, ctypes.c_void_p).value

    def order_of(i):
        def fp(j):
            return ctypes.cast(ctypes.c_void_p(flag_ptr + 4 * j), ctypes.POINTER(ctypes.c_int32))
        prev = (h2d_ev[(i - 1) % n_ev].cuda_event, cmp_ev[(i - 1) % n_ev].cuda_event, fp(i - 1)) if i > 0 \
            else (None, None, None)
        return (prev[0], h2d_ev[i % n_ev].cuda_event, prev[1], cmp_ev[i % n_ev].cuda_event, prev[2], fp(i))

    def lane(slot):  # one thread per context: items slot, slot + depth, ...
        try:
            for i in range(slot, count, depth):
                with window:
                    window.wait_for(lambda: failure or i < consumed[0] + depth)
                if failure:
                    return
                results[i] = run(i, slot, streams[slot], order_of(i))
                ready[i].set()
        except BaseException as exc:  # noqa: BLE001 - re-raised in the consumer
            failure.append(exc)
            for e in ready:
                e.set()
        finally:
            for i in range(slot, count, depth):  # never leave a later item waiting
                flags[i] = max(flags[i], 2)

    threads = [threading.Thread(target=lane, args=(k,), daemon=True) for k in range(depth)]
    for t in threads:
        t.start()
    try:
        for i in range(count):
            ready[i].wait()
            if results[i] is None:  # released by a lane's failure, not built: stop here
                raise failure[0]
            # (a result that completed before another item failed is still yielded, in order)
            r, results[i] = results[i], None
            with window:
                consumed[0] = i + 1
                window.notify_all()
            yield r
    finally:
        if not failure:  # stop lanes that are still waiting for the window
            failure.append(GeneratorExit())
        with window:
            window.notify_all()
        for t in threads:
            t.join()


def build_hs_kpoints(instances, policy=None, force_nonhpd: bool = False, depth: int = 2):
    """List form of ``iter_hs_kpoints``: every result equals the serial
    ``build_hs`` of that instance."""
    return list(iter_hs_kpoints(instances, policy, force_nonhpd, depth))


def build_hs_into(p, h, s, policy=None, force_nonhpd: bool = False, stream=None, lower_only: bool = False):
    """Host per-atom blocks in, device H/S out (torch tensors, row-major
    (>= n_g, n_g) holding the column-major matrices).  Used by the sharded
    multi-GPU path, whose partial H/S go straight into a reduce-scatter.
    ``lower_only``: lower triangles only, no mirror (HSB_OPT_LOWER_ONLY; the
    triangle-packed exchange reads nothing else)."""
    import torch

    _validate_shapes(p)
    pol = _policy(policy)
    n_g = int(p.dims.n_g)
    for name, t in (("h", h), ("s", s)):
        if t.dtype != torch.complex128 or t.dim() != 2 or t.shape[1] != n_g or t.shape[0] < n_g \
                or not t.is_contiguous():
            raise InputError(f"{name} must be a contiguous complex128 tensor of shape (>= {n_g}, {n_g})")
    prob, _keep = _host_problem(p)
    out = _lib.HsbOutput()
    out.location = _lib.HSB_LOC_DEVICE
    out.ld = n_g
    out.h, out.s = h.data_ptr(), s.data_ptr()
    if stream is None:
        stream = torch.cuda.current_stream(h.device)
    tim, info = _call_build(pol, prob, out, ctypes.c_void_p(stream.cuda_stream), force_nonhpd,
                            int(p.dims.n_atoms), lower_only=lower_only)
    return SplitCounts(tim.n_hpd, tim.n_nonhpd), _timings_dict(tim), info


# ---------------------------------------------------------------- device path

@dataclass
class DeviceProblem:
    """Stacked, device-resident instance (torch tensors as plain device memory).

    Column-major K x n_g matrices are stored as row-major (n_g, K) tensors,
    so ``a_stack`` is exactly ``matcore.stack(p.a_blocks)`` in memory.
    """

    dims: Dims
    a_stack: object   # torch.complex128 (n_g, K)
    b_stack: object
    t_aa: object      # torch.complex128 (n_atoms, n_l, n_l), [a] = column-major T_a
    t_ab: object
    t_bb: object
    u: object         # torch.float64 (K,)

    @classmethod
    def from_instance(cls, p, device: int = 0) -> "DeviceProblem":
        import torch

        validate_instance(p)
        dims = Dims(p.dims.n_atoms, p.dims.n_l, p.dims.n_g)
        dev = torch.device("cuda", device)

        def stack_t(blocks):
            host = np.concatenate([np.asarray(b, dtype=np.complex128).T for b in blocks], axis=1)
            return torch.from_numpy(np.ascontiguousarray(host)).to(dev)

        def mats(blocks):
            host = np.stack([np.asarray(b, dtype=np.complex128).T for b in blocks])
            return torch.from_numpy(np.ascontiguousarray(host)).to(dev)

        u = torch.from_numpy(np.concatenate([np.asarray(x, dtype=np.float64) for x in p.u_norms])).to(dev)
        return cls(dims, stack_t(p.a_blocks), stack_t(p.b_blocks), mats(p.t_aa), mats(p.t_ab),
                   mats(p.t_bb), u)


def build_hs_device(dp: DeviceProblem, h=None, s=None, policy=None, force_nonhpd: bool = False,
                    stream=None, s_ready=None, wait: bool = True, peer=None, host_outputs: bool = False,
                    slot: int = 0, order=None, phys=None, lower_only: bool = False):
    """Device-resident build: returns (H, S, SplitCounts, timings, atom_info).

    H and S are torch complex128 (n_g, n_g) tensors holding the column-major
    matrices (i.e. ``H.T`` is the matrix; for Hermitian H this equals
    ``H.conj()``).  Inputs are not modified.  ``s_ready`` (a torch.cuda.Event)
    is recorded on the stream as soon as S is final.  With ``wait=False`` the
    call returns once the work is enqueued (split counts, timings and atom
    info are then None); the results are ready in stream order.  ``peer``
    (distributed.PeerSlots) scatters this rank's partial H and S into the
    owners' receive slots instead of h and s (INT8 engine).  ``slot`` picks the
    library context, ``order`` chains the call after a previous pipelined one
    (see ``_lane_pipeline``).  ``host_outputs``
    returns H and S as column-major numpy arrays in (pinned) host memory
    instead, downloaded while the contractions run (the drop-in path's output
    streaming, lower triangles completed by the host mirror).  ``phys`` (an
    ``_lib.HsbPhys``, see physics.py) makes the call generate the matching
    coefficients into ``dp``'s A and B stacks first (hsb_build_hs_physical).
    ``lower_only``: H and S as lower triangles, no mirror (HSB_OPT_LOWER_ONLY).
    """
    import torch

    pol = _policy(policy)
    n_a, n_l, n_g = dp.dims.n_atoms, dp.dims.n_l, dp.dims.n_g
    k = n_a * n_l
    dev = dp.a_stack.device
    for name, shape, dtype in (("a_stack", (n_g, k), torch.complex128), ("b_stack", (n_g, k), torch.complex128),
                               ("t_aa", (n_a, n_l, n_l), torch.complex128),
                               ("t_ab", (n_a, n_l, n_l), torch.complex128),
                               ("t_bb", (n_a, n_l, n_l), torch.complex128), ("u", (k,), torch.float64)):
        tns = getattr(dp, name)
        if tuple(tns.shape) != shape or tns.dtype != dtype or not tns.is_contiguous() or tns.device != dev:
            raise InputError(f"{name} must be a contiguous {dtype} tensor of shape {shape} on {dev}")
    if host_outputs:
        if peer is not None or h is not None or s is not None or not wait:
            raise InputError("host_outputs excludes peer, h, s and wait=False")
        pol0 = _policy(policy)
        h_host, s_host = _host_matrix(n_g, pol0.pinned_outputs), _host_matrix(n_g, pol0.pinned_outputs)
    elif peer is None:
        if h is None:
            h = torch.empty((n_g, n_g), dtype=torch.complex128, device=dev)
        if s is None:
            s = torch.empty((n_g, n_g), dtype=torch.complex128, device=dev)
        for name, t in (("h", h), ("s", s)):
            if t.dtype != torch.complex128 or t.dim() != 2 or t.shape[1] != n_g or t.shape[0] < n_g \
                    or not t.is_contiguous() or t.device != dev:
                raise InputError(f"{name} must be a contiguous complex128 tensor of shape (>= {n_g}, {n_g})")
    prob = _lib.HsbProblem()
    prob.n_atoms, prob.n_l, prob.n_g = n_a, n_l, n_g
    prob.location = _lib.HSB_LOC_DEVICE
    prob.a_stack, prob.b_stack = dp.a_stack.data_ptr(), dp.b_stack.data_ptr()
    prob.t_aa_dev, prob.t_ab_dev, prob.t_bb_dev = dp.t_aa.data_ptr(), dp.t_ab.data_ptr(), dp.t_bb.data_ptr()
    prob.u_dev = dp.u.data_ptr()
    out = _lib.HsbOutput()
    out.location = _lib.HSB_LOC_HOST if host_outputs else _lib.HSB_LOC_DEVICE
    out.ld = n_g
    if host_outputs:
        out.h, out.s = h_host.ctypes.data, s_host.ctypes.data
    else:
        out.h = h.data_ptr() if peer is None else None
        out.s = s.data_ptr() if peer is None else None
    if s_ready is not None:
        s_ready.record(torch.cuda.current_stream(dev))  # materialise the CUDA event
        out.s_ready = s_ready.cuda_event
    if peer is not None:
        peer_struct = peer.struct()
        out.peer = ctypes.pointer(peer_struct)
    if order is not None:  # (h2d_after, h2d_done, compute_after, compute_done, order_in, order_out)
        (out.h2d_after, out.h2d_done, out.compute_after, out.compute_done, out.order_in, out.order_out) = order
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    tim, info = _call_build(pol, prob, out, ctypes.c_void_p(stream.cuda_stream), force_nonhpd, n_a, slot=slot,
                            wait=wait, phys=phys, lower_only=lower_only)
    if not wait:
        return h, s, None, None, None
    if host_outputs:
        h, s = h_host, s_host
    return h, s, SplitCounts(tim.n_hpd, tim.n_nonhpd), _timings_dict(tim), info
