"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Restatements of the reference algorithm (/root/reference/pkg/src/hsgen) used
to check the B200 path.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package, and only as the checker or the timed CPU baseline — never as part of
the product path (``paper_1611_00606_b200`` never imports it).

Parity pinning: ``alg1`` and ``brute`` are checked against fixtures produced
by running the reference itself (tests/golden/make_golden.py imports
``hsgen`` from /root/reference and runs ``build_hs``, ``h_reference``,
``s_reference`` and the serial kernels); see tests/test_oracle_golden.py.
The matching-coefficient restatement (``matching``) has no reference
implementation to pin against: parity unpinned by
the reference, pinned instead to closed forms and scipy's special functions.

Modules:
  alg1     — Algorithm 1 exactly as builder.build_hs sequences it, on
             scipy/OpenBLAS ZHERK/ZHER2K/ZGEMM (the paper's MKL-equivalent
             CPU path; the bench's CPU baseline).
  brute    — the defining per-atom sums of reference.h_reference /
             s_reference (Eqs. 4-7), vectorised per atom.
  kernels  — BLAS-convention restatements of kernels.herk / her2k / gemm /
             potrf_lower for kernel-level parity tests.
"""
