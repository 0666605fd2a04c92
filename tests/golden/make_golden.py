"""Generate the golden fixtures from the reference implementation itself.

Run in the development container, where the reference is mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``hsgen`` (the reference package, /root/reference/pkg/src/hsgen),
generates seeded instances with ``hsgen.probgen.generate``, runs
``hsgen.builder.build_hs``, the brute-force oracle ``hsgen.reference``
(h_reference / s_reference, small cases) and the serial kernels, and stores
inputs' digests and outputs as .npz files next to this script.  The GPU box
has no /root/reference, so tests compare against these files.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import hsgen  # noqa: E402
from hsgen import kernels as K  # noqa: E402

HERE = Path(__file__).resolve().parent

# (name, (n_atoms, n_l, n_g), seed, nonhpd_fraction, force_nonhpd, with_brute_oracle)
CASES = [
    ("tiny_mixed", (3, 4, 7), 5, 0.5, False, True),
    ("small_hpd", (4, 8, 64), 0, 0.0, False, True),
    ("small_mixed", (4, 8, 64), 1, 0.5, False, True),
    ("small_nonhpd", (2, 12, 48), 2, 1.0, False, True),
    ("forced", (3, 6, 40), 3, 0.0, True, True),
    ("ragged", (5, 7, 131), 7, 0.4, False, True),
    ("c1", (2, 49, 500), 0, 0.0, False, False),
]


def instance_digest(p) -> str:
    h = hashlib.sha256()
    for name in ("a_blocks", "b_blocks", "t_aa", "t_ab", "t_bb", "u_norms"):
        for blk in getattr(p, name):
            h.update(np.asarray(blk).tobytes(order="F"))
    return h.hexdigest()


def build_cases():
    meta = {}
    for name, dims, seed, frac, force, brute in CASES:
        t0 = time.perf_counter()
        p = hsgen.generate(hsgen.ProblemSpec(hsgen.Dims(*dims), seed=seed, nonhpd_fraction=frac))
        out = hsgen.build_hs(p, force_nonhpd=force)
        rec = {
            "h": out.h.matrix, "s": out.s.matrix,
            "split": np.array([out.split.hpd, out.split.nonhpd]),
            "ledger_kind": np.array([r.kind.value for r in out.ledger.records]),
            "ledger_section": np.array([r.section for r in out.ledger.records]),
            "ledger_dims": np.array([json.dumps(list(r.dims)) for r in out.ledger.records]),
            "ledger_flops": np.array([r.flops for r in out.ledger.records], dtype=np.int64),
        }
        if brute:
            rec["h_ref"] = hsgen.h_reference(p).matrix
            rec["s_ref"] = hsgen.s_reference(p).matrix
        np.savez_compressed(HERE / f"build_{name}.npz", **rec)
        meta[name] = {"dims": dims, "seed": seed, "nonhpd_fraction": frac, "force_nonhpd": force,
                      "digest": instance_digest(p), "seconds": time.perf_counter() - t0}
        print(name, meta[name], flush=True)
    return meta


def kernel_cases():
    rng = np.random.default_rng(1234)

    def cm(r, c):
        return np.asfortranarray(rng.standard_normal((r, c)) + 1j * rng.standard_normal((r, c)))

    rec = {}
    # herk (alpha real, beta in {0, 1, 0.5}), k x n operand, ragged sizes
    for i, (k, n, alpha, beta) in enumerate([(7, 5, 1.0, 0.0), (13, 70, 0.75, 1.0), (33, 65, -1.5, 0.5),
                                              (1, 1, 2.0, 0.0), (40, 129, 1.0, 0.0)]):
        a, c = cm(k, n), cm(n, n)
        rec[f"herk{i}_a"], rec[f"herk{i}_c"] = a, c.copy(order="F")
        rec[f"herk{i}_ab"] = np.array([alpha, beta])
        rec[f"herk{i}_out"] = K.herk(alpha, a, beta, c.copy(order="F"))
    for i, (k, n, alpha, beta) in enumerate([(9, 6, 1.0, 0.0), (17, 67, 0.5 + 0.25j, 1.0),
                                              (31, 64, 1.0 - 2.0j, 0.5), (2, 130, 1.0, 0.0)]):
        z, b, c = cm(k, n), cm(k, n), cm(n, n)
        rec[f"her2k{i}_z"], rec[f"her2k{i}_b"], rec[f"her2k{i}_c"] = z, b, c.copy(order="F")
        rec[f"her2k{i}_ab"] = np.array([alpha, beta], dtype=np.complex128)
        rec[f"her2k{i}_out"] = K.her2k(alpha, z, b, beta, c.copy(order="F"))
    gemm_cases = [("C", "N", 5, 6, 7, 1.0, 0.0), ("C", "N", 70, 66, 19, 1.0, 1.0), ("T", "N", 9, 65, 12, 0.5j, 0.0),
                  ("N", "N", 33, 17, 40, 1.0, 2.0 - 1.0j), ("N", "T", 8, 9, 10, -1.0, 0.0),
                  ("C", "C", 20, 21, 22, 1.0 + 1.0j, 0.5), ("T", "C", 64, 64, 3, 1.0, 0.0)]
    for i, (opa, opb, m, n, k, alpha, beta) in enumerate(gemm_cases):
        a = cm(m, k) if opa == "N" else cm(k, m)
        b = cm(k, n) if opb == "N" else cm(n, k)
        c = cm(m, n)
        rec[f"gemm{i}_a"], rec[f"gemm{i}_b"], rec[f"gemm{i}_c"] = a, b, c.copy(order="F")
        rec[f"gemm{i}_ops"] = np.array([opa, opb])
        rec[f"gemm{i}_ab"] = np.array([alpha, beta], dtype=np.complex128)
        rec[f"gemm{i}_out"] = K.gemm(alpha, opa, a, opb, b, beta, c.copy(order="F"))
    # potrf: HPD, indefinite (fails at a known minor), known-answer cases
    for i, n in enumerate([1, 5, 49, 121]):
        q, _ = np.linalg.qr(cm(n, n))
        d = rng.uniform(0.5, 2.0, n)
        t = (q * d) @ q.conj().T
        t = np.asfortranarray((t + t.conj().T) / 2)
        f, info = K.potrf_lower(t)
        rec[f"potrf{i}_t"], rec[f"potrf{i}_f"], rec[f"potrf{i}_info"] = t, f, np.array(info)
        d2 = d.copy()
        d2[int(np.argmin(d2))] = -0.05
        t2 = (q * d2) @ q.conj().T
        t2 = np.asfortranarray((t2 + t2.conj().T) / 2)
        f2, info2 = K.potrf_lower(t2)
        rec[f"potrf{i}_t_bad"], rec[f"potrf{i}_info_bad"] = t2, np.array(info2)
        assert f2 is None
    np.savez_compressed(HERE / "kernels.npz", **rec)


def main():
    kernel_cases()
    meta = build_cases()
    meta["_generator"] = {"hsgen_version": hsgen.__version__, "numpy": np.__version__,
                          "script": "tests/golden/make_golden.py"}
    (HERE / "meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
