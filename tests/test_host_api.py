"""Host-side logic of the drop-in boundary (no GPU): types, generator,
validation, flop model and the ledger the GPU build reports."""

import json

import numpy as np
import pytest

from conftest import golden_cases, load_case
from paper_1611_00606_b200 import (
    CONFIGS, Dims, Fill, GpuPolicy, HermitianResult, InputError, InvariantError, KernelKind, ProblemSpec,
    generate, heavy_fraction, preset_dims, rel_frob_error, section_flops, total_model_flops, validate_instance,
)
from paper_1611_00606_b200.ledger import flops_of
from paper_1611_00606_b200.pipeline import ledger_from_timings


def test_flops_of_frozen_values():
    # pkg/tests/test_kernels.py:404-413
    assert flops_of(KernelKind.GEMM, (3, 4, 3)) == 288
    assert flops_of(KernelKind.HER2K, (9273, 512 * 49)) == 17_258_241_724_416
    assert flops_of(KernelKind.HERK, (9273, 512 * 49)) == 8_629_120_862_208
    assert flops_of(KernelKind.DIAG_SCALE, (1, 1)) == 2
    assert flops_of(KernelKind.POTRF, (49,)) == 156_865
    assert flops_of(KernelKind.POTRF, (121,)) == 2_362_081
    assert flops_of(KernelKind.TRMM, (49, 9273)) == 4 * 49 * 49 * 9273
    assert flops_of(KernelKind.HEMM, (49, 9273)) == 8 * 49 * 49 * 9273


def test_config_model_flops_match_survey():
    # SURVEY.md section 8 table (nonhpd = 0)
    expected = {"C1": 538_431_730, "C2": 119_798_836_704, "C3": 5_031_259_458_592,
                "C4": 124_654_541_066_368}
    for name, flops in expected.items():
        assert total_model_flops(CONFIGS[name], 0) == flops
    assert heavy_fraction(preset_dims("NaCl", 4.0), 0) > 0.99


def test_section_flops_closed_form():
    # pkg/tests/test_report.py:106-
    per = section_flops(Dims(4, 3, 6), 1)
    assert per["Loop 1"] == 4 * 16 * 9 * 6
    assert per["U norm"] == 2 * 12 * 6
    with pytest.raises(InputError):
        section_flops(Dims(4, 3, 6), 5)


def test_dims_and_spec_validation():
    with pytest.raises(InputError):
        Dims(0, 1, 1)
    with pytest.raises(InputError):
        Dims(1.5, 1, 1)
    with pytest.raises(InputError):
        ProblemSpec(Dims(1, 1, 1), nonhpd_fraction=1.5)
    with pytest.raises(InputError):
        ProblemSpec(Dims(1, 1, 1), seed=-1)
    with pytest.raises(InputError):
        GpuPolicy(device=-1)


def test_validate_instance_rejects_broken_inputs():
    p = generate(ProblemSpec(Dims(2, 3, 4), seed=20))
    validate_instance(p)
    p.t_aa[0][0, 1] += 1.0  # pkg/tests/test_builder.py:296-300
    with pytest.raises(InvariantError):
        validate_instance(p)
    p = generate(ProblemSpec(Dims(2, 3, 4), seed=20))
    p.u_norms[1][0] = 0.0
    with pytest.raises(InvariantError):
        validate_instance(p)
    p = generate(ProblemSpec(Dims(2, 3, 4), seed=20))
    p.a_blocks[0][0, 0] = np.nan
    with pytest.raises(InvariantError):
        validate_instance(p)
    p = generate(ProblemSpec(Dims(2, 3, 4), seed=20))
    p.b_blocks.pop()
    with pytest.raises(InvariantError):
        validate_instance(p)


def test_hermitian_result_check():
    m = np.array([[1.0, 2 - 1j], [2 + 1j, 3.0]], dtype=complex, order="F")
    HermitianResult(m, Fill.FULL).check()
    bad = m.copy()
    bad[0, 1] = 5
    with pytest.raises(InvariantError):
        HermitianResult(bad, Fill.FULL).check()
    low = np.tril(m)
    full = HermitianResult(low, Fill.LOWER).mirrored()
    assert full.fill is Fill.FULL and rel_frob_error(full.matrix, m) == 0.0


@pytest.mark.parametrize("name", golden_cases())
def test_ledger_matches_reference_ledger(name):
    """The ledger the GPU build emits has the reference's records, in order."""
    p, fx, meta = load_case(name)
    dims = Dims(*meta["dims"])
    n_hpd = int(fx["split"][0])
    # routing: reconstruct per-atom info from the reference's Loop 2 records
    kinds = [str(k) for k in fx["ledger_kind"]]
    sections = [str(s) for s in fx["ledger_section"]]
    loop2 = [k for k, s in zip(kinds, sections) if s == "Loop 2"]
    info, i = [], 0
    while i < len(loop2):
        if loop2[i] == "potrf":
            info.append(0)
            i += 2
        else:
            info.append(-1 if meta["force_nonhpd"] else 1)
            i += 1
    assert sum(1 for x in info if x == 0) == n_hpd
    t = {k: 1.0 for k in ("loop1", "loop2", "unorm", "s1", "s2", "h1", "h2", "h3")}
    led = ledger_from_timings(dims, info, t, meta["force_nonhpd"])
    assert [r.kind.value for r in led] == kinds
    assert [r.section for r in led] == sections
    assert [list(r.dims) for r in led] == [json.loads(str(d)) for d in fx["ledger_dims"]]
    assert [r.flops for r in led] == fx["ledger_flops"].tolist()
    assert led.total_flops() == sum(section_flops(dims, dims.n_atoms - n_hpd).values())
    first_seen = list(dict.fromkeys(r.section for r in led))
    assert first_seen == list(dict.fromkeys(sections))


def test_report_summarize_and_table5():
    from paper_1611_00606_b200 import FlopLedger
    from paper_1611_00606_b200.report import TABLE5, compare_with_table5, format_table, summarize

    led = FlopLedger()
    led.add(KernelKind.HER2K, (100, 50), 0.002, "H1")
    led.add(KernelKind.HERK, (100, 50), 0.001, "S1")
    led.add(KernelKind.DIAG_SCALE, (50, 100), 0.0, "U norm")
    reps = summarize(led, peak_gflops=10.0)
    assert [r.section for r in reps] == ["U norm", "S1", "H1"]  # Table-5 order
    assert reps[0].gflops_per_s is None and reps[0].efficiency is None  # zero time -> absent
    assert reps[1].gflops_per_s == pytest.approx(4 * 50 * 100 * 100 / 0.001 / 1e9)
    assert "-" in format_table(reps) and "H1" in compare_with_table5(reps)
    assert [r.section for r in TABLE5] == ["Loop 1", "Loop 2", "U norm", "S1", "S2", "H1", "H2", "H3"]
    with pytest.raises(InputError):
        summarize(FlopLedger())


def test_int8_engine_moduli_choice():
    # engine.int8_moduli restates contract.cu oz_choose: the fewest moduli with
    # b >= 53 bits (a full FP64 mantissa) and K 2^(2b) below M/4
    import math

    from paper_1611_00606_b200 import int8_gemm_ops, int8_moduli
    from paper_1611_00606_b200.engine import DEFAULT_BITS, MAX_BITS, MODULI, SQRT_M1

    assert DEFAULT_BITS == 53
    for k in (1, 98, 7744, 11616, 30976, 46464):
        n_mod, b = int8_moduli(k)
        log2m = sum(math.log2(p) for p in MODULI[:n_mod])
        assert 53 <= b <= MAX_BITS and k * 2.0 ** (2 * b) < 2.0 ** log2m / 4  # |Re C'|, |Im C'| <= K 2^2b < M/2
        if n_mod > 11:
            prev = sum(math.log2(p) for p in MODULI[:n_mod - 1])
            assert math.floor((prev - 2 - math.log2(k)) / 2) < 53
    # C3's and C4's H / S reductions (K_tot = 2 N_A N_L): 17 moduli
    assert int8_moduli(7744) == (17, 54) and int8_moduli(30976) == (17, 53)
    assert int8_moduli(11616, 39) == (13, 41)  # the round-1 default, still selectable
    assert all(math.gcd(a, b) == 1 for i, a in enumerate(MODULI) for b in MODULI[i + 1:])
    # split complex arithmetic: odd moduli < 256, -1 a square mod each
    assert all(p % 2 == 1 and p < 256 and (j * j + 1) % p == 0 and abs(j) <= p // 2
               for p, j in zip(MODULI, SQRT_M1))
    assert int8_gemm_ops(8000, 7744) == 2 * 2 * 17 * 7744 * 8000 * 8001 // 2
    with pytest.raises(InputError):
        GpuPolicy(engine="fp16")


def _sym(v, p):
    r = v % p
    return r - p if r > p // 2 else r


def test_int8_split_complex_crt_exact():
    # CPU restatement of the INT8 engine's integer arithmetic (csrc/ozaki.cuh):
    # Gaussian-integer operands, residues phi1 = x + j y, phi2 = x - j y mod p_i
    # (int8 range), two real products per modulus (conjugation swaps the left
    # planes), reconstruction Re = (phi1 + phi2)/2, Im = (phi1 - phi2)/(2j) by the
    # explicit CRT with folded weights -- exact for |Re C|, |Im C| < M/2.
    import random

    from paper_1611_00606_b200.engine import MODULI, SQRT_M1, int8_moduli

    rng = random.Random(5)
    for conj in (True, False):
        k = 300
        n_mod, b = int8_moduli(k)
        mods, roots = MODULI[:n_mod], SQRT_M1[:n_mod]
        M = 1
        for p in mods:
            M *= p

        def gauss():
            x = rng.randint(-2 ** (b - 1), 2 ** (b - 1))
            y = rng.choice((-1, 1)) * (2 ** b - abs(x) - rng.randint(0, 3))
            return complex(0), x, y

        L = [gauss()[1:] for _ in range(k)]
        R = [gauss()[1:] for _ in range(k)]
        cre = sum((lx * rx + ly * ry) if conj else (lx * rx - ly * ry) for (lx, ly), (rx, ry) in zip(L, R))
        cim = sum((lx * ry - ly * rx) if conj else (lx * ry + ly * rx) for (lx, ly), (rx, ry) in zip(L, R))
        assert abs(cre) < M // 2 and abs(cim) < M // 2
        x_re = x_im = 0
        for p, j in zip(mods, roots):
            phi = [[_sym(x + j * y, p) for x, y in V] for V in (L, R)]
            psi = [[_sym(x - j * y, p) for x, y in V] for V in (L, R)]
            assert all(-128 <= v <= 127 for v in phi[0] + psi[0])
            lp1, lp2 = (psi[0], phi[0]) if conj else (phi[0], psi[0])
            f1 = _sym(sum(a * c for a, c in zip(lp1, phi[1])), p)
            f2 = _sym(sum(a * c for a, c in zip(lp2, psi[1])), p)
            mi = M // p
            inv_mi = pow(mi, -1, p)
            x_re += (f1 + f2) * (mi * (pow(2, -1, p) * inv_mi % p))
            x_im += (f1 - f2) * (mi * (pow(2 * j, -1, p) * inv_mi % p))
        x_re -= M * round(x_re / M)
        x_im -= M * round(x_im / M)
        assert (x_re, x_im) == (cre, cim)


def test_int8_crt_fraction_reconstruction():
    # The reconstruction of csrc/ozaki.cu (crt_frac): X / M as a two-limb
    # fixed-point sum of the residues, X = f * fl(M).  For every supported
    # modulus count, residues of integers |X| <= M/4 (the host's bound),
    # including tiny and extreme ones, must come back within a few ulp of X
    # plus the 2^-66 M truncation floor -- the FP64-width engine's contract.
    import math
    import random

    from paper_1611_00606_b200.engine import MODULI, SQRT_M1, crt_fraction, crt_weights

    rng = random.Random(7)
    for n_mod in range(11, len(MODULI) + 1):
        mods = MODULI[:n_mod]
        big_m = math.prod(mods)
        (w_re, w_im), m_f = crt_weights(n_mod)
        xs = [0, 1, -1, 5, big_m // 4, -(big_m // 4), 2 ** 60 + 3]
        xs += [rng.randint(-(big_m // 4), big_m // 4) for _ in range(40)]
        xs += [rng.randint(-2 ** 80, 2 ** 80) for _ in range(10)]
        for x_re in xs:
            x_im = rng.randint(-(big_m // 4), big_m // 4)
            # residues as the GEMM epilogue leaves them: phi1, phi2 of x_re + i x_im
            f1 = [_sym(x_re + j * x_im, p) for p, j in zip(mods, SQRT_M1)]
            f2 = [_sym(x_re - j * x_im, p) for p, j in zip(mods, SQRT_M1)]
            re = [a + b for a, b in zip(f1, f2)]
            im = [a - b for a, b in zip(f1, f2)]
            got_re = crt_fraction(re, w_re) * m_f
            got_im = crt_fraction(im, w_im) * m_f
            for got, want in ((got_re, x_re), (got_im, x_im)):
                tol = 4 * math.ulp(float(want)) + big_m * 2.0 ** -66
                assert abs(got - want) <= tol, (n_mod, want, got)


def test_int8_residue_dp4a_arithmetic():
    # CPU restatement of csrc/ozaki.cu's residue planes: x' (|x'| <= 2^55, an
    # exact double) split into lo + (hi - 2^31) 2^32 by a round-down magic add,
    # eight unsigned bytes dotted with the packed weights (mult 2^(8d) mod p) by
    # dp4a, phi1,2 = X +- Y reduced by the exact integer quotient
    # floor((v m + 2^31) / 2^32), m = rn(2^32 / p).  Includes the tie inputs
    # (x' = 2^31 mod 2^32) that a round-to-nearest split would break.
    import math
    import random
    import struct

    from paper_1611_00606_b200.engine import MODULI, SQRT_M1

    magic = 6755399441055744.0

    def lo32(d):
        return struct.unpack("<Q", struct.pack("<d", d))[0] & 0xFFFFFFFF

    def split(x):
        hm = math.floor(x * 2.0 ** -32) + magic
        return lo32((x - (hm - magic) * 4294967296.0) + magic), (lo32(hm) + 0x80000000) & 0xFFFFFFFF

    def dp4a(a, mult, d0, p, c):
        return c + sum(((a >> (8 * d)) & 0xFF) * _sym(mult * pow(2, 8 * (d0 + d), p), p) for d in range(4))

    def reduce(v, p):
        return v - p * ((v * (((1 << 32) + p // 2) // p) + (1 << 31)) >> 32)

    rng = random.Random(3)
    xs = [0.0, 1.0, -1.0, float(2 ** 55), float(-2 ** 55), float(2 ** 31), float(3 * 2 ** 31), float(-(2 ** 31)),
          9763880150499328.0]
    xs += [float(rng.randint(-2 ** 55, 2 ** 55) & ~((1 << rng.randint(0, 40)) - 1)) for _ in range(3000)]
    for x in xs:
        y = xs[rng.randrange(len(xs))]
        xl, xh = split(x)
        yl, yh = split(y)
        assert ((xh - 2 ** 31) << 32) + xl == int(x)
        for p, j in zip(MODULI, SQRT_M1):
            big_x = dp4a(xh, 1, 4, p, dp4a(xl, 1, 0, p, _sym(-pow(2, 63, p), p)))
            big_y = dp4a(yh, j, 4, p, dp4a(yl, j, 0, p, _sym(-j * pow(2, 63, p), p)))
            assert abs(big_x) + abs(big_y) < 2 ** 19
            assert reduce(big_x + big_y, p) == _sym(int(x) + j * int(y), p)
            assert reduce(big_x - big_y, p) == _sym(int(x) - j * int(y), p)


def test_int8_gemm_epilogue_reduction_exact():
    # csrc/ozaki.cu sym_mod_i32q: the GEMM epilogue's reduction of an int32
    # accumulator v to its symmetric residue: t = (v >> 16) c16 + (v & 0xffff),
    # q = floor((t m + 2^31) / 2^32), m = rn(2^32 / p); r = t - p q
    import random

    from paper_1611_00606_b200.engine import MODULI

    rng = random.Random(11)
    vs = [0, 1, -1, 2 ** 31 - 1, -2 ** 31, 65535, -65536] + [rng.randint(-2 ** 31, 2 ** 31 - 1) for _ in range(4000)]
    for p in MODULI:
        c16 = 65536 % p
        c16 = c16 - p if c16 > p // 2 else c16
        m = ((1 << 32) + p // 2) // p
        for v in vs:
            t = (v >> 16) * c16 + (v & 0xFFFF)
            assert abs(t) < 2 ** 22
            q = (t * m + (1 << 31)) >> 32
            assert t - p * q == _sym(v, p)
