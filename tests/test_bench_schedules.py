"""Host-side pins of bench.py's schedule handling (no GPU): the default schedule string parses into
the documented phases, low phases of the symmetric forms leave at rho_hat <= 2u of their format
(switch_tol = 2u sqrt(n), u = 2^-(m+1)), the literal form at rho_hat <= 1e-2, N > 1 runs the same schedule
(no fallback since round 2), and the certificate each run uses."""
import math

import pytest

bench = pytest.importorskip("bench")
ipr = pytest.importorskip("paper_1703_02283_b200")


def test_default_schedule_phases():
    form, ph = bench.schedule(bench.DEFAULT_SCHEDULE, 8192)
    assert form == "symmetric_triz" and ipr.FORM_BY_NAME[form] == ipr.IPR_FORM_SYMMETRIC_TRIZ   # reading R-37
    assert [ipr.PREC_NAMES[p.prec] for p in ph] == ["fp8", "bf16", "fp64crt"]
    assert ph[-1].mant_bits == ipr.IPR_MANT_ADAPTIVE and ph[-1].corr_prec == ipr.IPR_BF16
    assert ph[0].corr_prec == ipr.IPR_FP8 and ph[1].corr_prec == -1     # R-29: FP8 correction in the FP8 phase
    for p, m in zip(ph[:-1], (3, 7)):
        assert p.switch_tol == pytest.approx(2.0 * 2.0 ** -(m + 1) * math.sqrt(8192))
        assert p.plateau_ratio == 0.7 and p.plateau_arm == 0.5 and p.max_iters == 40
    assert ph[-1].switch_tol == 0.0 and ph[-1].max_iters == 0


def test_literal_low_phase_switch():
    form, ph = bench.schedule("bf16>fp64", 1024)
    assert form == "literal"
    assert ph[0].switch_tol == pytest.approx(1e-2 * math.sqrt(1024))


def test_parse_schedule_fields():
    form, parts = bench.parse_schedule("sym:bf16>fp64oz@23/cbf16>fp64crt@a/ctf32")
    assert form == "symmetric"
    assert parts == [("bf16", -1, -1), ("fp64oz", "bf16", 23), ("fp64crt", "tf32", -2)]


def test_multi_gpu_runs_the_same_schedule():
    # since round 2 the CRT phase, the tri form and the FP8 correction shard: bench.py
    # times the SAME schedule at every N -- no N > 1 substitution rule left in main()
    form, ph = bench.schedule(bench.DEFAULT_SCHEDULE, 8192)
    assert form == "symmetric_triz"
    assert [ipr.PREC_NAMES[p.prec] for p in ph] == ["fp8", "bf16", "fp64crt"]
    src = open(bench.__file__).read()
    assert "form_note" not in src and "p.prec = ipr.IPR_FP64" not in src

def test_auto_certificate_choice():
    # IPR_CERT_CRT (R-35) where it applies: a symmetric form with an fp64crt phase, p = 2 at any G or p = 3
    # on one GPU; the DMMA evaluation (R-30) otherwise; an explicit choice wins
    import bench
    assert bench.auto_cert(bench.DEFAULT_SCHEDULE, 2) == "crt"
    assert bench.auto_cert(bench.DEFAULT_SCHEDULE, 2, world=8) == "crt"
    assert bench.auto_cert("sym:bf16>fp64crt@a/cbf16", 3) == "crt"
    assert bench.auto_cert("sym:bf16>fp64crt@a/cbf16", 3, world=2) == "fp64"
    assert bench.auto_cert("symtri:bf16>fp64/cbf16", 2) == "fp64"        # no CRT phase: no CRT buffers
    assert bench.auto_cert("bf16>fp64", 2) == "fp64"                      # the literal form
    assert bench.auto_cert(bench.DEFAULT_SCHEDULE, 2, "fp64") == "fp64"
