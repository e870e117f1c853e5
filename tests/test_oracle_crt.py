"""Pins of the oracle's FP64_CRT format (reading R-28; Ozaki scheme II as the exact product of
b-bit quantised operands) and of the R-26 digit rule -- against exact rational arithmetic, an
extended-precision reference and properties the method needs, not against a retyped formula.

  * orc_gemm_crt == its definition evaluated with Python Fractions (exact), incl. zero rows / columns,
    quantisation ties, sums beyond 2^64 and cancelling signs;
  * the quantisation error obeys the a-priori bound 2^-b (row max * column abs-sum + ...);
  * at b = 62 it agrees with a long-double product to FP64 rounding (no dropped term or transposition);
  * orc_crt_bits matches the library's host-side rule (a CRT product must stay below M_18 / 2^1.02);
  * R-26 property: at the digit count S the rule picks for a target RMS residual t, the CRT product's RMS
    error is <= t / 2 on iterates of the method, and one digit fewer would exceed t / 4 somewhere --
    the rule neither starves the chain nor wastes more than one digit;
  * an FP64_CRT phase in a solve converges to the certified FP64 residual with rising bits.
PAPER.md:191-194 [Sec. 4.2] ("custom number of bits in the exponent and mantissa") is the passage the
format instantiates; PAPER.md:256-261 [Sec. 4.3.1] the runtime precision increase of R-26."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def _crt_exact(X, Y, b):
    """The definition, in exact rational arithmetic."""
    n = X.shape[0]

    def flog2(x):
        m, e = math.frexp(x)
        return e - 1

    e = [0 if np.abs(X[i]).max() == 0 else b - 1 - flog2(float(np.abs(X[i]).max())) for i in range(n)]
    f = [0 if np.abs(Y[:, j]).max() == 0 else b - 1 - flog2(float(np.abs(Y[:, j]).max())) for j in range(n)]
    Xb = [[round(Fraction(float(X[i, k])) * Fraction(2) ** e[i]) for k in range(n)] for i in range(n)]
    Yb = [[round(Fraction(float(Y[k, j])) * Fraction(2) ** f[j]) for j in range(n)] for k in range(n)]
    Z = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            P = sum(Xb[i][k] * Yb[k][j] for k in range(n))
            Z[i, j] = float(Fraction(P) * Fraction(2) ** (-(e[i] + f[j])))   # float(Fraction) rounds RNE
    return Z


@pytest.mark.parametrize("b", [1, 3, 7, 17, 31, 45, 53, 59, 62])
def test_gemm_crt_equals_exact_definition(b):
    rng = np.random.default_rng(b)
    n = 11
    X = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-30, 31, n)[:, None]
    Y = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-30, 31, n)[None, :]
    X[3] = 0.0          # zero row
    Y[:, 5] = 0.0       # zero column
    X[4, :] = -X[4, :]  # sign mix
    np.testing.assert_array_equal(oracle.gemm_crt(X, Y, b), _crt_exact(X, Y, b))


def test_gemm_crt_ties_carries_and_cancellation():
    # ties: x 2^e = k + 1/2 must round to even; b = 62 products of 2^61-size integers summed over 16
    # terms exceed 2^64 (carry into the third word); exact cancellation to 0 and to a tiny remainder
    n = 16
    X = np.zeros((n, n))
    Y = np.zeros((n, n))
    X[0, :2] = [1.0, 2.0 ** -3 * 5.0]      # b = 3: max 1 -> e = 2: 4 and 2.5 -> 2 (tie to even)
    Y[:2, 0] = [1.0, 1.0]
    X[1, :] = 1.0 - 2.0 ** -40
    Y[:, 1] = 1.0 - 2.0 ** -41
    X[2, :8] = 1.0
    X[2, 8:] = -1.0
    Y[:, 2] = 3.0                          # row 2 . col 2 = 0 exactly
    Y[0, 3] = 1.0
    Y[8, 3] = -(1.0 - 2.0 ** -50)          # row 2 . col 3 = 2^-50
    for b in (3, 53, 62):
        np.testing.assert_array_equal(oracle.gemm_crt(X, Y, b), _crt_exact(X, Y, b))
    Z = oracle.gemm_crt(X, Y, 3)
    assert Z[0, 0] == 1.5                  # (4 + 2) / 4, the tie 2.5 -> 2
    assert oracle.gemm_crt(X, Y, 62)[2, 2] == 0.0


@pytest.mark.parametrize("b", [17, 31, 45, 59])
def test_gemm_crt_within_quantisation_bound(b):
    # |xbar - 2^e x| <= 1/2, i.e. |dx_ik| <= 2^-b max_k |x_ik| (and the same per column of Y):
    # |Z - XY|_ij <= 2^-b (rmax_i colsum_j + rowsum_i cmax_j) + n 2^-2b rmax_i cmax_j + 2^-53 |XY|_ij
    n = 96
    A = synth.spd(n, 10.0, 7)
    C = np.linalg.inv(A)
    C = (C + C.T) / 2
    L = np.longdouble
    exact = A.astype(L) @ C.astype(L)
    Z = oracle.gemm_crt(A, C, b)
    ra = np.abs(A).max(axis=1)[:, None]
    cc = np.abs(C).max(axis=0)[None, :]
    bound = (2.0 ** -b * (ra * np.abs(C).sum(axis=0)[None, :] + np.abs(A).sum(axis=1)[:, None] * cc)
             + n * 2.0 ** (-2 * b) * ra * cc) * (1 + 1e-9) + 2.0 ** -53 * np.abs(exact.astype(np.float64))
    err = np.abs(Z.astype(L) - exact).astype(np.float64)
    assert np.all(err <= bound), float(np.max(err / bound))
    # and the bound is not vacuous: the error uses a sizeable part of it at low b
    if b == 17:
        assert np.max(err / bound) > 0.05


def test_gemm_crt_b62_is_the_product():
    # at b = 62 the quantisation error (2^-62 of the row maximum) is below FP64 rounding: the CRT product
    # equals X Y to a few ulp -- catches a transposed operand or a dropped term in the definition
    rng = np.random.default_rng(5)
    n = 64
    X, Y = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    L = np.longdouble
    exact = (X.astype(L) @ Y.astype(L)).astype(np.float64)
    Z = oracle.gemm_crt(X, Y, 62)
    mag = np.abs(X) @ np.abs(Y)
    assert np.all(np.abs(Z - exact) <= 4 * 2.0 ** -53 * mag)
    assert not np.allclose(oracle.gemm_crt(X, Y, 62), exact.T, atol=1e-3)


def test_crt_bits_rule_matches_library():
    ipr = pytest.importorskip("paper_1703_02283_b200")   # host-side table, no GPU
    for n in (1, 64, 1000, 8192, 32768, 46000, 50000, 65535):
        for S in range(2, 10):
            assert oracle.crt_bits(S, n) == ipr.ipr_test_crt_table(18, S, n)["b_for"], (S, n)
    assert oracle.crt_bits(9, 8192) == 59 and oracle.crt_bits(9, 65535) == 59
    assert [oracle.digits_for_m(m) for m in (0, 7, 23, 31, 52)] == [2, 3, 5, 7, 9]


@pytest.mark.parametrize("n", [64, 128, 256])
def test_adaptive_digit_rule_property(n):
    # R-26 picks S for a target RMS residual t; the FP64_CRT product then carries b = crt_bits(S) bits.
    # Property the method needs: the product's RMS error (its contribution to rho_hat) stays below t / 2,
    # on the operands the FP64 phase actually multiplies (A and C ~ A^{-1/2}).  Minimality: with one
    # digit less some target would see an error above t / 4.
    A = synth.spd(n, 2.0, 3)
    r = oracle.solve(A, 2, [oracle.phase()], 1e-13, 60, form=oracle.FORM_SYMMETRIC)
    C = r.C_best
    L = np.longdouble
    exact = A.astype(L) @ C.astype(L)
    worst, worst_fewer = 0.0, 0.0
    prev_S = 0
    for t in (1e-2, 1e-3, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12, 1e-14):
        S = oracle.oz_digits(t, n)
        assert S >= prev_S                         # more digits for a smaller target
        prev_S = S
        b = oracle.crt_bits(S, n)
        assert oracle.oz_adaptive_m(S) == min(52, b)   # stored bits = product bits (below 52)
        err = float(np.sqrt(np.sum((oracle.gemm_crt(A, C, b).astype(L) - exact) ** 2) / n))
        worst = max(worst, err / t)
        if S > 3:
            errm = float(np.sqrt(np.sum((oracle.gemm_crt(A, C, oracle.crt_bits(S - 1, n)).astype(L) - exact) ** 2) / n))
            worst_fewer = max(worst_fewer, errm / t)
    assert worst <= 0.5, worst
    assert worst_fewer > 0.25, worst_fewer


def test_crt_phase_solve_converges_with_rising_bits():
    A = synth.spd(80, 2.0, 4)
    low = oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    for form in (oracle.FORM_SYMMETRIC, oracle.FORM_SYMMETRIC_TRI):
        r = oracle.solve(A, 2, [low, oracle.phase(oracle.FP64_CRT, mant_bits=oracle.MANT_ADAPTIVE,
                                                  corr_prec=oracle.BF16)], 1e-12, 80, form=form)
        ms = [x["mant_bits"] for x in r.records if x["phase"] == 1]
        assert r.outcome == oracle.CONVERGED and r.records[-1]["rho_cert"] <= 1e-12
        assert ms == sorted(ms) and ms[0] < 52 and ms[-1] == 52
    # a fixed 17-bit CRT phase cannot go below its quantisation floor: it plateaus far above 1e-12
    r = oracle.solve(A, 2, [oracle.phase(oracle.FP64_CRT, mant_bits=7, max_iters=30)], 1e-12, 30,
                     form=oracle.FORM_SYMMETRIC)
    assert r.outcome == oracle.ITER_LIMIT and min(r.rho) > 1e-6
    # not defined for the literal form (the GPU refuses it too)
    with pytest.raises(ValueError):
        oracle.solve(A, 2, [oracle.phase(oracle.FP64_CRT)], 1e-12, 10)


def test_gemm_crt_pairs_are_elements_of_the_product():
    rng = np.random.default_rng(11)
    n = 40
    X, Y = rng.standard_normal((n, n)), rng.standard_normal((n, n)) * 1e5
    for b in (5, 31, 62):
        I, J = rng.integers(0, n, 300), rng.integers(0, n, 300)
        np.testing.assert_array_equal(oracle.gemm_crt_pairs(X, Y, b, I, J), oracle.gemm_crt(X, Y, b)[I, J])
