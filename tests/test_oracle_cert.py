"""Pins of the oracle's CRT certificate (reading R-35; not in the paper -- it makes the north
star's "residual <= 1e-12" a proven statement about the returned matrix, the paper's stopping residual
being ||I - C^p A|| of Eq. (1)).

  cert_grid(C, b):  C rounded to the coarser of its row's and column's b-bit grids
  resid_dd(A, X, p): ||I - X^p A||_F in double-double arithmetic

Pinned against: exact rational arithmetic (Fraction) on cancellation-heavy inputs where an FP64
evaluation is wrong in its leading digit, the diagonal closed form, and the invariants the certificate
needs from the grid (exact b-bit row AND column quantisation, symmetry, idempotence, half-grid error,
diagonal row maxima kept); the solve mirror against the FP64-chain certificate of the same trajectory.
"""
from fractions import Fraction
import math

import numpy as np
import pytest

import oracle
import synth


def _exact_resid(A, X, p):
    n = A.shape[0]
    Af = [[Fraction(float(v)) for v in r] for r in A]
    Xf = [[Fraction(float(v)) for v in r] for r in X]
    T = Af
    for _ in range(p):
        T = [[sum(Xf[i][k] * T[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    s = sum(((1 if i == j else 0) - T[i][j]) ** 2 for i in range(n) for j in range(n))
    return math.sqrt(float(s)) if s < 1 else math.sqrt(s)   # float(s): one rounding of the exact sum


def _near_root(n, p, seed, kappa=3.0):
    A, lam, Q = synth.spd(n, kappa, seed, return_eig=True)
    X = (Q * lam ** (-1.0 / p)) @ Q.T
    return A, (X + X.T) / 2


@pytest.mark.parametrize("p", [1, 2, 3])
def test_resid_dd_equals_exact_rational_residual_under_cancellation(p):
    # X within ~1e-15 of A^{-1/p}: the residual is ~1e-15 and an FP64 evaluation carries rounding of the
    # same size; the double-double evaluation must agree with the exact rational value to 1e-12 relative
    A, X = _near_root(6, p, 11 + p)
    exact = _exact_resid(A, X, p)
    assert 0 < exact < 1e-13
    got = oracle.resid_dd(A, X, p)
    assert got == pytest.approx(exact, rel=1e-12)
    fp64 = np.linalg.norm(np.eye(6) - np.linalg.matrix_power(X, p) @ A)
    assert abs(fp64 - exact) > 1e-6 * exact       # the FP64 evaluation is visibly off (why dd exists)


def test_resid_dd_far_from_convergence_and_non_symmetric():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((5, 5))
    X = rng.standard_normal((5, 5)) * 0.3
    for p in (1, 2, 3):
        assert oracle.resid_dd(A, X, p) == pytest.approx(_exact_resid(A, X, p), rel=1e-15)


def test_resid_dd_diagonal_closed_form():
    # diagonal A, X: I - X^p A = diag(1 - x_i^p a_i), each entry exact in rational arithmetic
    a = synth.diag_spd(32, 50.0, 4).diagonal().copy()
    x = a ** -0.5
    A, X = np.diag(a), np.diag(x)
    want = math.sqrt(float(sum((1 - Fraction(float(xi)) ** 2 * Fraction(float(ai))) ** 2
                               for xi, ai in zip(x, a))))
    assert oracle.resid_dd(A, X, 2) == pytest.approx(want, rel=1e-13)


def _row_exp(C, b):
    m = np.abs(C).max(axis=1)
    e = np.zeros(C.shape[0], dtype=np.int64)
    nz = m > 0
    e[nz] = b - 1 - np.floor(np.log2(m[nz])).astype(np.int64)
    return e


@pytest.mark.parametrize("b", [62, 40, 20])
def test_cert_grid_invariants(b):
    n = 48
    rng = np.random.default_rng(b)
    S = rng.standard_normal((n, n)) * np.exp(rng.uniform(-30, 5, (n, n)))
    C = (S + S.T) / 2
    C[7, :] = 0.0
    C[:, 7] = 0.0                                   # a zero row / column
    C[3, 3] = 2.0 ** 40                             # rows with very different maxima
    Ct = oracle.cert_grid(C, b)
    np.testing.assert_array_equal(Ct, Ct.T)         # symmetric in, symmetric out
    np.testing.assert_array_equal(oracle.cert_grid(Ct, b), Ct)   # idempotent
    e = _row_exp(C, b)                              # the exponents of C (the certificate keeps them)
    g = np.minimum(e[:, None], e[None, :])
    assert np.all(np.abs(Ct - C) <= np.ldexp(1.0, -(g + 1)))   # at most half a grid step
    for i in range(n):                              # what the certificate needs: exact b-bit rows AND columns
        for j in range(n):
            if Ct[i, j] == 0.0:
                continue
            v = Fraction(float(Ct[i, j])) * Fraction(2) ** int(e[i])
            assert v.denominator == 1 and abs(v) <= 2 ** b
            w = Fraction(float(Ct[i, j])) * Fraction(2) ** int(e[j])
            assert w.denominator == 1 and abs(w) <= 2 ** b
    # an element whose own ulp is no finer than its grid is unchanged
    ulp = np.ldexp(1.0, np.frexp(np.abs(C))[1] - 53)
    keep = (C != 0) & (ulp >= np.ldexp(1.0, -g))
    assert keep.any() or b < 53
    np.testing.assert_array_equal(Ct[keep], C[keep])


def test_cert_grid_moves_only_small_elements_at_62_bits():
    A, X = _near_root(64, 2, 5, kappa=2.0)
    Ct = oracle.cert_grid(X, 62)
    d = np.abs(Ct - X)
    rowmax = np.abs(X).max(axis=1)
    moved = d > 0
    assert np.all(np.abs(X[moved]) < rowmax[np.nonzero(moved)[0]] * 2.0 ** -8)
    assert d.max() <= 2.0 ** -62 * rowmax.max()
    np.testing.assert_array_equal(np.abs(Ct).max(axis=1), rowmax)   # diagonal maxima: on their own grid
    assert abs(oracle.resid_dd(A, Ct, 2) - oracle.resid_dd(A, X, 2)) < 1e-16


@pytest.mark.parametrize("form", [oracle.FORM_SYMMETRIC_TRI, oracle.FORM_SYMMETRIC])
def test_solve_with_crt_certificate_mirrors_the_fp64_certificate_trajectory(form):
    # the certificate changes only what certifies (and the answer's grid rounding), not the trajectory:
    # same records and decisions; the answer is cert_grid of the FP64-mode answer; its certificate is the
    # double-double residual of that answer, within the FP64 evaluation noise of the FP64-mode certificate
    n = 96
    A = synth.spd(n, 2.0, 7)
    ph = [oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
          oracle.phase(corr_prec=oracle.BF16)]
    a = oracle.solve(A, 2, ph, 1e-12, 100, form=form, cert="fp64")
    b = oracle.solve(A, 2, ph, 1e-12, 100, form=form, cert="crt")
    assert a.outcome == b.outcome == oracle.CONVERGED
    assert [r["decision"] for r in a.records] == [r["decision"] for r in b.records]
    for x, y in zip(a.records, b.records):
        assert x["rho"] == y["rho"] or (np.isnan(x["rho"]) and np.isnan(y["rho"]))
    np.testing.assert_array_equal(b.C_best, oracle.cert_grid(a.C_best, 62))
    cb = b.records[-1]["rho_cert"]
    assert cb == oracle.resid_dd(A, b.C_best, 2) <= 1e-12
    assert abs(cb - a.records[-1]["rho_cert"]) < 64 * 2.0 ** -53 * n


@pytest.mark.parametrize("p", [1, 2, 3])
def test_resid_rows_dd_exact_rows(p):
    # every row against exact rational arithmetic; their sum is the squared full residual
    A, X = _near_root(5, p, 30 + p)
    n = 5
    Af = [[Fraction(float(v)) for v in r] for r in A]
    Xf = [[Fraction(float(v)) for v in r] for r in X]
    T = Af
    for _ in range(p):
        T = [[sum(Xf[i][k] * T[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    want = [float(sum(((1 if i == j else 0) - T[i][j]) ** 2 for j in range(n))) for i in range(n)]
    got = oracle.resid_rows_dd(A, X, p, range(n))
    np.testing.assert_allclose(got, want, rtol=1e-12)
    assert math.sqrt(got.sum()) == pytest.approx(oracle.resid_dd(A, X, p), rel=1e-13)
