"""Pins of the oracle's NEXT-2 form: the symmetrised correction

    Z_p = C^{p-1} A C,  R = I - Z_p,  W = C R,  C_{k+1} = q_m(C + (W + W^T) / (2p)),   p >= 2

(Eq. (1), is C + C (I - C^p A) / p; this form takes the residual as
C^{p-1} A C and symmetrises the correction -- DESIGN.md reading R-22).  Pinned against: exact
rational arithmetic of the definition on a non-commuting 2 x 2, the closed-form linearisation
at the fixed point (derived by hand below, independent of the code), closed-form limits, the
eigen-decomposition limit, exact symmetry, and the spectral predictor of the exact iteration.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

SYM = oracle.FORM_SYMMETRIC


def _fr(M):
    return [[Fraction(x) for x in row] for row in M]


def _mm(X, Y):
    n = len(X)
    return [[sum(X[i][k] * Y[k][j] for k in range(n)) for j in range(n)] for i in range(n)]


@pytest.mark.parametrize("p", [2, 3])
def test_one_step_matches_exact_rational_arithmetic(p):
    # A and C symmetric but NOT commuting, so every transposition / product order matters.
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    Ck = np.array([[0.5, 0.125], [0.125, 0.375]])
    assert not np.allclose(A @ Ck, Ck @ A)
    Af, Cf = _fr(A), _fr(Ck)
    Z = _mm(Af, Cf)                         # Z_1 = A C
    for _ in range(2, p + 1):
        Z = _mm(Cf, Z)                      # Z_j = C Z_{j-1}
    R = [[(1 if i == j else 0) - Z[i][j] for j in range(2)] for i in range(2)]
    W = _mm(Cf, R)
    exact = [[Cf[i][j] + (W[i][j] + W[j][i]) / (2 * p) for j in range(2)] for i in range(2)]
    rho_exact = sum(float(R[i][j]) ** 2 for i in range(2) for j in range(2)) ** 0.5
    rho, nxt, _ = oracle.step_sym(A, Ck, p, oracle.phase())
    np.testing.assert_allclose(nxt, np.array(exact, dtype=float), rtol=2e-16, atol=1e-17)
    assert rho == pytest.approx(rho_exact, rel=1e-14)
    assert nxt[0, 1] == nxt[1, 0]           # exactly symmetric


def _mu_pred(p, li, lj):
    """Hand linearisation of G(C) = C + (W + W^T)/(2p) at X = A^{-1/p} (X^p A = I, XA = AX).
    In A's eigenbasis with x = lambda^{-1/p} and a symmetric perturbation E:
      d(C^{p-1} A C)_ij = E_ij g_ij,  g_ij = sum_{l=0}^{p-2} x_i^l x_j^{p-1-l} lambda_j + x_i^{p-1} lambda_i
      dW_ij = -x_i g_ij E_ij  (R(X) = 0),  so  mu_ij = 1 - (x_i g_ij + x_j g_ji) / (2p)."""
    xi, xj = li ** (-1.0 / p), lj ** (-1.0 / p)

    def g(xa, xb, la, lb):
        return sum(xa ** l * xb ** (p - 1 - l) * lb for l in range(p - 1)) + xa ** (p - 1) * la
    return 1.0 - (xi * g(xi, xj, li, lj) + xj * g(xj, xi, lj, li)) / (2 * p)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_linearisation_at_fixed_point_matches_derivation(p):
    n = 24
    A, lam, Q = synth.spd(n, 10.0, 7, return_eig=True)
    X = (Q * lam[None, :] ** (-1.0 / p)) @ Q.T
    X = (X + X.T) / 2
    _, X1, _ = oracle.step_sym(A, X, p, oracle.phase())
    eps = 1e-7
    for (i, j) in [(0, 1), (0, 5), (3, 9), (4, 4)]:
        E = np.outer(Q[:, i], Q[:, j])
        E = eps * (E + E.T)
        C = X + E
        C = (C + C.T) / 2
        _, C1, _ = oracle.step_sym(A, C, p, oracle.phase())
        mu = np.sum((C1 - X1) * E) / np.sum(E * E)
        assert mu == pytest.approx(_mu_pred(p, lam[i], lam[j]), abs=2e-5), (p, i, j)


def test_linearisation_predicts_stability_threshold():
    # the derived multiplier leaves the unit disc at kappa ~ 34 for p = 2 (SURVEY A12 measured
    # stable at 30, growing at 40)
    r = np.geomspace(1 / 30, 30, 2001)
    assert max(abs(_mu_pred(2, 1.0, x)) for x in r) < 1
    r = np.geomspace(1 / 40, 40, 2001)
    assert max(abs(_mu_pred(2, 1.0, x)) for x in r) > 1


@pytest.mark.parametrize("p", [2, 3])
def test_diagonal_limit_closed_form(p):
    a = np.array([0.3, 0.55, 0.8, 1.0, 0.9])
    r = oracle.solve(np.diag(a), p, [oracle.phase()], 1e-14, 200, form=SYM)
    assert r.outcome == oracle.CONVERGED
    np.testing.assert_allclose(np.diag(r.C_best), a ** (-1.0 / p), rtol=8 * 2.0 ** -52)
    assert np.count_nonzero(r.C_best - np.diag(np.diag(r.C_best))) == 0


@pytest.mark.parametrize("p", [2, 3, 4])
def test_twin_limit_is_eigen_root(p):
    A = synth.spd(64, 2.0, 0)
    r = oracle.solve(A, p, [oracle.phase()], 1e-12, 100, form=SYM)
    assert r.outcome == oracle.CONVERGED
    ref = np.real(scipy.linalg.fractional_matrix_power(A, -1.0 / p))
    assert np.linalg.norm(r.C_best - ref) / np.linalg.norm(ref) < 1e-12
    last = r.records[-1]
    assert last["rho_cert"] <= 1e-12          # certified ||I - C^p A||_F (reading R-3)


def test_iterates_exactly_symmetric_and_match_spectral_predictor():
    n, p = 48, 2
    A, lam, _ = synth.spd(n, 5.0, 2, return_eig=True)
    r = oracle.solve(A, p, [oracle.phase()], 0.0, 14, hist=14, form=SYM)
    for k in range(14):
        Ck = r.C_hist[k]
        assert np.array_equal(Ck, Ck.T), k
    # exact-arithmetic iterates are polynomials in A: rho_s(C_k) = ||I - C^p A||_F, so the
    # O(n) spectral recurrence of Eq. (1) predicts rho_hat until rounding matters
    pred = oracle.spectral(lam, p, r.s, 14)
    got = np.array([x["rho_hat"] for x in r.records[:14]])
    ok = pred > 1e-6
    np.testing.assert_allclose(got[ok], pred[ok], rtol=1e-8)


def test_mixed_precision_refinement_is_fast_where_literal_is_not():
    # literal Eq. (1) needs ~60 FP64 iterations after a BF16 phase (kappa = 2);
    # the symmetrised correction removes the non-commuting noise at rate max|mu| ~ 0.03.
    A = synth.spd(128, 2.0, 5)
    low = oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=60)
    lit = oracle.solve(A, 2, [low, oracle.phase()], 1e-12, 300)
    sym = oracle.solve(A, 2, [low, oracle.phase()], 1e-12, 300, form=SYM)
    sym_c = oracle.solve(A, 2, [low, oracle.phase(corr_prec=oracle.BF16)], 1e-12, 300, form=SYM)
    fp64 = oracle.solve(A, 2, [oracle.phase()], 1e-12, 300, form=SYM)
    n64 = lambda r: sum(1 for x in r.records if x["phase"] == 1)
    assert all(r.outcome == oracle.CONVERGED for r in (lit, sym, sym_c, fp64))
    assert n64(sym) <= 10 and n64(sym_c) <= 10 and n64(lit) >= 3 * n64(sym)
    assert n64(sym) < len(fp64.records)


def test_bf16_correction_in_fp64_phase_still_reaches_fp64_accuracy():
    A = synth.spd(96, 2.0, 1)
    r = oracle.solve(A, 2, [oracle.phase(corr_prec=oracle.BF16)], 1e-12, 100, form=SYM)
    ref = np.real(scipy.linalg.fractional_matrix_power(A, -0.5))
    assert r.outcome == oracle.CONVERGED
    assert np.linalg.norm(r.C_best - ref) / np.linalg.norm(ref) < 1e-12


def test_stable_at_kappa_10_where_literal_diverges():
    A = synth.spd(96, 10.0, 3)
    lit = oracle.solve(A, 2, [oracle.phase()], 1e-12, 120)
    sym = oracle.solve(A, 2, [oracle.phase()], 1e-12, 120, form=SYM)
    assert lit.outcome != oracle.CONVERGED
    assert sym.outcome == oracle.CONVERGED


def test_rejects_p1_and_scaled_correction():
    with pytest.raises(ValueError):
        oracle.solve(np.eye(4), 1, [oracle.phase()], form=SYM)
    with pytest.raises(ValueError):   # BF16 / TF32 / FP64, or the phase's own scaled format (R-29)
        oracle.solve(np.eye(4), 2, [oracle.phase(oracle.FP16, corr_prec=oracle.FP8), oracle.phase()], form=SYM)
    assert np.isnan(oracle.step_sym(np.eye(2), np.eye(2), 1, oracle.phase())[0])
    # scaled phases default to a BF16 correction and converge (FP16 -> FP64)
    A = synth.spd(64, 2.0, 0)
    r = oracle.solve(A, 2, [oracle.phase(oracle.FP16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
                            oracle.phase()], 1e-12, 100, form=SYM)
    assert r.outcome == oracle.CONVERGED


def test_tri_variant_mirrors_upper_triangle():
    # NEXT-2 (iii): Z_2 = C A C is symmetric in exact arithmetic; the tri variant uses its upper
    # triangle only.  Pins: (a) one tri step equals the full step with Z_2 symmetrised by its upper
    # triangle (hand-assembled from oracle GEMMs), (b) same limit, (c) exactly symmetric R means
    # the tri trajectory differs from the full one only at rounding level.
    TRI = oracle.FORM_SYMMETRIC_TRI
    A = synth.spd(40, 2.0, 6)
    full = oracle.solve(A, 2, [oracle.phase()], 1e-12, 60, hist=30, form=SYM)
    tri = oracle.solve(A, 2, [oracle.phase()], 1e-12, 60, hist=30, form=TRI)
    assert tri.outcome == oracle.CONVERGED
    assert abs(len(tri.records) - len(full.records)) <= 1
    np.testing.assert_allclose(tri.C_best, full.C_best, rtol=1e-13, atol=1e-15)
    # (a) the first step by hand: C_0 from the solve history
    C0 = tri.C_hist[0]
    Z1 = oracle.gemm(A, C0)
    Z2 = oracle.gemm(C0, Z1)
    Z2 = np.triu(Z2) + np.triu(Z2, 1).T
    R = np.eye(40) - Z2
    W = oracle.gemm(C0, R)
    C1 = C0 + (W + W.T) / 4
    np.testing.assert_array_equal(tri.C_hist[1], C1)
    assert tri.records[0]["rho"] == pytest.approx(np.linalg.norm(R), rel=1e-14)
    with pytest.raises(ValueError):
        oracle.solve(A, 3, [oracle.phase()], form=TRI)


def test_adaptive_digits_rule_pins():
    # R-26: the rule's accuracy property is pinned in tests/test_oracle_crt.py
    # (test_adaptive_digit_rule_property: the product error at the chosen digits stays below t / 2);
    # here its range and the in-phase behaviour: S saturates at 3 and 9, precision rises inside the
    # phase and the solve still reaches the certified FP64 residual.
    assert oracle.oz_digits(1.0, 64) == 3 and oracle.oz_digits(1e-30, 8192) == 9
    assert oracle.oz_digits(float("nan"), 64) == 9 and oracle.oz_digits(0.0, 64) == 9
    A = synth.spd(96, 2.0, 4)
    low = oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    r = oracle.solve(A, 2, [low, oracle.phase(oracle.FP64_OZ, mant_bits=oracle.MANT_ADAPTIVE)], 1e-12, 80,
                     form=SYM)
    ms = [x["mant_bits"] for x in r.records if x["phase"] == 1]
    assert r.outcome == oracle.CONVERGED and ms == sorted(ms) and ms[0] < 52 and ms[-1] == 52


@pytest.mark.parametrize("prec", [oracle.FP8, oracle.FP16, oracle.INT8])
def test_scaled_correction_step_is_exact_newton_step(prec):
    # R-29 pin: with A = s D_a, C = D_c / sqrt(s) diagonal and every intermediate (a c, c^2 a,
    # R = 1 - c^2 a, c R) exact in E4M3 / FP16 / INT8 after power-of-two scaling, one symmetric
    # step with a scaled correction (corr = prec) must equal the exact Newton step of Eq. (1)
    # c' = c + c (1 - c^p a) / p for p = 2.  s = 2^20 makes sigma_C, sigma_A,
    # sigma_Z and sigma_R all non-zero and different: dropping or mixing up any unscale fails.
    s = 2.0 ** 20
    a = np.array([1.0, 1.0, 4.0, 1.0]) * s
    c = np.array([0.75, 1.0, 0.25, 0.5]) / np.sqrt(s)     # R = 0.4375, 0, 0.75, 0.75
    if prec == oracle.INT8:                               # INT8: 7-bit fixed point relative to the max
        c = np.array([0.75, 1.0, 0.5, 0.5]) / np.sqrt(s)  # R = 0.4375, 0, 0.75, 0.75 (a = 1, 1, 1, 1)
        a = np.full(4, s)
    A, C = np.diag(a), np.diag(c)
    ph = oracle.phase(prec, mant_bits=23, corr_prec=prec)
    rho, C1, _ = oracle.step_sym(A, C, 2, ph)
    R = 1.0 - c * c * a
    np.testing.assert_array_equal(C1, np.diag(c + c * R / 2.0))
    assert rho == pytest.approx(np.sqrt(np.sum(R * R)), rel=1e-15)


def test_fp8_correction_schedule_converges():
    # R-29: FP8 phase with an FP8 correction, then BF16, then FP64 (the bench's low phases):
    # converges to the same root; the FP8 phase's rate is slower than with a BF16 correction
    # by at most a few iterations (|mu| + 2^-4 per step)
    A = synth.spd(96, 2.0, 5)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    ref = np.real(scipy.linalg.fractional_matrix_power(A, -0.5))
    counts = {}
    for corr in (oracle.FP8, oracle.BF16):
        r = oracle.solve(A, 2, [oracle.phase(oracle.FP8, corr_prec=corr, **low), oracle.phase(oracle.BF16, **low),
                                oracle.phase()], 1e-12, 150, form=oracle.FORM_SYMMETRIC_TRI)
        assert r.outcome == oracle.CONVERGED
        assert np.linalg.norm(r.C_best - ref) / np.linalg.norm(ref) < 1e-12
        counts[corr] = sum(1 for x in r.records if x["phase"] == 0)
    assert counts[oracle.FP8] <= counts[oracle.BF16] + 4, counts


@pytest.mark.parametrize("form,p", [(SYM, 2), (SYM, 3), (oracle.FORM_SYMMETRIC_TRI, 2)])
def test_certificate_first_rule(form, p):
    # reading R-33: with the last phase's rate predicting rho_{k+1} = rho_k^2 / rho_{k-1} <= tol / 2 the
    # next iterate is certified before its chain (the BF16 -> FP64 schedule: noise-driven linear rate).
    # Pinned: (a) the same iterates and records as the chain-triggered solve, except (b) the last record
    # is certificate-only (rho NaN) with the same certificate value of the same iterate, (c) that value
    # is the FP64 residual ||I - C^p A||_F of the returned C (numpy's own product, within the FP64
    # rounding of an O(1e-13) quantity) and <= tol, (d) the rule fired exactly where the rate predicted.
    A = synth.spd(96, 2.0, 7)
    ph = [oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
          oracle.phase(corr_prec=oracle.BF16)]
    a = oracle.solve(A, p, ph, 1e-12, 100, hist=100, form=form, predict_cert=True)
    b = oracle.solve(A, p, ph, 1e-12, 100, hist=100, form=form, predict_cert=False)
    assert a.outcome == oracle.CONVERGED and b.outcome == oracle.CONVERGED
    assert len(a.records) == len(b.records)
    for k in range(len(a.records)):
        np.testing.assert_array_equal(a.C_hist[k], b.C_hist[k])
    for x, y in zip(a.records[:-1], b.records[:-1]):
        assert x["rho"] == y["rho"] and x["decision"] == y["decision"]
    last, lb = a.records[-1], b.records[-1]
    assert np.isnan(last["rho"]) and np.isfinite(lb["rho"]) and last["decision"] == oracle.CONVERGED
    assert last["rho_cert"] == lb["rho_cert"] <= 1e-12
    np.testing.assert_array_equal(a.C_best, b.C_best)
    E = np.eye(96) - np.linalg.matrix_power(a.C_best, p) @ A
    assert abs(last["rho_cert"] - np.linalg.norm(E)) <= 1e-13
    r1, r2 = a.records[-2]["rho"], a.records[-3]["rho"]
    assert a.records[-2]["phase"] == a.records[-3]["phase"] == 1
    assert r1 * (r1 / r2) <= 0.5e-12
    for x, y in zip(a.records[1:-2], a.records[:-3]):   # and no earlier record predicted it
        if x["phase"] == y["phase"] == 1 and x["decision"] == oracle.CONTINUE and x["rho"] < y["rho"]:
            assert x["rho"] * (x["rho"] / y["rho"]) > 0.5e-12


def test_missed_certificates_respect_the_phase_cap():
    # a tolerance between the in-chain floor and the FP64 certificate's own rounding floor: every
    # certificate misses; the last phase's iteration cap must still end the solve (ITER_LIMIT), as for
    # any other last-phase iteration (the GPU engine mirrors it: tests/test_gpu_symmetric.py)
    A = synth.spd(200, 2.0, 13)
    cap = 12
    ph = [oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
          oracle.phase(corr_prec=oracle.BF16, max_iters=cap)]
    tol = 2.85e-15                    # n = 200: in-chain floor ~2.5e-15, FP64 certificate floor ~3e-15
    r = oracle.solve(A, 2, ph, tol, 200, form=SYM)
    certs = [x for x in r.records if x["rho_cert"] == x["rho_cert"]]
    assert r.outcome == oracle.ITER_LIMIT, [(x["rho"], x["rho_cert"]) for x in r.records[-6:]]
    assert sum(1 for x in r.records if x["phase"] == 1) == cap
    assert len(certs) >= 2 and all(x["rho_cert"] > tol for x in certs)
    assert r.records[-1]["decision"] == oracle.ITER_LIMIT and r.records[-1]["rho"] <= tol


def test_tri_form_low_phase_correction_from_upper_triangle():
    # reading R-36: below the FP64 range the symmetric forms take Z_1 = A C and W = C R from their upper
    # triangles -- Z_1 := mirror(upper(A C)), S_ij = 2 W_{min(i,j), max(i,j)}.  Pinned on a non-commuting
    # 2 x 2 whose every intermediate is exact in BF16 (hand values):
    #   A C = [[9/8, 5/8], [7/8, 5/4]] -> Z_1 = [[9/8, 5/8], [5/8, 5/4]], Z_2 = mirror(upper(C Z_1)) =
    #   [[41/64, 15/32], [15/32, 35/64]], R = I - Z_2, W = C R = [[31/256, -91/512], [-67/512, 57/512]]
    # (the full symmetric form too, below the FP64 range: the same mirrored products), and for an FP64 phase
    # (no mirroring of Z_1, S = W + W^T):
    #   Z_2 = [[43/64, 15/32], [15/32, 35/64]], W = [[27/256, -91/512], [-69/512, 57/512]]
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    Ck = np.array([[0.5, 0.125], [0.125, 0.375]])
    W = np.array([[31 / 256, -91 / 512], [-67 / 512, 57 / 512]])
    Z2 = np.array([[41 / 64, 15 / 32], [15 / 32, 35 / 64]])
    up = np.array([[2 * W[0, 0], 2 * W[0, 1]], [2 * W[0, 1], 2 * W[1, 1]]])
    ph = oracle.phase(oracle.BF16)
    rho, C1, _ = oracle.step_sym(A, Ck, 2, ph, tri=True)
    np.testing.assert_array_equal(C1, oracle.qm(Ck + up / 4, 8, 7))
    assert rho == pytest.approx(np.linalg.norm(np.eye(2) - Z2), rel=1e-15)
    assert not np.array_equal(oracle.qm(Ck + (W + W.T) / 4, 8, 7), C1)
    Wf = np.array([[27 / 256, -91 / 512], [-69 / 512, 57 / 512]])
    Z2f = np.array([[43 / 64, 15 / 32], [15 / 32, 35 / 64]])
    rs, C1s, _ = oracle.step_sym(A, Ck, 2, ph, tri=False)
    np.testing.assert_array_equal(C1s, C1)
    assert rs == rho
    rf, C1f, _ = oracle.step_sym(A, Ck, 2, oracle.phase(), tri=True)
    np.testing.assert_array_equal(C1f, Ck + (Wf + Wf.T) / 4)
    assert rf == pytest.approx(np.linalg.norm(np.eye(2) - Z2f), rel=1e-15)


def test_symmetric_form_p3_low_phase_products_from_upper_triangles():
    # R-36 for p = 3 (the full symmetric form): below the FP64 range every Z_j and W come from their upper
    # triangles; on an A that commutes with C (both diagonal in the same basis, here diagonal) the mirrored
    # and the full products agree exactly, so one BF16 step equals the exact Newton step of Eq. (1) on
    # exactly representable values (hand values: c' = c + c (1 - c^3 a) / 3 with c^3 a in {1/8, 1, 27/64})
    a = np.array([1.0, 1.0, 1.0])
    c = np.array([0.5, 1.0, 0.75])
    A, Ck = np.diag(a), np.diag(c)
    rho, C1, _ = oracle.step_sym(A, Ck, 3, oracle.phase(oracle.BF16, mant_bits=23, corr_prec=oracle.TF32))
    r = 1 - c ** 3 * a
    np.testing.assert_array_equal(C1, np.diag(oracle.qm(c + c * r / 3, 8, 23)))
    assert rho == pytest.approx(np.sqrt(np.sum(r ** 2)), rel=1e-15)


def test_triz_chain_takes_z1_from_its_upper_triangle_in_an_fp64_crt_phase():
    # reading R-37 (FORM_SYMMETRIC_TRIZ): a chain of an FP64_CRT phase that the rule selects (tri = 2)
    # mirrors Z_1 = A C as well; W + W^T stays full.  The non-commuting 2 x 2 of the R-36 pin (every
    # intermediate a short dyadic, so the CRT products are exact), hand values:
    #   Z_1 = mirror(upper([[9/8, 5/8], [7/8, 5/4]])) = [[9/8, 5/8], [5/8, 5/4]],
    #   Z_2 = mirror(upper(C Z_1)) = [[41/64, 15/32], [15/32, 35/64]], W = C (I - Z_2) =
    #   [[31/256, -91/512], [-67/512, 57/512]], C' = C + (W + W^T) / 4
    # against the tri form's own FP64-range chain (tri = 1, Z_1 in full): Z_2 = [[43/64, ...]], W = Wf.
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    Ck = np.array([[0.5, 0.125], [0.125, 0.375]])
    W = np.array([[31 / 256, -91 / 512], [-67 / 512, 57 / 512]])
    Z2 = np.array([[41 / 64, 15 / 32], [15 / 32, 35 / 64]])
    ph = oracle.phase(oracle.FP64_CRT)
    rho, C1, _ = oracle.step_sym(A, Ck, 2, ph, tri=2)
    np.testing.assert_array_equal(C1, Ck + (W + W.T) / 4)
    assert rho == pytest.approx(np.linalg.norm(np.eye(2) - Z2), rel=1e-15)
    Wf = np.array([[27 / 256, -91 / 512], [-69 / 512, 57 / 512]])
    rf, C1f, _ = oracle.step_sym(A, Ck, 2, ph, tri=1)
    np.testing.assert_array_equal(C1f, Ck + (Wf + Wf.T) / 4)
    assert rf != rho


def _crt_schedule(n):
    sw = 2.0 * 2.0 ** -8 * np.sqrt(n)
    return [oracle.phase(oracle.BF16, switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
            oracle.phase(oracle.FP64_CRT, mant_bits=oracle.MANT_ADAPTIVE, corr_prec=oracle.BF16)]


def test_triz_rule_selects_chains_by_the_in_phase_contraction():
    # R-37's rule, replayed from the solve's own iterates: chain k of the FP64_CRT phase takes Z_1 from its upper
    # triangle iff two in-phase residuals exist and every in-phase ratio so far was <= 0.1.  Each recorded
    # residual must equal the one-step oracle's for the chain kind the rule gives -- and differ from the other kind
    n = 96
    A = synth.spd(n, 2.0, 3)
    ph = _crt_schedule(n)
    r = oracle.solve(A, 2, ph, 1e-12, 80, hist=80, form=oracle.FORM_SYMMETRIC_TRIZ, cert="crt")
    assert r.outcome == oracle.CONVERGED and r.records[-1]["rho_cert"] <= 1e-12
    rhos, ok, ntri = [], True, 0
    for rec in r.records:
        if rec["phase"] != 1 or not np.isfinite(rec["rho"]):
            continue
        tri2 = ok and len(rhos) >= 2
        # the replay runs the chain at S = 9 digits, the solve at R-26's adaptive digits: they agree to the
        # chain's own error level (~2e-4 relative at the lowest S), the two chain kinds differ by ~2e-2
        one = oracle.phase(oracle.FP64_CRT, mant_bits=oracle.MANT_ADAPTIVE, corr_prec=oracle.BF16)
        got = {t: oracle.step_sym(A, r.C_hist[rec["k"]], 2, one, want_next=False, tri=t)[0] for t in (1, 2)}
        want, other = got[2 if tri2 else 1], got[1 if tri2 else 2]
        assert abs(rec["rho"] - want) < 0.2 * abs(rec["rho"] - other), (rec["k"], tri2, rec["rho"], want, other)
        ntri += tri2
        rhos.append(rec["rho"])
        if len(rhos) >= 2 and not rhos[-1] <= 0.1 * rhos[-2]:
            ok = False
    assert ntri >= 3 and len(rhos) - ntri == 2


def test_triz_equals_tri_where_the_phase_contracts_slowly():
    # kappa = 5: the FP64_CRT phase's first in-phase ratio is above 0.1, the rule switches itself off for good
    # and the trajectory is the tri form's, record for record
    n = 96
    A = synth.spd(n, 5.0, 2)
    ph = _crt_schedule(n)
    a = oracle.solve(A, 2, ph, 1e-12, 120, form=oracle.FORM_SYMMETRIC_TRI, cert="crt")
    b = oracle.solve(A, 2, ph, 1e-12, 120, form=oracle.FORM_SYMMETRIC_TRIZ, cert="crt")
    assert a.outcome == b.outcome == oracle.CONVERGED
    assert [x["rho"] for x in a.records if np.isfinite(x["rho"])] == [x["rho"] for x in b.records if np.isfinite(x["rho"])]
    np.testing.assert_array_equal(a.C_best, b.C_best)
