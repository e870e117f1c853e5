"""Pins of the oracle's NEXT-2 (ii) coupled form (reading R-27):
M = X^p A, N = ((p+1) I - M)/p, X_{k+1} = X_k N_k, M_{k+1} = N_k^p M_k, M re-anchored per phase.
Pinned against hand values, the literal form it equals in exact arithmetic (an independent
implementation: Eq. (1)'s chain), the eigen-decomposition limit, and SURVEY Table A3's behaviour
(bounded where Eq. (1) diverges; frozen low-precision noise)."""
import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

CPL = oracle.FORM_COUPLED


def test_scalar_hand_values():
    # A = [4]: C0 = 4 / 16 = 0.25; M0 = 0.25^2 * 4 = 0.25 (rho 0.75); N0 = (3 - 0.25)/2 = 1.375;
    # X1 = 0.34375 (= Eq. (1): (3 * 0.25 - 0.25^3 * 4)/2); M1 = N0^2 M0 = 0.47265625 (rho 0.52734375)
    r = oracle.solve(np.array([[4.0]]), 2, [oracle.phase()], 0.0, 3, hist=3, form=CPL)
    assert [h[0, 0] for h in r.C_hist[:2]] == [0.25, 0.34375]
    assert [x["rho"] for x in r.records[:2]] == [0.75, 0.52734375]


@pytest.mark.parametrize("p", [1, 2, 3])
def test_equals_literal_form_early(p):
    # in exact arithmetic the coupled iterates ARE Eq. (1)'s; in FP64 they agree to rounding
    A = synth.spd(64, 2.0, 3)
    lit = oracle.solve(A, p, [oracle.phase()], 0.0, 8, hist=8)
    cpl = oracle.solve(A, p, [oracle.phase()], 0.0, 8, hist=8, form=CPL)
    for k in range(8):
        assert np.linalg.norm(lit.C_hist[k] - cpl.C_hist[k]) <= 1e-13 * np.linalg.norm(lit.C_hist[k])


@pytest.mark.parametrize("p", [1, 2, 3])
def test_twin_limit_and_certificate(p):
    A = synth.spd(64, 2.0, 0)
    r = oracle.solve(A, p, [oracle.phase()], 1e-12, 100, form=CPL)
    assert r.outcome == oracle.CONVERGED and r.records[-1]["rho_cert"] <= 1e-12
    ref = np.real(scipy.linalg.fractional_matrix_power(A, -1.0 / p))
    assert np.linalg.norm(r.C_best - ref) / np.linalg.norm(ref) < 1e-12


def test_bounded_where_literal_diverges():
    # SURVEY Table A3: coupled p = 2 at kappa = 1e3 reaches ~3e-7 and stays bounded; Eq. (1) diverges
    n = 256
    A = synth.spd(n, 1e3, 1)
    lit = oracle.solve(A, 2, [oracle.phase()], 1e-12, 120)
    cpl = oracle.solve(A, 2, [oracle.phase()], 1e-12, 120, form=CPL)
    assert lit.outcome in (oracle.DIVERGED, oracle.NONFINITE) or lit.rho.min() > 1.0
    X = cpl.C_best
    assert np.linalg.norm(np.eye(n) - X @ X @ A) < 1e-5
    assert np.isfinite(cpl.rho).all() and cpl.rho[-10:].max() < 1e-12      # M stays at I


def test_low_precision_noise_is_frozen():
    # the coupled form cannot remove noise a BF16 phase left in X:
    # ||I - M|| reaches the FP64 floor while the certified ||I - X^2 A|| stays at the BF16 level
    A = synth.spd(128, 2.0, 3)
    low = oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    r = oracle.solve(A, 2, [low, oracle.phase()], 1e-12, 40, form=CPL)
    assert r.outcome != oracle.CONVERGED
    assert min(x["rho"] for x in r.records) < 1e-13
    cert = [x["rho_cert"] for x in r.records if x["rho_cert"] == x["rho_cert"]]
    assert cert and min(cert) > 1e-3
