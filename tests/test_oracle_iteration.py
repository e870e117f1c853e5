"""Pins of the oracle's iteration (Eq. 1-3, PAPER.md:66-88 [Sec. 2]) against hand values,
closed forms, library routines (numpy/scipy), brute force, invariants and the spectral
predictor (an independent O(n) recurrence of the exact-arithmetic iteration)."""
import math

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth
from tests import golden

G = golden.load()


def _rows(kind):
    return [k for k, v in G.items() if v["kind"] == kind]


@pytest.mark.parametrize("name", _rows("step"))
def test_golden_step(name):
    g = G[name]
    A = golden.matrix(g["inputs"]["A"])
    Ck = golden.matrix(g["inputs"]["C"])
    rho, nxt, _ = oracle.step(A, Ck, int(g["inputs"]["p"]), oracle.phase())
    np.testing.assert_allclose(nxt, np.atleast_2d(g["expected"]), rtol=1e-15, atol=1e-16,
                               err_msg=g["cite"])


@pytest.mark.parametrize("name", _rows("rho"))
def test_golden_residual(name):
    g = G[name]
    rho, _, _ = oracle.step(golden.matrix(g["inputs"]["A"]), golden.matrix(g["inputs"]["C"]),
                            int(g["inputs"]["p"]), oracle.phase(), want_next=False)
    assert rho == pytest.approx(g["expected"], rel=1e-15), g["cite"]


def test_golden_bf16_step():
    g = G["step_bf16_scalar"]
    _, nxt, _ = oracle.step(np.array([[4.0]]), np.array([[0.4]]), 2, oracle.phase(oracle.BF16))
    assert nxt[0, 0] == g["expected"], g["cite"]


def test_golden_c0():
    g = G["c0_diag22"]
    A = golden.matrix(g["inputs"]["A"])
    n1, ninf, md = oracle.norms(A)
    np.testing.assert_array_equal(oracle.c0(A, n1 * ninf, oracle.phase()), np.array(g["expected"]))


def test_golden_diag_roots():
    g = G["root_diag_4_9"]
    r = oracle.solve(golden.matrix(g["inputs"]["A"]), 2, [oracle.phase()], 1e-14, 200)
    assert r.outcome == oracle.CONVERGED
    np.testing.assert_allclose(np.diag(r.C_best), g["expected"], rtol=4e-16)
    g = G["root_diag_4_16"]
    lam, V = oracle.jacobi(golden.matrix(g["inputs"]["A"]))
    np.testing.assert_allclose(np.diag(oracle.inv_proot_eig(lam, V, 2)), g["expected"], rtol=1e-15)


def test_norms_vs_numpy():
    A = synth.spd(96, 50.0, 3)
    n1, ninf, md = oracle.norms(A)
    assert n1 == pytest.approx(np.linalg.norm(A, 1), rel=1e-14)
    assert ninf == pytest.approx(np.linalg.norm(A, np.inf), rel=1e-14)
    assert md == np.max(np.diag(A))
    B = np.arange(12.0).reshape(3, 4)[:, :3] - 4.0   # integer-valued: sums are exact
    B = np.ascontiguousarray(B)
    n1, ninf, _ = oracle.norms(B)
    assert n1 == np.abs(B).sum(0).max() and ninf == np.abs(B).sum(1).max()
    assert n1 != ninf                                   # catches a swapped row/column sum


def test_symmetry_check():
    A = synth.spd(32, 10.0, 0)
    assert oracle.is_symmetric(A)
    B = A.copy()
    B[3, 7] = np.nextafter(B[3, 7], 1.0)
    assert not oracle.is_symmetric(B)
    with pytest.raises(ValueError):
        oracle.solve(B, 2, [oracle.phase()])


def test_gemm_vs_numpy_and_exact_integers():
    rng = np.random.default_rng(7)
    X, Y = rng.standard_normal((70, 70)), rng.standard_normal((70, 70))
    Z = oracle.gemm(X, Y)
    bound = 70 * 2.0 ** -53 * (np.abs(X) @ np.abs(Y))
    assert np.all(np.abs(Z - X @ Y) <= 2 * bound)
    Xi = rng.integers(-50, 50, (33, 33)).astype(float)
    Yi = rng.integers(-50, 50, (33, 33)).astype(float)
    np.testing.assert_array_equal(oracle.gemm(Xi, Yi), Xi @ Yi)   # orientation + exactness


def test_gemm_rows_matches_gemm():
    rng = np.random.default_rng(8)
    X, Y = rng.standard_normal((40, 40)), rng.standard_normal((40, 40))
    Z = np.zeros((40, 40))
    oracle.gemm_rows(X, Y, Z, 5, 17)
    np.testing.assert_array_equal(Z[5:17], oracle.gemm(X, Y)[5:17])
    assert np.all(Z[:5] == 0) and np.all(Z[17:] == 0)


def test_c0_is_scaled_transpose():
    A = synth.spd(40, 10.0, 1)
    n1, ninf, _ = oracle.norms(A)
    np.testing.assert_array_equal(oracle.c0(A, n1 * ninf, oracle.phase()), A.T / (n1 * ninf))
    c0b = oracle.c0(A, n1 * ninf, oracle.phase(oracle.BF16))
    ref = (A.T / (n1 * ninf)).astype(np.float32)
    import torch
    refb = torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
    # single rounding from FP64 vs rounding via FP32 may differ only on double-rounding ties
    assert np.mean(c0b == refb) > 0.999


def test_identity_is_fixed_point():
    # A = I: s = 1, C_0 = I, rho = 0.
    r = oracle.solve(np.eye(8), 3, [oracle.phase()], 1e-12, 10)
    assert r.outcome == oracle.CONVERGED and r.records[0]["rho"] == 0.0
    np.testing.assert_array_equal(r.C_best, np.eye(8))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_diagonal_limit_closed_form(p):
    # P4: diagonal A -> diag(a_i^{-1/p}), off-diagonals exactly zero.
    A = synth.diag_spd(24, 1e3, p)
    r = oracle.solve(A, p, [oracle.phase()], 0.0, 400)
    C = r.C_best
    a = np.diag(A)
    assert np.all(C[~np.eye(24, dtype=bool)] == 0.0)
    np.testing.assert_allclose(np.diag(C), a ** (-1.0 / p), rtol=8 * 2.0 ** -52)


def test_jacobi_vs_numpy_eigh():
    A = synth.spd(48, 30.0, 2)
    lam, V = oracle.jacobi(A)
    ref = np.linalg.eigvalsh(A)
    np.testing.assert_allclose(lam, ref, rtol=1e-13)
    np.testing.assert_allclose(V @ np.diag(lam) @ V.T, A, atol=1e-13)
    np.testing.assert_allclose(V.T @ V, np.eye(48), atol=1e-13)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_inv_proot_eig_vs_scipy(p):
    A = synth.spd(32, 20.0, 4)
    lam, V = oracle.jacobi(A)
    X = oracle.inv_proot_eig(lam, V, p)
    ref = np.real(scipy.linalg.fractional_matrix_power(A, -1.0 / p))
    np.testing.assert_allclose(X, ref, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_stable_twin_converges_to_root(p):
    # kappa = 2 < kappa_p: FP64 reaches rho <= 1e-12 and the limit A^{-1/p}.
    A = synth.spd(64, 2.0, 0)
    r = oracle.solve(A, p, [oracle.phase()], 1e-12, 100)
    assert r.outcome == oracle.CONVERGED and r.records[-1]["rho"] <= 1e-12
    lam, V = oracle.jacobi(A)
    X = oracle.inv_proot_eig(lam, V, p)
    assert np.linalg.norm(r.C_best - X) / np.linalg.norm(X) < 1e-12
    if p == 1:   # P7: Newton-Schulz: C A = I
        assert np.linalg.norm(r.C_best @ A - np.eye(64)) < 1e-12


def test_spectral_predictor_matches_trajectory():
    # P5: rho_hat_k of the matrix iteration equals the eigenvalue recurrence until rounding.
    A, lam, _ = synth.spd(128, 10.0, 5, return_eig=True)
    r = oracle.solve(A, 2, [oracle.phase()], 0.0, 30)
    pred = oracle.spectral(lam, 2, r.s, 30)
    got = np.array([x["rho_hat"] for x in r.records])
    mask = pred[: got.size] > 1e-7
    assert mask.sum() > 10
    np.testing.assert_allclose(got[mask], pred[: got.size][mask], rtol=1e-9)
    # the spectral predictor at k = 0 is Eq. (2) in eigen-space: t_i in (0, 2) (P9)
    t0 = lam ** 3 / r.s ** 2
    assert np.all((t0 > 0) & (t0 < 2))


def test_spectral_predictor_closed_form_scalar():
    # n = 1: t_0 = a^{p+1}/s^p with s = a^2 -> t_0 = a^{1-p}; one step by hand for a = 4, p = 2:
    # t_0 = 0.25, t_1 = 0.25 * ((3 - 0.25)/2)^2 = 0.47265625.
    out = oracle.spectral(np.array([4.0]), 2, 16.0, 2)
    assert out[0] == 0.75 and out[1] == pytest.approx(1 - 0.47265625, rel=1e-15)


def test_contraction_golden():
    g = G["contraction_scalar"]   # Eq. (2) value |1 - C0^p A| for a 1x1 case
    rho, _, _ = oracle.step(np.array([[4.0]]), np.array([[0.0625]]), 2, oracle.phase(), False)
    assert rho == g["expected"]


def test_invariants_stable_regime():
    # P8: exact iterates are polynomials in A -> symmetric and commuting with A.
    A, lam, _ = synth.spd(64, 2.0, 6, return_eig=True)
    r = oracle.solve(A, 2, [oracle.phase()], 1e-12, 40, hist=40, gamma_normA2=float(lam.max()))
    for k, rec in enumerate(r.records):
        Ck = r.C_hist[k]
        assert np.linalg.norm(Ck - Ck.T) <= 1e-14 * np.linalg.norm(Ck)
        assert rec["gamma"] < 1e-14


def test_unstable_config_c1_behaviour():
    # Config C1 (n=64, kappa=1e2, p=2, FP64): Eq. (1) is only locally stable for kappa < 2.44
    # (SURVEY F2), so rho bottoms out (~5e-5) and then diverges; the best iterate is returned.
    c = synth.CONFIGS["C1"]
    A = synth.spd(c["n"], c["kappa"], c["seed"])
    r = oracle.solve(A, 2, [oracle.phase()], 1e-12, 200)
    assert r.outcome == oracle.DIVERGED
    rho = r.rho
    kmin = int(np.argmin(rho))
    assert 1e-7 < rho[kmin] < 1e-3 and kmin > 15
    lam, V = oracle.jacobi(A)
    X = oracle.inv_proot_eig(lam, V, 2)
    assert np.linalg.norm(r.C_best - X) / np.linalg.norm(X) < 10 * rho[kmin]


def test_rtz_storage_and_plateau_ordering():
    # P12 / PAPER.md:256-258: the precision-limited plateau rises as stored bits fall.
    A = synth.spd(64, 2.0, 7)
    mins = []
    for m in [4, 7, 10, 16, 23]:
        r = oracle.solve(A, 2, [oracle.phase(oracle.FP64, mant_bits=m)], 0.0, 40)
        mins.append(r.rho.min())
    assert all(a >= b for a, b in zip(mins, mins[1:])), mins
    assert mins[0] > 1e3 * mins[-1]


def test_iterations_grow_with_p():
    # more iterations as p grows (exact-arithmetic counts, kappa = 2).
    A = synth.spd(64, 2.0, 8)
    its = []
    for p in [1, 2, 3, 4]:
        r = oracle.solve(A, p, [oracle.phase()], 1e-12, 100)
        assert r.outcome == oracle.CONVERGED
        its.append(len(r.records))
    assert its == sorted(its), its


def test_mixed_schedule_reaches_fp64():
    # BF16 phase (armed plateau, R-5) then FP64 refinement on the stable twin.
    A = synth.spd(64, 2.0, 9)
    ph = [oracle.phase(oracle.BF16, switch_tol=1e-2, plateau_ratio=0.7, plateau_arm=0.5,
                       max_iters=40), oracle.phase(oracle.FP64)]
    r = oracle.solve(A, 2, ph, 1e-12, 300)
    assert r.outcome == oracle.CONVERGED
    phases = [x["phase"] for x in r.records]
    assert phases[0] == 0 and phases[-1] == 1 and phases == sorted(phases)
    sw = [x for x in r.records if x["decision"] == oracle.SWITCH]
    assert len(sw) == 1 and sw[0]["rho"] <= 1e-2 * 10


def test_fp16_phase_scaling_keeps_small_entries():
    # Reading R-20: scaled FP16 operands; without the scale 2^-24 would flush C0's small entries.
    A = synth.spd(128, 10.0, 11)
    r = oracle.solve(A, 2, [oracle.phase(oracle.FP16, max_iters=40)], 0.0, 40)
    rb = oracle.solve(A, 2, [oracle.phase(oracle.BF16, max_iters=40)], 0.0, 40)
    assert r.rho.min() < rb.rho.min()         # 10 stored bits beat 7


def test_matvec_probe():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((50, 50))
    v = synth.probe_vectors(50, 1, 0)[0]
    np.testing.assert_allclose(oracle.matvec(X, v), X @ v, rtol=1e-13, atol=1e-13)
