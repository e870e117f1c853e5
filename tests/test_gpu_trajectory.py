"""GPU trajectory parity (Levels 0-3 of DESIGN.md "Parity contract"), through the C-ABI.

Level 0: diagonal A -> every iterate bit-identical to the oracle (each dot product has one
         non-zero term, so only the epilogue's fixed FP64 op order matters).
Level 2: stable kappa=2 twins -> FP64 iterates within 1e-10 relative, same iteration count,
         final rho <= 1e-12 (north star tolerances).
Level 3: BASELINE config C1 (unstable regime): Level-2 tolerances until the oracle's
         commutator diagnostic gamma_k exceeds tol/4, then envelope agreement.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")


@pytest.mark.parametrize("p", [1, 2, 3])
def test_diagonal_bit_exact_fp64(p):
    A = synth.diag_spd(100, 1e3, p)
    r = oracle.solve(A, p, [oracle.phase()], 0.0, 60, hist=60)
    out, tr, hist, best = run_gpu_trajectory(A, p, [ipr.make_phase("fp64")], 0.0, 60)
    assert len(tr) == len(r.records)
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)
    rg = np.array([t["rho"] for t in tr])
    np.testing.assert_allclose(rg, r.rho, rtol=1e-13, atol=1e-300)
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]


@pytest.mark.parametrize("m,rtz", [(7, 0), (16, 1), (23, 0)])
def test_diagonal_bit_exact_storage_sweep(m, rtz):
    A = synth.diag_spd(64, 1e2, 7)
    phs_o = [oracle.phase(oracle.FP64, mant_bits=m, round=rtz, plateau_ratio=0.7, plateau_arm=0.5),
             oracle.phase(oracle.FP64)]
    phs_g = [ipr.make_phase("fp64", mant_bits=m, round=rtz, plateau_ratio=0.7, plateau_arm=0.5),
             ipr.make_phase("fp64")]
    r = oracle.solve(A, 3, phs_o, 1e-13, 80, hist=80)
    out, tr, hist, best = run_gpu_trajectory(A, 3, phs_g, 1e-13, 80)
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)


@pytest.mark.parametrize("n,p", [(300, 2), (256, 1), (200, 3)])
def test_stable_twin_fp64(n, p):
    A = synth.spd(n, 2.0, 5)
    r = oracle.solve(A, p, [oracle.phase()], 1e-12, 60, hist=60)
    assert r.outcome == oracle.CONVERGED
    out, tr, hist, best = run_gpu_trajectory(A, p, [ipr.make_phase("fp64")], 1e-12, 60)
    assert out == ipr.IPR_CONVERGED
    # same iteration count (R-6: +-1 only if the oracle's crossing is within 1e-10 of the tol)
    rr = r.records[-1]["rho"]
    if abs(rr - 1e-12) > 1e-10 * 1e-12:
        assert len(tr) == len(r.records)
    for k, Ck in hist.items():
        if k < len(r.records):
            assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    assert tr[-1]["rho"] <= 1e-12
    assert rel_fro(best, r.C_best) <= 1e-10
    if p == 1:  # Newton-Schulz limit C A = I
        assert np.linalg.norm(best @ A - np.eye(n)) < 1e-11


def test_certified_residual_fp64():
    A = synth.spd(256, 2.0, 6)
    s = ipr.Solver(torch.from_numpy(A).cuda(), 2, [ipr.make_phase("fp64")], 1e-12)
    assert s.iterate(100) == ipr.IPR_CONVERGED
    rin, rc = s.residual(False), s.residual(True)
    # literal form, FP64 phase: the in-chain residual is the literal DMMA chain of the returned
    # iterate, i.e. the certificate itself (R-30)
    assert rin <= 1e-12 and rc == rin
    s.close()


def test_config_c1_level3():
    c = synth.CONFIGS["C1"]
    A, lam, _ = synth.spd(c["n"], c["kappa"], c["seed"], return_eig=True)
    r = oracle.solve(A, 2, [oracle.phase()], 1e-12, 120, hist=120, gamma_normA2=float(lam.max()))
    out, tr, hist, best = run_gpu_trajectory(A, 2, [ipr.make_phase("fp64")], 1e-12, 120)
    gam = np.array([x["gamma"] for x in r.records])
    kstar = int(np.argmax(gam > 2.5e-11)) if np.any(gam > 2.5e-11) else len(gam)
    assert kstar > 10
    for k, Ck in hist.items():
        if k < kstar:
            assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    rg = np.array([t["rho"] for t in tr])
    ro = r.rho
    assert abs(int(np.argmin(rg)) - int(np.argmin(ro))) <= 1
    assert ro.min() / 4 <= rg.min() <= 4 * ro.min()
    assert out == ipr.IPR_DIVERGED and r.outcome == oracle.DIVERGED
