"""-m gpu: the CRT certificate (IPR_CERT_CRT, reading R-35) through the C-ABI against the oracle.

The certificate claims a proven upper bound on the EXACT residual ||I - Ct^2 A||_F of the matrix it returns
(Ct: the candidate rounded to the coarser of its row / column 62-bit grids).  Checked here against the
oracle's independent evaluation of that quantity (orc_cert_grid + the double-double residual orc_resid_dd):
  * the bound is >= the exact residual, and its evaluated part is within the bound's own error terms of it
    -- on converged answers (~1e-13) and on iterates far from convergence, at ragged and multi-band sizes;
  * the returned answer is exactly the oracle's grid rounding of the candidate (idempotent);
  * a solve certified this way follows the oracle's trajectory (same decisions, Level-2 answer);
  * ipr_residual(certify=1) reproduces the in-solve certificate bit for bit; certify=2 is the DMMA evaluation.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1703_02283_b200 as ipr
import synth
from tests.gpu_util import rel_fro

pytestmark = pytest.mark.gpu

LOW = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)


def _gpu_phases(fp8=False):
    ph = [ipr.make_phase("bf16", **LOW),
          ipr.make_phase("fp64crt", mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec="bf16")]
    if fp8:
        ph.insert(0, ipr.make_phase("fp8", corr_prec="fp8", **LOW))
    return ph


def _orc_phases(fp8=False):
    ph = [oracle.phase(oracle.BF16, **LOW),
          oracle.phase(oracle.FP64_CRT, mant_bits=oracle.MANT_ADAPTIVE, corr_prec=oracle.BF16)]
    if fp8:
        ph.insert(0, oracle.phase(oracle.FP8, corr_prec=oracle.FP8, **LOW))
    return ph


def _solve(A_np, max_iters=200, fp8=False, cert="crt"):
    A = torch.from_numpy(A_np).cuda()
    s = ipr.Solver(A, 2, _gpu_phases(fp8), 1e-12, form="symmetric_tri", cert=cert)
    out = s.iterate(max_iters)
    return s, out


def _check_bound(A_np, info, C_cert, bound):
    exact = oracle.resid_dd(A_np, C_cert, 2)
    assert bound >= exact, (bound, exact)
    # the evaluated part differs from the exact residual only by the terms the bound adds
    assert abs(info["est"] - exact) <= info["beta"] + 1e-9 * exact, (info, exact)
    assert bound <= exact + 2 * info["beta"] + 1e-9 * exact + 1e-300
    return exact


@pytest.mark.parametrize("n", [256, 520])
def test_certificate_of_a_converged_solve_bounds_the_exact_residual(n):
    A_np = synth.spd(n, 2.0, 40 + n)
    s, out = _solve(A_np)
    assert out == ipr.IPR_CONVERGED
    tr = s.trace()
    info = ipr.ipr_test_cert_info(s.ctx)
    assert tr[-1]["rho_cert"] == info["bound"] <= 1e-12
    assert s.residual(1) == tr[-1]["rho_cert"]           # re-check = the certificate, bit for bit
    dmma = s.residual(2)
    C = s.finalize().cpu().numpy()
    np.testing.assert_array_equal(C, oracle.cert_grid(C, 62))   # the answer is its own grid rounding
    exact = _check_bound(A_np, info, C, info["bound"])
    assert info["moduli"] == ipr.ipr_test_crt_table(18, 62, n)["n_for"]
    assert abs(dmma - exact) <= 64 * n * 2.0 ** -53      # the FP64 evaluation within its rounding noise


@pytest.mark.parametrize("n,iters", [(520, 3), (2080, 21)])
def test_certificate_of_unconverged_iterates(n, iters):
    # bound vs exact far from convergence (rho ~ 1e-1 .. 1e-6): ragged n, and 2080 = 9 pair-column tiles:
    # the tri Y product's mirror crosses two bands of the tile order
    A_np = synth.spd(n, 2.0, 7)
    s, out = _solve(A_np, max_iters=iters)
    assert out == ipr.IPR_RUNNING
    bound = s.residual(1)
    info = ipr.ipr_test_cert_info(s.ctx)
    assert info["bound"] == bound
    C = s.iterate_copy(1).cpu().numpy()                 # the best iterate (the bound is for its rounding)
    s.close()
    exact = _check_bound(A_np, info, oracle.cert_grid(C, 62), bound)
    assert exact > 1e-12                                 # not converged


def test_crt_certified_solve_follows_the_oracle_trajectory():
    n = 320
    A_np = synth.spd(n, 2.0, 21)
    r = oracle.solve(A_np, 2, _orc_phases(True), 1e-12, 120, form=oracle.FORM_SYMMETRIC_TRI, cert="crt")
    s, out = _solve(A_np, fp8=True)
    tr = s.trace()
    C = s.finalize().cpu().numpy()
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    assert rel_fro(C, r.C_best) <= 1e-10
    assert oracle.resid_dd(A_np, C, 2) <= tr[-1]["rho_cert"] <= 1e-12   # the bound vs the exact residual of C
    # the oracle's own certified value (the exact residual of ITS answer, a Level-2 neighbour of C)
    assert abs(tr[-1]["rho_cert"] - r.records[-1]["rho_cert"]) <= 0.2 * r.records[-1]["rho_cert"]


def test_crt_certificate_streams_the_certified_matrix_to_a_host_output():
    n = 256
    A_np = synth.spd(n, 2.0, 3)
    A = torch.from_numpy(A_np).cuda()
    s = ipr.Solver(A, 2, _gpu_phases(), 1e-12, form="symmetric_tri", cert="crt")
    host = torch.empty((n, n), dtype=torch.float64).pin_memory()
    s.set_output(host)
    assert s.iterate(200) == ipr.IPR_CONVERGED
    dev = s.iterate_copy(1).cpu()
    s.finalize(host)
    assert torch.equal(host, dev)
    np.testing.assert_array_equal(host.numpy(), oracle.cert_grid(host.numpy(), 62))


def test_crt_certificate_unsupported_configurations():
    A = torch.from_numpy(synth.spd(64, 2.0, 0)).cuda()
    for form, phases in [("literal", [ipr.make_phase("fp64")]),
                         ("symmetric_tri", [ipr.make_phase("bf16", **LOW), ipr.make_phase("fp64")])]:
        s = ipr.Solver(A, 2, phases, 1e-12, form=form, cert="crt")
        with pytest.raises(ipr.IprError) as e:
            s.iterate(1)
        assert e.value.status == ipr.IPR_E_UNSUPPORTED
        s.close()


def test_crt_certificate_out_of_range_falls_back_to_the_dmma_evaluation():
    # A scaled by 2^500: C ~ 2^-500, whose row exponents leave the (-400, 400) range the certificate's exact
    # scalings cover -- the certificate of such a candidate is R-30's FP64 DMMA evaluation of Ct instead,
    # i.e. ipr_residual(certify=1) == ipr_residual(certify=2).  (Eq. (3)'s C_0 is not scale-invariant for
    # p = 2 -- C_0^2 A scales as 2^-sc -- so such a solve does not converge in a test's budget: the
    # certificate is exercised on its early iterates.)
    n = 256
    A = torch.from_numpy(np.ldexp(synth.spd(n, 2.0, 9), 500)).cuda()
    s = ipr.Solver(A, 2, [ipr.make_phase("fp64crt", mant_bits=ipr.IPR_MANT_ADAPTIVE)], 1e-12,
                   form="symmetric_tri", cert="crt")
    assert s.iterate(2) == ipr.IPR_RUNNING
    r1 = s.residual(1)
    info = ipr.ipr_test_cert_info(s.ctx)
    assert info["bound"] == r1 and info["beta"] != info["beta"]        # the DMMA value, no bound terms
    assert r1 == s.residual(2)
    s.close()


@pytest.mark.parametrize("n", [1, 17, 128])
def test_crt_certificate_tiny_sizes(n):
    A_np = synth.spd(n, 2.0, 70 + n) if n > 1 else np.array([[0.7]])
    s, out = _solve(A_np)
    assert out == ipr.IPR_CONVERGED
    info = ipr.ipr_test_cert_info(s.ctx)
    C = s.finalize().cpu().numpy()
    exact = _check_bound(A_np, info, C, info["bound"])
    assert exact <= 1e-12


@pytest.mark.parametrize("n", [256, 520])
def test_crt_certificate_p3(n):
    # p = 3 (one GPU): Y = Ct Ct exact, T = Ct Ytilde exact (Y symmetric, so its row quantisation is the
    # column operand), P = Ttilde Atilde; the bound carries ||Ct||_inf (dY + eY) through T
    A_np = synth.spd(n, 2.0, 80 + n)
    A = torch.from_numpy(A_np).cuda()
    s = ipr.Solver(A, 3, _gpu_phases(), 1e-12, form="symmetric", cert="crt")
    assert s.iterate(200) == ipr.IPR_CONVERGED
    tr = s.trace()
    info = ipr.ipr_test_cert_info(s.ctx)
    assert tr[-1]["rho_cert"] == info["bound"] <= 1e-12
    assert s.residual(1) == info["bound"]
    C = s.finalize().cpu().numpy()
    np.testing.assert_array_equal(C, oracle.cert_grid(C, 62))
    exact = oracle.resid_dd(A_np, C, 3)
    assert exact <= info["bound"] and abs(info["est"] - exact) <= info["beta"] + 1e-9 * exact
    # unconverged iterates too (the trajectory's early records)
    s2 = ipr.Solver(A, 3, _gpu_phases(), 1e-12, form="symmetric", cert="crt")
    s2.iterate(6)
    b2 = s2.residual(1)
    i2 = ipr.ipr_test_cert_info(s2.ctx)
    C2 = s2.iterate_copy(1).cpu().numpy()
    s2.close()
    e2 = oracle.resid_dd(A_np, oracle.cert_grid(C2, 62), 3)
    assert e2 <= b2 and abs(i2["est"] - e2) <= i2["beta"] + 1e-9 * e2 and e2 > 1e-12


def test_crt_certificate_after_a_dmma_last_phase():
    # the certificate needs a CRT phase somewhere in the schedule (its buffers) and an FP64 last phase:
    # BF16 > CRT(23 bits) > FP64 on the DMMA pipe, certified by the CRT bound
    import bench
    n = 520
    A_np = synth.spd(n, 2.0, 17)
    form, ph = bench.schedule("symtri:bf16>fp64crt@23/cbf16>fp64/cbf16", n)
    s = ipr.Solver(torch.from_numpy(A_np).cuda(), 2, ph, 1e-12, form=form, cert="crt")
    assert s.iterate(300) == ipr.IPR_CONVERGED
    tr = s.trace()
    info = ipr.ipr_test_cert_info(s.ctx)
    assert tr[-1]["rho_cert"] == info["bound"] <= 1e-12 and tr[-1]["phase"] == 2
    C = s.finalize().cpu().numpy()
    _check_bound(A_np, info, C, info["bound"])
