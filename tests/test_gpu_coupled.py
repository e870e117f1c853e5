"""GPU parity of NEXT-2 (ii), the coupled form (reading R-27), through the C-ABI
(ipr_set_form(IPR_FORM_COUPLED)) against the oracle's FORM_COUPLED: diagonal A bit-exact, kappa = 2
trajectories at the Level-2 tolerance, BASELINE-family kappa = 1e3 bounded like the oracle."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

LOW = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)


@pytest.mark.parametrize("p,name", [(2, "fp64"), (1, "fp64"), (3, "fp64"), (2, "bf16"), (2, "tf32")])
def test_diagonal_bit_exact(p, name):
    A = synth.diag_spd(200, 1e2, 5)
    if name == "fp64":
        pg, po = [ipr.make_phase("fp64")], [oracle.phase()]
    else:
        OPR = {"bf16": oracle.BF16, "tf32": oracle.TF32}
        pg = [ipr.make_phase(name, **LOW), ipr.make_phase("fp64")]
        po = [oracle.phase(OPR[name], **LOW), oracle.phase()]
    r = oracle.solve(A, p, po, 1e-13, 150, hist=150, form=oracle.FORM_COUPLED)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-13, 150, form="coupled")
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)


@pytest.mark.parametrize("n,p", [(300, 2), (520, 3)])
def test_fp64_twin_trajectory(n, p):
    A = synth.spd(n, 2.0, 12)
    r = oracle.solve(A, p, [oracle.phase()], 1e-12, 60, hist=60, form=oracle.FORM_COUPLED)
    out, tr, hist, best = run_gpu_trajectory(A, p, [ipr.make_phase("fp64")], 1e-12, 60, form="coupled")
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert abs(len(tr) - len(r.records)) <= 1
    for k, Ck in hist.items():
        if k < len(r.records):
            assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    assert tr[-1]["rho_cert"] <= 1e-12


def test_kappa_1e3_bounded_like_oracle():
    n = 512
    A = synth.spd(n, 1e3, 1)
    r = oracle.solve(A, 2, [oracle.phase(max_iters=60)], 1e-12, 60, form=oracle.FORM_COUPLED)
    out, tr, hist, best = run_gpu_trajectory(A, 2, [ipr.make_phase("fp64", max_iters=60)], 1e-12, 60,
                                             keep=False, form="coupled")
    cert_g = np.linalg.norm(np.eye(n) - best @ best @ A)
    cert_o = np.linalg.norm(np.eye(n) - r.C_best @ r.C_best @ A)
    assert cert_g < 1e-4 and cert_o < 1e-4
    assert cert_g <= 4 * cert_o and cert_o <= 4 * cert_g        # Level-3 envelope
