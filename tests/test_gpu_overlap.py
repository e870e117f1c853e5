"""GPU vs oracle on the paper-shaped overlap workload (synth.overlap stands in
for the H2O overlap matrices of PAPER.md:178-185).  N = 768 at the paper's 25 % density:
  * kappa = 2 twin (shifted), p = 2, symmetric form, BF16 -> FP64: Level 2;
  * natural kappa (~1e3), p = 1, Newton-Schulz FP64 (the form the paper names for p = 1,
    PAPER.md:79-81): trajectories within the Level-2 FP64 tolerance, converged to 1e-10."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")


def test_overlap_twin_symmetric_mixed_level2():
    A = synth.overlap(768, seed=0, kappa=2.0)
    lowg = ipr.make_phase("bf16", plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    lowo = oracle.phase(oracle.BF16, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    r = oracle.solve(A, 2, [lowo, oracle.phase(corr_prec=oracle.BF16)], 1e-12, 80, hist=80,
                     form=oracle.FORM_SYMMETRIC_TRI)
    out, tr, hist, best = run_gpu_trajectory(A, 2, [lowg, ipr.make_phase("fp64", corr_prec="bf16")], 1e-12, 80,
                                             form="symmetric_tri")
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    sw_o = [x["k"] for x in r.records if x["decision"] == oracle.SWITCH]
    sw_g = [t["k"] for t in tr if t["decision"] == ipr.IPR_DEC_SWITCH]
    assert len(sw_o) == len(sw_g) == 1 and abs(sw_o[0] - sw_g[0]) <= 1
    for k, Ck in hist.items():
        if k <= sw_o[0]:
            assert rel_fro(Ck, r.C_hist[k]) <= 4 * 2.0 ** -7, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12


def test_overlap_natural_kappa_newton_schulz():
    A = synth.overlap(768, seed=0)
    r = oracle.solve(A, 1, [oracle.phase()], 1e-10, 80, hist=80, form=oracle.FORM_NEWTON_SCHULZ)
    A_t = torch.from_numpy(A).cuda()
    s = ipr.Solver(A_t, 1, [ipr.make_phase("fp64")], 1e-10, form="newton_schulz")
    hist = {}
    for k in range(80):
        out = s.iterate(1)
        if out != ipr.IPR_RUNNING:
            break
        hist[k + 1] = s.iterate_copy(0).cpu().numpy()
    tr = s.trace()
    best = s.finalize().cpu().numpy()
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert abs(len(tr) - len(r.records)) <= 1
    for k, Ck in hist.items():
        if k < len(r.records):
            assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    assert np.linalg.norm(best @ A - np.eye(768)) <= 1e-9
