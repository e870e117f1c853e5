"""The FP64 convergence certificate (R-30, R-32) through the C-ABI.

`ipr_residual(certify=1)` -- and the in-solve certificate of the symmetric / coupled forms, which
runs the same function -- is ||I - C^p A||_F of an FP64 iterate evaluated on the DMMA pipe.  For
p = 2 it is ||I - Y A||_F with Y = C C computed on its upper tiles and mirrored (G = 1) or as full
column panels (G > 1; tests/test_gpu_multirank.py demands the same bits).  Pinned here against
80-bit long-double evaluations of the definition (numpy longdouble, independent of the oracle and
of the CUDA path), on iterates far enough from convergence that the residual dominates the FP64
rounding (a misplaced tile, a wrong mirror or a transposed operand changes it at O(1)), and the
DMMA product of a bitwise-symmetric C with itself is checked to be bitwise symmetric (the
premise of the tri / full-panel equivalence)."""
import numpy as np
import pytest

import synth
from tests.gpu_util import torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")


def _ld_residual(C, A, p):
    """||I - C^p A||_F in 80-bit long double, right-to-left (the definition)."""
    Cl = C.astype(np.longdouble)
    X = A.astype(np.longdouble)
    for _ in range(p):
        X = Cl @ X
    E = np.eye(len(C), dtype=np.longdouble) - X
    return float(np.sqrt((E * E).sum()))


@pytest.mark.parametrize("n", [300, 1000, 2304])
def test_dmma_square_of_symmetric_is_symmetric(n):
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n))
    C = torch_cuda((X + X.T) / 2)
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_gemm(ipr.IPR_FP64, n, C, C, Z)
    Zh = Z.cpu().numpy()
    assert np.array_equal(Zh, Zh.T)


@pytest.mark.parametrize("n,p,form,sched", [(300, 2, "symmetric_tri", "fp64"), (520, 2, "symmetric_tri", "bf16"),
                                            (520, 2, "symmetric", "fp64"), (520, 3, "symmetric", "fp64"),
                                            (300, 2, "literal", "fp64"), (300, 3, "literal", "bf16")])
def test_certificate_of_best_iterate_vs_long_double(n, p, form, sched):
    A = synth.spd(n, 2.0, 21)
    s = ipr.Solver(torch_cuda(A), p, [ipr.make_phase(sched)], 1e-12, form=form)
    assert s.iterate(3) == ipr.IPR_RUNNING
    rho = s.residual(True)
    best = s.iterate_copy(1).cpu().numpy()
    ref = _ld_residual(best, A, p)
    assert ref > 1e-6                       # far from convergence: the residual dominates rounding
    assert rho == pytest.approx(ref, rel=1e-10)
    assert s.residual(True) == rho          # deterministic
    s.close()


@pytest.mark.parametrize("form", ["symmetric", "symmetric_tri"])
def test_converged_certificate_is_the_recheck(form):
    A = synth.spd(520, 2.0, 22)
    s = ipr.Solver(torch_cuda(A), 2, [ipr.make_phase("bf16", plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
                                      ipr.make_phase("fp64", corr_prec="bf16")], 1e-12, form=form)
    assert s.iterate(200) == ipr.IPR_CONVERGED
    tr = s.trace()
    assert tr[-1]["rho_cert"] <= 1e-12
    assert s.residual(True) == tr[-1]["rho_cert"]
    best = s.finalize().cpu().numpy()
    # the FP64 evaluation of a residual at the 1e-13 level is dominated by its own rounding: only a
    # loose agreement with the long-double value is a property (both are O(1e-13), neither O(1))
    assert _ld_residual(best, A, 2) <= 1e-12
