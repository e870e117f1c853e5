"""Pins of the oracle's NEXT-1 form: the Newton-Schulz ordering X_{k+1} = X_k (2I - A X_k) of the
p = 1 iteration (PAPER.md:79-81 [Sec. 2] names Newton-Schulz)."""
import numpy as np
import pytest

import oracle
import synth
from tests import golden

G = golden.load()


@pytest.mark.parametrize("name", ["ns_p1_scalar", "ns_p1_2x2"])
def test_golden_ns_step(name):
    g = G[name]
    _, nxt, _ = oracle.step_ns(golden.matrix(g["inputs"]["A"]), golden.matrix(g["inputs"]["C"]), oracle.phase())
    np.testing.assert_allclose(nxt, np.atleast_2d(g["expected"]), rtol=1e-15, atol=1e-16, err_msg=g["cite"])


def test_golden_ns_residual_and_difference_from_literal():
    g = G["rho_ns_2x2"]
    A, X = golden.matrix(g["inputs"]["A"]), golden.matrix(g["inputs"]["C"])
    rho, nxt, _ = oracle.step_ns(A, X, oracle.phase())
    assert rho == pytest.approx(g["expected"], rel=1e-15)
    _, lit, _ = oracle.step(A, X, 1, oracle.phase())      # C(2I - CA): a different ordering
    assert not np.allclose(nxt, lit)


def test_ns_limit_is_inverse():
    A = synth.spd(96, 50.0, 3)
    r = oracle.solve(A, 1, [oracle.phase()], 1e-12, 100, form=oracle.FORM_NEWTON_SCHULZ)
    assert r.outcome == oracle.CONVERGED
    np.testing.assert_allclose(r.C_best @ A, np.eye(96), atol=1e-11)
    np.testing.assert_allclose(r.C_best, np.linalg.inv(A), rtol=1e-9, atol=1e-12)


def test_ns_is_stable_where_literal_is_not():
    # config C2 family (kappa=1e3, p=1): literal Eq. (1) diverges (SURVEY F3 / Table A6b),
    # the Newton-Schulz ordering converges (its error is quadratic in E, no linear term).
    A = synth.spd(256, 1e3, 1)
    lit = oracle.solve(A, 1, [oracle.phase()], 1e-10, 120)
    ns = oracle.solve(A, 1, [oracle.phase()], 1e-10, 120, form=oracle.FORM_NEWTON_SCHULZ)
    assert lit.outcome in (oracle.DIVERGED, oracle.NONFINITE) or lit.rho.min() > 1e-6
    assert ns.outcome == oracle.CONVERGED


def test_ns_mixed_precision_refines_quickly():
    # PAPER.md:346-350 "refined into a precise solution in very few additional iterations":
    # true for the NS ordering (SURVEY Table A6b) -- fewer FP64 iterations than all-FP64.
    A = synth.spd(256, 1e2, 2)
    fp64 = oracle.solve(A, 1, [oracle.phase()], 1e-10, 200, form=oracle.FORM_NEWTON_SCHULZ)
    mixed = oracle.solve(A, 1, [oracle.phase(oracle.BF16, switch_tol=1e-2 * 16, plateau_ratio=0.7,
                                             plateau_arm=0.5, max_iters=60), oracle.phase()],
                         1e-10, 200, form=oracle.FORM_NEWTON_SCHULZ)
    assert fp64.outcome == oracle.CONVERGED and mixed.outcome == oracle.CONVERGED
    n_fp64_after = sum(1 for x in mixed.records if x["phase"] == 1)
    assert n_fp64_after < len(fp64.records)


def test_ns_rejects_p_other_than_1():
    with pytest.raises(ValueError):
        oracle.solve(np.eye(4), 2, [oracle.phase()], form=oracle.FORM_NEWTON_SCHULZ)
