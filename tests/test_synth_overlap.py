"""The paper-shaped overlap workload generator (Sec. 4.1:
SPD, entries in [-1, 1], 25 % non-zeros at N = 768/786, density halving as N doubles)."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("n", [768, 1536])
def test_structure_matches_paper(n):
    S, info = synth.overlap(n, seed=3, return_info=True)
    d = synth.OVERLAP_PRESETS[n]
    assert np.array_equal(S, S.T)
    assert np.all(np.diag(S) == 1.0)
    assert np.abs(S).max() <= 1.0
    assert abs(np.count_nonzero(S) / n ** 2 - d) <= 0.1 * d
    assert np.linalg.eigvalsh(S)[0] > 0          # SPD
    assert oracle.is_symmetric(S)


def test_density_halves_as_n_doubles():
    ds = [synth.OVERLAP_PRESETS[n] for n in (768, 1536, 3072, 6144)]
    assert all(0.45 < b / a < 0.55 for a, b in zip(ds, ds[1:]))


def test_deterministic_and_kappa_shift():
    a = synth.overlap(200, 0.25, seed=7)
    b = synth.overlap(200, 0.25, seed=7)
    assert np.array_equal(a, b)
    S = synth.overlap(300, 0.25, seed=1, kappa=2.0)
    ev = np.linalg.eigvalsh(S)
    assert ev[-1] / ev[0] == pytest.approx(2.0, rel=1e-9)
    assert np.allclose(np.diag(S), 1.0) and np.array_equal(S, S.T)


def test_small_case_spd_by_jacobi():
    S = synth.overlap(64, 0.25, seed=2)
    lam, _ = oracle.jacobi(S)
    assert lam.min() > 0
