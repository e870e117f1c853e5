"""GPU parity of IPR_FP64_OZ (reading R-23): FP64 GEMMs emulated on the INT8 tensor cores
by the Ozaki scheme I (9 digits, 9 K-concatenated kind::i8 GEMMs, FP64 combination).

Kernel level: the emulated product is as accurate as the FP64 DMMA product against an
extended-precision (80-bit long double) reference -- the property that lets the oracle's FP64
GEMM stand for it; exact on small integers.  Trajectory level: the symmetric forms' FP64 phase
on IPR_FP64_OZ within the Level-2 FP64 tolerance of the oracle (1e-10, certified rho <= 1e-12)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")


def _gemm(prec, X, Y):
    n = X.shape[0]
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_gemm(prec, n, torch.from_numpy(np.ascontiguousarray(X)).cuda(),
                      torch.from_numpy(np.ascontiguousarray(Y.T)).cuda(), Z)
    return Z.cpu().numpy()


@pytest.mark.parametrize("n", [1, 200, 513, 1024])
def test_ozaki_integers_exact(n):
    rng = np.random.default_rng(n)
    X = rng.integers(-1000, 1001, (n, n)).astype(np.float64)
    Y = rng.integers(-1000, 1001, (n, n)).astype(np.float64)
    np.testing.assert_array_equal(_gemm(ipr.IPR_FP64_OZ, X, Y), X @ Y)


@pytest.mark.parametrize("n,kappa", [(512, 2.0), (1536, 2.0), (1024, 1e3)])
def test_ozaki_as_accurate_as_dmma(n, kappa):
    A, lam, Q = synth.spd(n, kappa, 3, return_eig=True)
    C = (Q * lam ** -0.5) @ Q.T
    C = (C + C.T) / 2
    exact = A.astype(np.longdouble) @ C.astype(np.longdouble)
    e_oz = np.linalg.norm((_gemm(ipr.IPR_FP64_OZ, A, C) - exact).astype(np.float64))
    e_dm = np.linalg.norm((_gemm(ipr.IPR_FP64, A, C) - exact).astype(np.float64))
    assert e_oz <= 2.0 * e_dm, (e_oz, e_dm)


@pytest.mark.parametrize("form,sched", [("symmetric", "fp64oz"), ("symmetric_tri", "fp64oz"),
                                        ("symmetric_tri", "bf16>fp64oz/cbf16"), ("symmetric", "tf32>fp64oz")])
def test_ozaki_fp64_phase_level2(form, sched):
    n, p = 520, 2
    A = synth.spd(n, 2.0, 12)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    OPR = {"bf16": oracle.BF16, "tf32": oracle.TF32, "fp64oz": oracle.FP64_OZ}
    pg, po = [], []
    parts = sched.split(">")
    for i, part in enumerate(parts):
        prec, _, corr = part.partition("/c")
        kw = {} if i == len(parts) - 1 else low
        pg.append(ipr.make_phase(prec, corr_prec=corr or -1, **kw))
        po.append(oracle.phase(OPR[prec], corr_prec=OPR[corr] if corr else -1, **kw))
    oform = oracle.FORM_SYMMETRIC if form == "symmetric" else oracle.FORM_SYMMETRIC_TRI
    r = oracle.solve(A, p, po, 1e-12, 80, hist=80, form=oform)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-12, 80, form=form)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert abs(len(tr) - len(r.records)) <= 1
    if len(parts) == 1:      # all-FP64 trajectories agree per iterate (Level 2)
        for k, Ck in hist.items():
            if k < len(r.records):
                assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    else:                    # mixed: the low phase within 4 * 2^-m, the refined answer within 1e-10
        m = {"bf16": 7, "tf32": 10}[parts[0].partition("/c")[0]]
        sw = next(k for k, x in enumerate(r.records) if x["decision"] == oracle.SWITCH)
        for k in range(1, sw + 1):
            assert rel_fro(hist[k], r.C_hist[k]) <= 4 * 2.0 ** -m, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12


def test_ozaki_unsupported_outside_symmetric_forms():
    A = torch.from_numpy(synth.spd(64, 2.0, 0)).cuda()
    s = ipr.Solver(A, 2, [ipr.make_phase("fp64oz")], 1e-12)
    with pytest.raises(ipr.IprError) as e:
        s.iterate(1)
    assert e.value.status == ipr.IPR_E_UNSUPPORTED
    s.close()


def test_adaptive_digits_level2_and_storage_rule():
    # R-26: digits / stored bits chosen per iteration from the expected residual; the oracle
    # mirrors the storage rule (its arithmetic stays FP64).  Same per-iteration stored bits (ties
    # aside), final C within 1e-10 and certified rho <= 1e-12.
    n, p = 520, 2
    A = synth.spd(n, 2.0, 12)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    pg = [ipr.make_phase("bf16", **low), ipr.make_phase("fp64oz", mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec="bf16")]
    po = [oracle.phase(oracle.BF16, **low), oracle.phase(oracle.FP64_OZ, mant_bits=oracle.MANT_ADAPTIVE,
                                                         corr_prec=oracle.BF16)]
    r = oracle.solve(A, p, po, 1e-12, 80, hist=80, form=oracle.FORM_SYMMETRIC_TRI)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-12, 80, form="symmetric_tri")
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    mg = [t["mant_bits"] for t in tr if t["phase"] == 1]
    mo = [x["mant_bits"] for x in r.records if x["phase"] == 1]
    assert len(set(mg)) >= 3 and mg[-1] == 52                   # precision rises inside the phase
    agree = sum(a == b for a, b in zip(mg, mo))
    assert agree >= min(len(mg), len(mo)) - 1, (mg, mo)
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12
