"""GPU parity of IPR_FORM_SYMMETRIC_TRIZ (reading R-37): the tri form whose FP64_CRT phase takes
Z_1 = Ahat Chat from its upper tiles too while the phase contracts fast (every in-phase ratio <= 0.1, from the
third chain on; sticky off).  Against the oracle's FORM_SYMMETRIC_TRIZ on a schedule both sides run on the
same bits up to the last rounding: a 7-bit-storage FP64_CRT phase (exact products, BF16-sized storage noise
that does not commute with A -- what the mirror feeds back) and then the adaptive FP64_CRT phase with the BF16
correction.  The two chain kinds differ by ~2e-2 in rho; GPU and oracle agree far below that."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")


def _phases(n):
    low = dict(switch_tol=2.0 * 2.0 ** -8 * np.sqrt(n), plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    pg = [ipr.make_phase("fp64crt", mant_bits=7, **low),
          ipr.make_phase("fp64crt", mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec="bf16")]
    po = [oracle.phase(oracle.FP64_CRT, mant_bits=7, **low),
          oracle.phase(oracle.FP64_CRT, mant_bits=oracle.MANT_ADAPTIVE, corr_prec=oracle.BF16)]
    return pg, po


@pytest.mark.parametrize("n", [520, 648])
def test_triz_trajectory_and_rule_match_the_oracle(n):
    A = synth.spd(n, 2.0, 12)
    pg, po = _phases(n)
    r = oracle.solve(A, 2, po, 1e-12, 120, form=oracle.FORM_SYMMETRIC_TRIZ)
    rt = oracle.solve(A, 2, po, 1e-12, 120, form=oracle.FORM_SYMMETRIC_TRI)
    out, tr, _, best = run_gpu_trajectory(A, 2, pg, 1e-12, 120, keep=False, form="symmetric_triz")
    out_t, tr_t, _, _ = run_gpu_trajectory(A, 2, pg, 1e-12, 120, keep=False, form="symmetric_tri")
    assert out == out_t == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    g = [t for t in tr if t["phase"] == 1 and t["rho"] == t["rho"]]
    gt = [t for t in tr_t if t["phase"] == 1 and t["rho"] == t["rho"]]
    o = [x for x in r.records if x["phase"] == 1 and x["rho"] == x["rho"]]
    ot = [x for x in rt.records if x["phase"] == 1 and x["rho"] == x["rho"]]
    assert len(g) == len(o) and len(gt) == len(ot)
    # the rule, from the GPU's own residuals: tri Z_1 from the third chain on while every ratio was <= 0.1
    ok, want = True, []
    for i, t in enumerate(g):
        want.append(1 if (ok and i >= 2) else 0)
        if i >= 1 and not g[i]["rho"] <= 0.1 * g[i - 1]["rho"]:
            ok = False
    assert [t["ztri"] for t in g] == want and sum(want) >= 3
    assert all(t["ztri"] == 0 for t in tr_t) and all(t["ztri"] == 0 for t in tr if t["phase"] == 0)
    # Level 2: chain by chain against the oracle of the same form (the other form is ~2e-2 away)
    for i, (a, b) in enumerate(zip(g, o)):
        assert a["rho"] == pytest.approx(b["rho"], rel=2e-3, abs=2e-13), (i, a["rho"], b["rho"])
    for i, (a, b) in enumerate(zip(gt, ot)):
        assert a["rho"] == pytest.approx(b["rho"], rel=2e-3, abs=2e-13), (i, a["rho"], b["rho"])
    i3 = want.index(1) + 1          # the first residual a mirrored Z_1 shaped
    if i3 < min(len(g), len(gt)):
        assert abs(g[i3]["rho"] - gt[i3]["rho"]) > 5e-3 * gt[i3]["rho"]
        assert abs(o[i3]["rho"] - ot[i3]["rho"]) > 5e-3 * ot[i3]["rho"]
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12


def test_triz_equals_tri_on_a_slowly_contracting_phase():
    # kappa = 5: the first in-phase ratio is above 0.1 -- no chain is mirrored, bit-identical to the tri form
    n = 520
    A = synth.spd(n, 5.0, 2)
    pg, _ = _phases(n)
    out_a, tr_a, _, Ca = run_gpu_trajectory(A, 2, pg, 1e-12, 200, keep=False, form="symmetric_tri")
    out_b, tr_b, _, Cb = run_gpu_trajectory(A, 2, pg, 1e-12, 200, keep=False, form="symmetric_triz")
    assert out_a == out_b == ipr.IPR_CONVERGED
    assert [t["rho"] for t in tr_a if t["rho"] == t["rho"]] == [t["rho"] for t in tr_b if t["rho"] == t["rho"]]
    assert all(t["ztri"] == 0 for t in tr_b)
    np.testing.assert_array_equal(Ca, Cb)


def test_triz_headline_schedule_crt_certificate_two_bands():
    # n = 2304: two tile bands of the tri scheduler; the bench's schedule with the CRT certificate (R-35): the
    # certified bound holds for the returned matrix whatever produced it -- checked against the oracle's
    # double-double residual of that matrix on sampled rows, and C^2 A v = v on probe vectors
    import bench
    n = 2304
    A_np = synth.spd(n, 2.0, 5)
    A = torch.from_numpy(A_np).cuda()
    form, phases = bench.schedule("symtriz:fp8/cfp8>bf16>fp64crt@a/cbf16", n)
    s = ipr.Solver(A, 2, phases, 1e-12, form=form, cert="crt")
    s.iterate(300)
    tr, out = s.trace(), s.outcome
    C = s.finalize().cpu().numpy()
    assert out == ipr.IPR_CONVERGED and tr[-1]["rho_cert"] <= 1e-12
    assert sum(t["ztri"] for t in tr) >= 3
    np.testing.assert_array_equal(C, C.T)
    rows = np.array([0, 1, 127, 128, 1151, 1152, 2047, 2303])
    part = oracle.resid_rows_dd(A_np, C, 2, rows)
    assert np.sqrt(part.sum() * n / len(rows)) <= 3.0 * tr[-1]["rho_cert"]   # sampled rows: the bound's order
    for v in synth.probe_vectors(n, 3, 2):
        x = C @ (C @ (A_np @ v))
        assert np.linalg.norm(x - v) / np.linalg.norm(v) < 1e-12
