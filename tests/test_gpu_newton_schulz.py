"""GPU parity of NEXT-1, the Newton-Schulz ordering X_{k+1} = X_k (2I - A X_k) of the p = 1
iteration, through the C-ABI (ipr_set_form) vs the oracle's
FORM_NEWTON_SCHULZ.  Same parity levels as the literal form."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

OPR = {"fp64": oracle.FP64, "tf32": oracle.TF32, "bf16": oracle.BF16, "fp16": oracle.FP16}


def run_ns(A_np, phases, final_tol, max_iters):
    A = torch_cuda(A_np)
    s = ipr.Solver(A, 1, phases, final_tol, form="newton_schulz")
    hist = {}
    for k in range(max_iters):
        out = s.iterate(1)
        if out != ipr.IPR_RUNNING:
            break
        hist[k + 1] = s.iterate_copy(0).cpu().numpy()
    tr = s.trace()
    best = s.finalize().cpu().numpy()
    return out, tr, hist, best


@pytest.mark.parametrize("name", ["fp64", "bf16", "tf32", "fp16"])
def test_ns_diagonal_bit_exact(name):
    A = synth.diag_spd(200, 1e3, 9)
    if name == "fp64":
        pg, po = [ipr.make_phase("fp64")], [oracle.phase()]
    else:
        pg = [ipr.make_phase(name, switch_tol=1e-2, plateau_ratio=0.7, plateau_arm=0.1, max_iters=40),
              ipr.make_phase("fp64")]
        po = [oracle.phase(OPR[name], switch_tol=1e-2, plateau_ratio=0.7, plateau_arm=0.1, max_iters=40),
              oracle.phase()]
    r = oracle.solve(A, 1, po, 1e-13, 120, hist=120, form=oracle.FORM_NEWTON_SCHULZ)
    out, tr, hist, best = run_ns(A, pg, 1e-13, 120)
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)


@pytest.mark.parametrize("n,kappa", [(300, 2.0), (512, 1e2)])
def test_ns_fp64_trajectory(n, kappa):
    A = synth.spd(n, kappa, 12)
    r = oracle.solve(A, 1, [oracle.phase()], 1e-11, 100, hist=100, form=oracle.FORM_NEWTON_SCHULZ)
    out, tr, hist, best = run_ns(A, [ipr.make_phase("fp64")], 1e-11, 100)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert abs(len(tr) - len(r.records)) <= 1
    for k, Ck in hist.items():
        if k < len(r.records):
            assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert np.linalg.norm(best @ A - np.eye(n)) < 1e-10


@pytest.mark.parametrize("name", ["bf16", "tf32", "fp16"])
def test_ns_mixed_level2_and_refinement_wins(name):
    # config C2 family (p = 1, kappa = 1e3, n = 1024): the NS ordering converges, and the mixed
    # schedule needs FEWER FP64 iterations than all-FP64 (SURVEY Table A6b) -- "refined into a
    # precise solution in very few additional iterations".
    # kappa = 1e3 is outside the stable-twin regime.  Level 3 of DESIGN.md section 4: Level-2 drift
    # until the oracle's commutator onset k* (gamma_k > 2^-m), then envelopes.  Here gamma stays below
    # 2^-m through the whole low phase (k* = 66 / 33 > the switch), so Level 2 applies throughout --
    # with reading R-31: in the Newton-Schulz linear phase (x <- x (2 - lambda x) doubles the small
    # eigencomponents, so a relative difference is carried forward undamped) every iteration can add
    # one stored rounding u_m = 2^-(m+1) of difference between the GPU (FP32 accumulation) and the
    # oracle (FP64), so the drift grows at most linearly: 4 2^-m + k u_m (measured: BF16 1.10 x 4 2^-7 at
    # the worst k, TF32 / FP16 6.7e-3 at k = 22, bound 1.5e-2).  Envelopes after the switch: switch
    # +-2, converged, answer within 1e-8 (FP64-phase drift of two valid runs, SURVEY Table A5a), and
    # the refinement claim.
    c = synth.CONFIGS["C2"]
    A, lam, _ = synth.spd(c["n"], c["kappa"], c["seed"], return_eig=True)
    m = {"bf16": 7, "tf32": 10, "fp16": 10}[name]
    tol = 1e-9
    sw = 1e-2 * np.sqrt(c["n"])
    pg = [ipr.make_phase(name, switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.1, max_iters=60), ipr.make_phase("fp64")]
    po = [oracle.phase(OPR[name], switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.1, max_iters=60), oracle.phase()]
    r = oracle.solve(A, 1, po, tol, 200, hist=200, form=oracle.FORM_NEWTON_SCHULZ,
                     gamma_normA2=float(lam.max()))
    out, tr, hist, best = run_ns(A, pg, tol, 200)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    sw_o = next(k for k, x in enumerate(r.records) if x["decision"] == oracle.SWITCH)
    sw_g = next(k for k, x in enumerate(tr) if x["decision"] == ipr.IPR_DEC_SWITCH)
    assert abs(sw_g - sw_o) <= 2
    gam = np.array([x["gamma"] for x in r.records])
    kstar = int(np.argmax(gam > 2.0 ** -m)) if np.any(gam > 2.0 ** -m) else len(gam)
    drift = []
    for k in range(1, min(sw_o, sw_g, kstar) + 1):
        d = rel_fro(hist[k], r.C_hist[k])
        drift.append(d)
        assert d <= 4 * 2.0 ** -m + k * 2.0 ** -(m + 1), (k, d)
    print(f"{name}: k*={kstar} switch={sw_o} max drift / 4 2^-m = {max(drift) / (4 * 2.0 ** -m):.3f}")
    assert rel_fro(best, r.C_best) <= 1e-8
    fp64_only = oracle.solve(A, 1, [oracle.phase()], tol, 200, form=oracle.FORM_NEWTON_SCHULZ)
    n_fp64_mixed = sum(1 for t in tr if t["prec"] == "fp64")
    assert n_fp64_mixed < len(fp64_only.records)


@pytest.mark.parametrize("name", ["bf16", "tf32", "fp16"])
def test_ns_mixed_twin_level2(name):
    n = 512
    A = synth.spd(n, 10.0, 14)
    m = {"bf16": 7, "tf32": 10, "fp16": 10}[name]
    sw = 1e-2 * np.sqrt(n)
    pg = [ipr.make_phase(name, switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.1, max_iters=60), ipr.make_phase("fp64")]
    po = [oracle.phase(OPR[name], switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.1, max_iters=60), oracle.phase()]
    r = oracle.solve(A, 1, po, 1e-12, 200, hist=200, form=oracle.FORM_NEWTON_SCHULZ)
    out, tr, hist, best = run_ns(A, pg, 1e-12, 200)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    sw_o = next(k for k, x in enumerate(r.records) if x["decision"] == oracle.SWITCH)
    sw_g = next(k for k, x in enumerate(tr) if x["decision"] == ipr.IPR_DEC_SWITCH)
    x = r.records[sw_o]
    tie = abs(x["rho"] - sw) <= 4 * 2.0 ** -m * x["rho"]
    assert sw_g == sw_o or (tie and abs(sw_g - sw_o) <= 1)
    for k in range(1, min(sw_o, sw_g) + 1):
        assert rel_fro(hist[k], r.C_hist[k]) <= 4 * 2.0 ** -m, k
    assert tr[-1]["rho"] <= 1e-12
    assert rel_fro(best, r.C_best) <= 1e-10


def test_ns_requires_p1():
    A = torch_cuda(synth.spd(64, 2.0, 1))
    s = ipr.Solver(A, 2, [ipr.make_phase("fp64")], 1e-12, form="newton_schulz")
    with pytest.raises(ipr.IprError) as e:
        s.iterate(1)
    assert e.value.status == ipr.IPR_E_INVALID_ARG
    s.close()
