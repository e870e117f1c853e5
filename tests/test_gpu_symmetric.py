"""GPU parity of NEXT-2, the symmetrised-correction form (reading R-22)

    Z_1 = Ahat Chat, Z_j = Chat qin(Z_{j-1}), Rhat = qc(I - Z_p), W = qc(C) Rhat,
    C_{k+1} = q_m(C + (W + W^T)/(2p)),

through the C-ABI (ipr_set_form(IPR_FORM_SYMMETRIC), ipr_phase.corr_prec) against the oracle's
FORM_SYMMETRIC.  Parity levels as for the literal form: diagonal A bit-exact
(every dot product has one non-zero term), kappa = 2 twins within the north-star tolerances,
bitwise symmetry and run-to-run determinism of the GPU iterates."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory, torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

OPR = {"fp64": oracle.FP64, "tf32": oracle.TF32, "bf16": oracle.BF16, "fp16": oracle.FP16, "fp8": oracle.FP8}
LOW = dict(switch_tol=0.0, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)


def schedules(name):
    """(gpu phases, oracle phases) of a named schedule; 'x/cy' = phase x with correction y."""
    pg, po = [], []
    parts = name.split(">")
    for i, part in enumerate(parts):
        prec, _, corr = part.partition("/c")
        kw = {} if i == len(parts) - 1 else LOW
        pg.append(ipr.make_phase(prec, corr_prec=corr or -1, **kw))
        po.append(oracle.phase(OPR[prec], corr_prec=OPR[corr] if corr else -1, **kw))
    return pg, po


FORMS = {"symmetric": oracle.FORM_SYMMETRIC, "symmetric_tri": oracle.FORM_SYMMETRIC_TRI}


def run_sym(A, p, name, tol, iters, form="symmetric"):
    pg, po = schedules(name)
    r = oracle.solve(A, p, po, tol, iters, hist=iters, form=FORMS[form])
    g = run_gpu_trajectory(A, p, pg, tol, iters, form=form)
    return r, g


@pytest.mark.parametrize("p,name,form", [(2, "fp64", "symmetric"), (3, "fp64", "symmetric"),
                                         (2, "fp64/cbf16", "symmetric"), (2, "bf16>fp64", "symmetric"),
                                         (2, "tf32>fp64/cbf16", "symmetric"), (3, "bf16>fp64/ctf32", "symmetric"),
                                         (2, "bf16/ctf32>fp64", "symmetric"), (2, "fp64", "symmetric_tri"),
                                         (2, "bf16>fp64/cbf16", "symmetric_tri"), (2, "tf32>fp64", "symmetric_tri"),
                                         (2, "fp16>fp64/cbf16", "symmetric_tri"), (3, "fp16/ctf32>fp64", "symmetric"),
                                         # R-29: scaled correction (FP32 scratch of R + sigma_R)
                                         (2, "fp8/cfp8>fp64", "symmetric_tri"), (2, "fp8/cfp8>fp64", "symmetric"),
                                         (3, "fp16/cfp16>fp64", "symmetric")])
def test_diagonal_bit_exact(p, name, form):
    A = synth.diag_spd(200, 1e3, 9)
    r, (out, tr, hist, best) = run_sym(A, p, name, 1e-13, 120, form)
    assert r.outcome == oracle.CONVERGED and out == ipr.IPR_CONVERGED
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)
    for t, x in zip(tr, r.records):
        assert t["rho"] == pytest.approx(x["rho"], rel=1e-12, abs=1e-300, nan_ok=True)   # NaN: R-33
    assert tr[-1]["rho_cert"] <= 1e-13


@pytest.mark.parametrize("n,p,form", [(300, 2, "symmetric"), (300, 3, "symmetric"), (520, 2, "symmetric"),
                                      (300, 2, "symmetric_tri"), (520, 2, "symmetric_tri")])
def test_fp64_twin_trajectory(n, p, form):
    A = synth.spd(n, 2.0, 12)
    r, (out, tr, hist, best) = run_sym(A, p, "fp64", 1e-12, 60, form)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert abs(len(tr) - len(r.records)) <= 1
    for k, Ck in hist.items():
        assert np.array_equal(Ck, Ck.T), f"GPU iterate {k} not bitwise symmetric"
        if k < len(r.records):
            assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12


@pytest.mark.parametrize("name,m,form", [("bf16>fp64/cbf16", 7, "symmetric"), ("tf32>fp64/cbf16", 10, "symmetric"),
                                         ("bf16>fp64", 7, "symmetric"), ("bf16>tf32>fp64/cbf16", 7, "symmetric"),
                                         ("bf16>fp64/cbf16", 7, "symmetric_tri"), ("fp16>fp64/cbf16", 10, "symmetric_tri"),
                                         ("bf16>tf32>fp64/cbf16", 7, "symmetric_tri"),
                                         ("fp8/cfp8>bf16>fp64/cbf16", 4, "symmetric_tri")])   # R-29
def test_mixed_level2(name, m, form):
    # Level 2: low-phase iterates within 4 * 2^-m of the oracle, the same switch
    # iteration (R-6: +-1 only at a tie), final C within 1e-10, certified rho <= 1e-12; and the
    # refinement claim: the FP64 phase needs far fewer iterations than the literal form (F4).
    n, p = 384, 2
    A = synth.spd(n, 2.0, 4)
    r, (out, tr, hist, best) = run_sym(A, p, name, 1e-12, 120, form)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    sw_g = [t["k"] for t in tr if t["decision"] == ipr.IPR_DEC_SWITCH]
    sw_o = [x["k"] for x in r.records if x["decision"] == oracle.SWITCH]
    assert len(sw_g) == len(sw_o) and all(abs(a - b) <= 1 for a, b in zip(sw_g, sw_o)), (sw_g, sw_o)
    for k, Ck in hist.items():
        if k <= sw_o[0]:
            assert rel_fro(Ck, r.C_hist[k]) <= 4 * 2.0 ** -m, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12
    n64 = sum(1 for t in tr if t["phase"] == len(sw_g))
    assert n64 <= 12, n64


@pytest.mark.parametrize("form", ["symmetric", "symmetric_tri"])
def test_run_to_run_deterministic_and_symmetric(form):
    A = synth.spd(640, 2.0, 3)
    pg, _ = schedules("bf16>fp64/cbf16")
    res = []
    for _ in range(2):
        out, tr, hist, best = run_gpu_trajectory(A, 2, pg, 1e-12, 60, form=form)
        res.append((tr, best))
        assert np.array_equal(best, best.T)
    (t1, b1), (t2, b2) = res
    for key in ("rho", "delta", "decision", "rho_cert"):
        assert np.array_equal([a[key] for a in t1], [a[key] for a in t2], equal_nan=True), key
    # every continuing record has its update's delta; a converged record has none when the p = 2
    # certification ran before the update (include/ipr.h: "NaN if none")
    assert all(np.isfinite(a["delta"]) for a in t1 if a["decision"] == ipr.IPR_DEC_CONTINUE)
    np.testing.assert_array_equal(b1, b2)


def test_config_c3_family_level3_envelope():
    # BASELINE config C3's family (kappa = 1e4, p = 2) at n = 1024: the form is unstable there
    # (kappa > 34, reading R-22), so Level 3: same outcome class and min rho within 4x.
    A = synth.spd(1024, 1e4, 2)
    pg, po = schedules("bf16>fp64/cbf16")
    r = oracle.solve(A, 2, po, 1e-12, 80, form=oracle.FORM_SYMMETRIC)
    out, tr, _, _ = run_gpu_trajectory(A, 2, pg, 1e-12, 80, keep=False, form="symmetric")
    mg = min(t["rho"] for t in tr if np.isfinite(t["rho"]))        # R-33 records have rho = NaN
    mo = min(x["rho"] for x in r.records if np.isfinite(x["rho"]))
    assert mg <= 4 * mo and mo <= 4 * mg
    assert (out == ipr.IPR_CONVERGED) == (r.outcome == oracle.CONVERGED)


def test_errors():
    A = torch_cuda(synth.spd(64, 2.0, 0))
    s = ipr.Solver(A, 1, [ipr.make_phase("fp64")], 1e-12, form="symmetric")
    with pytest.raises(ipr.IprError) as e:
        s.iterate(1)
    assert e.value.status == ipr.IPR_E_INVALID_ARG
    s.close()
    s = ipr.Solver(A, 2, [ipr.make_phase("fp16", max_iters=3, corr_prec="fp8"), ipr.make_phase("fp64")], 1e-12,
                   form="symmetric")
    with pytest.raises(ipr.IprError) as e:   # a scaled correction format is not defined
        s.iterate(1)
    assert e.value.status == ipr.IPR_E_UNSUPPORTED
    s.close()
    with pytest.raises(ipr.IprError) as e:
        ipr.Solver(A, 2, [ipr.make_phase("bf16", corr_prec="fp64")], 1e-12, form="symmetric")
    assert e.value.status == ipr.IPR_E_INVALID_ARG


def test_tri_close_to_full_and_errors():
    A = synth.spd(512, 2.0, 8)
    pg, _ = schedules("bf16>fp64/cbf16")
    _, t_full, _, b_full = run_gpu_trajectory(A, 2, pg, 1e-12, 60, keep=False, form="symmetric")
    _, t_tri, _, b_tri = run_gpu_trajectory(A, 2, pg, 1e-12, 60, keep=False, form="symmetric_tri")
    assert rel_fro(b_tri, b_full) <= 1e-12
    assert abs(len(t_tri) - len(t_full)) <= 1
    At = torch_cuda(A)
    s = ipr.Solver(At, 3, [ipr.make_phase("fp64")], 1e-12, form="symmetric_tri")
    with pytest.raises(ipr.IprError) as e:
        s.iterate(1)
    assert e.value.status == ipr.IPR_E_INVALID_ARG
    s.close()


def test_fused_symmetric_update_matches_separate():
    # EPI_SYMUPD (off by default, IPR_FUSED_SYMUPD=1): S = W + W^T from one K-concatenated upper-triangle
    # GEMM with the update in its epilogue -- same trajectory class as W GEMM + k_sym_update, checked in a
    # subprocess so the process-wide switch does not leak into the other tests
    import os, subprocess, sys, json
    code = (
        "import json, numpy as np, synth, torch, paper_1703_02283_b200 as ipr\n"
        "from tests.gpu_util import run_gpu_trajectory\n"
        "A = synth.spd(640, 2.0, 3)\n"
        "low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)\n"
        "pg = [ipr.make_phase('bf16', **low), ipr.make_phase('fp64crt', mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec='bf16')]\n"
        "out, tr, hist, best = run_gpu_trajectory(A, 2, pg, 1e-12, 80, form='symmetric_tri')\n"
        "np.save('/tmp/ipr_fused_best.npy', best)\n"
        "print(json.dumps(dict(out=out, n=len(tr), cert=tr[-1]['rho_cert'], sym=bool(np.array_equal(best, best.T)))))\n")
    env = dict(os.environ, IPR_FUSED_SYMUPD="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["out"] == ipr.IPR_CONVERGED and res["cert"] <= 1e-12 and res["sym"], res
    fused = np.load("/tmp/ipr_fused_best.npy")
    A = synth.spd(640, 2.0, 3)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    pg = [ipr.make_phase("bf16", **low), ipr.make_phase("fp64crt", mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec="bf16")]
    out, tr, hist, best = run_gpu_trajectory(A, 2, pg, 1e-12, 80, form="symmetric_tri")
    assert out == ipr.IPR_CONVERGED
    assert rel_fro(fused, best) <= 1e-10
    assert abs(res["n"] - len(tr)) <= 1


def test_missed_certificates_respect_the_phase_cap():
    # the oracle's test_missed_certificates_respect_the_phase_cap on the GPU (n = 32768 showed the need:
    # in-chain rho below 1e-12, FP64 certificate floor 1.86e-12 -- every certificate missed until the
    # caller's budget): a tolerance between the two floors ends at the last phase's cap, ITER_LIMIT
    n, cap = 300, 10
    A = synth.spd(n, 2.0, 33)
    pg = [ipr.make_phase("bf16", **LOW), ipr.make_phase("fp64", corr_prec="bf16", max_iters=cap)]
    out, tr, _, _ = run_gpu_trajectory(A, 2, pg, 1e-14, 200, keep=False, form="symmetric")
    assert out == ipr.IPR_ITER_LIMIT
    assert sum(1 for t in tr if t["phase"] == 1) == cap
    assert tr[-1]["decision"] == ipr.IPR_ITER_LIMIT       # terminal decisions equal the outcome codes
    assert sum(1 for t in tr if t["rho_cert"] == t["rho_cert"]) >= 2


@pytest.mark.parametrize("sched", ["symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", "symtri:bf16>fp64/cbf16"])
def test_run_to_run_deterministic_scaled_tri_phases(sched):
    # R-36's GEMM 1 on the upper tiles writes the lower elements of its diagonal tiles only through the
    # mirror stores (an FP32-scratch path that also stored them raced with those mirrors -- found by
    # tools/z1_det_probe.py): n = 2048 (8 diagonal pair tiles), every record and the answer bit-identical
    import bench
    A = torch.from_numpy(synth.spd(2048, 2.0, 9)).cuda()
    form, ph = bench.schedule(sched, 2048)
    res = []
    for _ in range(2):
        s = ipr.Solver(A, 2, ph, 1e-12, form=form, cert="crt" if "crt" in sched else "fp64")
        s.iterate(200)
        res.append((s.trace(), s.finalize().cpu().numpy()))
    (t1, b1), (t2, b2) = res
    assert t1[-1]["decision"] == 1   # IPR_DEC_CONVERGED
    for key in ("rho", "delta", "decision", "rho_cert"):
        assert np.array_equal([a[key] for a in t1], [a[key] for a in t2], equal_nan=True), key
    np.testing.assert_array_equal(b1, b2)
