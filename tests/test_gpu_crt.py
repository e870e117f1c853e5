"""GPU parity of IPR_FP64_CRT (reading R-28): FP64 GEMMs on the INT8 tensor cores by the
Ozaki scheme II -- rows / columns quantised to b-bit integers, the integer product exact modulo
N pairwise coprime moduli (one kind::i8 GEMM each), Chinese-remainder reconstruction in exact
sliced FP64 arithmetic.

Kernel level: bit-exact on integer operands that the quantisation keeps (b = 17); at b = 59 the
error against an extended-precision reference is within the bound of the method (quantisation
2^-b relative to the row / column maximum, plus the final rounding), and comparable to the FP64
DMMA product, and element-wise against the oracle's definition of the CRT product (oracle.gemm_crt:
the b-bit quantisations' exact integer product, one rounding).  Trajectory level: the symmetric forms'
FP64-range phase on IPR_FP64_CRT against the oracle's FP64_CRT phase (the same quantised products at
the same per-chain bits, R-26 / R-28), at the Level-2 FP64 tolerance."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")


def _gemm(prec, X, Y, digits=9, signed=False):
    n = X.shape[0]
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_set_digits(digits)
    ipr.ipr_test_crt_signed(signed)       # symmetric residues (s8 x s8), the large-K convention
    try:
        ipr.ipr_test_gemm(prec, n, torch.from_numpy(np.ascontiguousarray(X)).cuda(),
                          torch.from_numpy(np.ascontiguousarray(Y.T)).cuda(), Z)
    finally:
        ipr.ipr_test_set_digits(9)
        ipr.ipr_test_crt_signed(False)
    return Z.cpu().numpy()


@pytest.mark.parametrize("signed", [False, True])
@pytest.mark.parametrize("n", [1, 200, 513, 1024])
def test_crt_integers_exact(n, signed):
    # digits 3 -> b = 17 bits: |x| <= 2^10 is kept exactly, |Pbar| < 2^53 (exact reconstruction); both
    # residue conventions (u8 residues in [0, m) below K = 33025, symmetric s8 residues beyond)
    rng = np.random.default_rng(n)
    X = rng.integers(-1024, 1025, (n, n)).astype(np.float64)
    Y = rng.integers(-1024, 1025, (n, n)).astype(np.float64)
    np.testing.assert_array_equal(_gemm(ipr.IPR_FP64_CRT, X, Y, digits=3, signed=signed), X @ Y)


@pytest.mark.parametrize("signed", [False, True])
def test_crt_long_rows_sampled_vs_oracle_definition(signed):
    # K = 8448 > 8192: the residue split's two-pass (non-shared-memory) path, both conventions, against
    # the oracle's exact CRT definition on sampled elements (the full product is too large for the oracle)
    n, b = 8448, ipr.ipr_test_crt_table(18, 9, 8448)["b_for"]
    rng = np.random.default_rng(88)
    X = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-20, 21, n)[:, None]
    Y = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-20, 21, n)[None, :]
    Zg = _gemm(ipr.IPR_FP64_CRT, X, Y, 9, signed)
    I, J = rng.integers(0, n, 3000), rng.integers(0, n, 3000)
    Zo = oracle.gemm_crt_pairs(X, Y, b, I, J)
    d = np.abs(Zg[I, J] - Zo)
    assert np.all(d <= 2 * np.spacing(np.abs(Zo))), float(np.max(d / np.spacing(np.abs(Zo))))
    assert float(np.mean(Zg[I, J] == Zo)) >= 0.9


@pytest.mark.parametrize("n,kappa,digits", [(512, 2.0, 9), (1536, 2.0, 9), (1024, 1e3, 9), (777, 2.0, 5)])
def test_crt_error_within_method_bound(n, kappa, digits):
    A, lam, Q = synth.spd(n, kappa, 3, return_eig=True)
    C = (Q * lam ** -0.5) @ Q.T
    C = (C + C.T) / 2
    b = ipr.ipr_test_crt_table(18, digits, n)["b_for"]
    assert b == 7 * digits - 4
    L = np.longdouble
    exact = A.astype(L) @ C.astype(L)
    Z = _gemm(ipr.IPR_FP64_CRT, A, C, digits)
    err = np.abs(Z.astype(L) - exact)
    # |xhat - x| <= 2^-b max_k |x_ik| (rows of A), the same for the columns of C; final rounding 2 u
    ra = np.abs(A).max(axis=1)[:, None].astype(L)
    cc = np.abs(C).max(axis=0)[None, :].astype(L)
    bound = 2.0 ** -b * (ra * np.abs(C).sum(axis=0)[None, :] + (np.abs(A).sum(axis=1)[:, None] + n * ra * 2.0 ** -b) * cc)
    bound = bound * (1 + 1e-12) + 2.0 ** -51 * np.abs(exact)
    assert np.all(err <= bound), float(np.max(err / bound))
    if digits == 9:
        e_cr = np.linalg.norm(err.astype(np.float64))
        e_dm = np.linalg.norm((_gemm(ipr.IPR_FP64, A, C) - exact).astype(np.float64))
        assert e_cr <= 2.0 * e_dm, (e_cr, e_dm)


@pytest.mark.parametrize("signed", [False, True])
@pytest.mark.parametrize("n,digits", [(1, 9), (37, 3), (256, 5), (300, 9), (513, 7), (1024, 9)])
def test_crt_gemm_matches_oracle_definition(n, digits, signed):
    # R-28's definition computed exactly by the oracle (integer product exact, one rounding) vs the
    # GPU's modular products + sliced FP64 reconstruction, element by element, on operands with rows /
    # columns spanning 2^+-40 (so e_i, f_j differ per row / column) and both signs
    rng = np.random.default_rng(1000 + n)
    X = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-40, 41, n)[:, None]
    Y = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-40, 41, n)[None, :]
    if n > 2:
        X[1] = 0.0                     # a zero row: e = 0, Z row exactly 0
        Y[:, 2] = 0.0
    b = ipr.ipr_test_crt_table(18, digits, n)["b_for"]
    assert b == oracle.crt_bits(digits, n)
    Zg = _gemm(ipr.IPR_FP64_CRT, X, Y, digits, signed)
    Zo = oracle.gemm_crt(X, Y, b)
    ulp = np.spacing(np.abs(Zo))
    d = np.abs(Zg - Zo)
    assert np.all(d <= 2 * ulp), float(np.max(d / ulp))
    exact_frac = float(np.mean(Zg == Zo))
    assert exact_frac >= 0.9, exact_frac


def test_crt_matches_digits_scheme():
    # schemes I and II compute the same FP64 product to within their (FP64-level) errors
    n = 640
    A = synth.spd(n, 2.0, 4)
    C = np.linalg.inv(A)
    C = (C + C.T) / 2
    z1, z2 = _gemm(ipr.IPR_FP64_OZ, A, C), _gemm(ipr.IPR_FP64_CRT, A, C)
    assert np.max(np.abs(z1 - z2)) <= 64 * n * 2.0 ** -53 * np.max(np.abs(A)) * np.max(np.abs(C))


@pytest.mark.parametrize("form,sched", [("symmetric", "fp64crt"), ("symmetric_tri", "fp64crt"),
                                        ("symmetric_tri", "bf16>fp64crt/cbf16")])
def test_crt_fp64_phase_level2(form, sched):
    n, p = 520, 2
    A = synth.spd(n, 2.0, 12)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    OPR = {"bf16": oracle.BF16, "fp64crt": oracle.FP64_CRT}
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
    if len(parts) == 1:
        for k, Ck in hist.items():
            if k < len(r.records):
                assert rel_fro(Ck, r.C_hist[k]) <= 1e-10, k
    else:
        sw = next(k for k, x in enumerate(r.records) if x["decision"] == oracle.SWITCH)
        for k in range(1, sw + 1):
            assert rel_fro(hist[k], r.C_hist[k]) <= 4 * 2.0 ** -7, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12
    nm = ipr.ipr_test_crt_table(18, 59, n)["n_for"]                            # b = 59 at n = 520
    # chain records (a certificate-only record, reading R-33, runs no CRT product: moduli 0)
    assert all(t["moduli"] == nm for t in tr if t["phase"] == len(parts) - 1 and t["rho"] == t["rho"])


@pytest.mark.parametrize("signed", [False, True])
def test_crt_adaptive_level2_and_storage_rule(signed):
    ipr.ipr_test_crt_signed(signed)      # the whole solve with the large-K residue convention too
    try:
        _adaptive_level2()
    finally:
        ipr.ipr_test_crt_signed(False)


def _adaptive_level2():
    n, p = 520, 2
    A = synth.spd(n, 2.0, 12)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    pg = [ipr.make_phase("bf16", **low), ipr.make_phase("fp64crt", mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec="bf16")]
    po = [oracle.phase(oracle.BF16, **low), oracle.phase(oracle.FP64_CRT, mant_bits=oracle.MANT_ADAPTIVE,
                                                         corr_prec=oracle.BF16)]
    r = oracle.solve(A, p, po, 1e-12, 80, hist=80, form=oracle.FORM_SYMMETRIC_TRI)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-12, 80, form="symmetric_tri")
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    mg = [t["mant_bits"] for t in tr if t["phase"] == 1]
    mo = [x["mant_bits"] for x in r.records if x["phase"] == 1]
    assert len(set(mg)) >= 3 and mg[-1] == 52
    agree = sum(a == b for a, b in zip(mg, mo))
    assert agree >= min(len(mg), len(mo)) - 1, (mg, mo)
    mods = [t["moduli"] for t in tr if t["phase"] == 1 and t["rho"] == t["rho"]]   # chain records (R-33)
    assert mods == sorted(mods) and mods[0] < mods[-1] == ipr.ipr_test_crt_table(18, 59, n)["n_for"]
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12


def test_crt_unsupported_outside_symmetric_forms():
    A = torch.from_numpy(synth.spd(64, 2.0, 0)).cuda()
    s = ipr.Solver(A, 2, [ipr.make_phase("fp64crt")], 1e-12)
    with pytest.raises(ipr.IprError) as e:
        s.iterate(1)
    assert e.value.status == ipr.IPR_E_UNSUPPORTED
    s.close()


def test_crt_product_full_size_sampled_rows():
    # the bench's launch configuration (n = 8192, 2 moduli per launch, S = 9 -> b = 59, 17 moduli):
    # sampled rows of Z = A A against the oracle's FP64 matvec, within the method's bound plus the
    # reference's own FP64 rounding
    n = 8192
    A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
    Z = torch.empty_like(A)
    ipr.ipr_test_gemm(ipr.IPR_FP64_CRT, n, A, A, Z)      # A symmetric: its K-major form is A itself
    A_np, Z_np = A.cpu().numpy(), Z.cpu().numpy()
    b = ipr.ipr_test_crt_table(18, 9, n)["b_for"]
    absA = np.abs(A_np)
    rmax = absA.max(axis=1)
    colsum = absA.sum(axis=0)
    for i in [0, 1, 4097, 8191]:
        ref = oracle.matvec(A_np, A_np[i])            # row i of A A (A symmetric)
        mag = oracle.matvec(absA, absA[i])
        bound = 2.0 ** -b * (rmax[i] * colsum + (absA[i].sum() + n * rmax[i] * 2.0 ** -b) * rmax) \
            + 2.0 ** -51 * np.abs(ref) + n * 2.0 ** -53 * mag
        assert np.all(np.abs(Z_np[i] - ref) <= bound), (i, float(np.max(np.abs(Z_np[i] - ref) / bound)))


@pytest.mark.parametrize("form,p,sched", [
    ("symmetric_tri", 2, "bf16>fp64crt@23/cbf16>fp64crt/cbf16"),   # staged precision: 23 stored bits, then 52
    ("symmetric_tri", 2, "tf32>fp64crt/ctf32"),                     # TF32 correction GEMM
    ("symmetric", 3, "bf16>fp64crt/cbf16"),                          # p = 3 (full symmetric form)
    ("symmetric_tri", 2, "fp8>bf16>fp64crt@a/cbf16"),               # BF16 correction in the FP8 phase
    ("symmetric_tri", 2, "fp8/cfp8>bf16>fp64crt@a/cbf16"),          # the bench's headline schedule (R-29)
])
def test_crt_schedules_level2(form, p, sched):
    n = 520
    A = synth.spd(n, 2.0, 12)
    low = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)
    OPR = {"bf16": oracle.BF16, "tf32": oracle.TF32, "fp8": oracle.FP8, "fp64crt": oracle.FP64_CRT}
    pg, po = [], []
    parts = sched.split(">")
    for i, part in enumerate(parts):
        part, _, m = part.partition("@")
        if "/c" in m:
            m, _, corr = m.partition("/c")
            part = part + "/c" + corr
        prec, _, corr = part.partition("/c")
        mb = (-2 if m == "a" else int(m)) if m else -1
        kw = {} if i == len(parts) - 1 else low
        pg.append(ipr.make_phase(prec, mant_bits=mb, corr_prec=corr or -1, **kw))
        po.append(oracle.phase(OPR[prec], mant_bits=mb, corr_prec=OPR[corr] if corr else -1, **kw))
    oform = oracle.FORM_SYMMETRIC if form == "symmetric" else oracle.FORM_SYMMETRIC_TRI
    r = oracle.solve(A, p, po, 1e-12, 120, hist=120, form=oform)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-12, 120, form=form)
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert abs(len(tr) - len(r.records)) <= 2
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12
    assert any(t["moduli"] > 0 for t in tr)
    C = best
    # defining property: C^p A = I on probe vectors
    for v in synth.probe_vectors(n, 3, 2):
        x = A @ v
        for _ in range(p):
            x = C @ x
        assert np.linalg.norm(x - v) / np.linalg.norm(v) < 1e-11


def test_crt_extreme_row_scales():
    # rows / columns scaled by 2^+-900: the split's exponent e_i leaves the pow2 range (|e| > 1022) and
    # the finish must unscale by 2^-(e_i + f_j) without under/overflow -- exact on integers times powers
    # of two (the scaled product is representable)
    n = 256
    rng = np.random.default_rng(3)
    X = rng.integers(-64, 65, (n, n)).astype(np.float64)
    Y = rng.integers(-64, 65, (n, n)).astype(np.float64)
    rs = np.where(np.arange(n) % 3 == 0, 2.0 ** -900, np.where(np.arange(n) % 3 == 1, 2.0 ** 900, 1.0))
    cs = np.where(np.arange(n) % 2 == 0, 2.0 ** -60, 2.0 ** 60)
    Xs, Ys = X * rs[:, None], Y * cs[None, :]
    Z = _gemm(ipr.IPR_FP64_CRT, Xs, Ys, digits=3)
    ref = (X @ Y) * rs[:, None] * cs[None, :]
    np.testing.assert_array_equal(Z, ref)
