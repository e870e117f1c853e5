"""GPU parity of the tcgen05 path (BF16 / FP16 / TF32 operands, FP32 accumulation in TMEM).

Kernel level: small-integer operands make every partial sum exact in FP32, so the tcgen05 GEMM
must equal the oracle's FP64 triple loop bit for bit -- this pins the TMA / UMMA descriptor
layouts (a transposed or mis-strided operand fails it).  Random operands: within the FP32
accumulation bound.  Trajectory level: diagonal A bit-exact in every low phase (P4), and the
stable twin within 4 * 2^-m per iteration up to the switch with the same switch iteration,
then the FP64 answer within 1e-10 (north star tolerances)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory, torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

RNG = np.random.default_rng(5)
PRECS = {"bf16": (ipr.IPR_BF16, oracle.BF16), "tf32": (ipr.IPR_TF32, oracle.TF32),
         "fp16": (ipr.IPR_FP16, oracle.FP16)}


def _as_operand(x, prec):
    """numpy float64 values (already on the operand grid) -> CUDA tensor in the operand format."""
    if prec == ipr.IPR_BF16:
        return torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).view(torch.int16).cuda()
    if prec == ipr.IPR_FP16:
        return torch.from_numpy(x.astype(np.float16).view(np.int16)).cuda()
    return torch.from_numpy(x.astype(np.float32)).cuda()


def _gemm(prec, X, Y):
    n = X.shape[0]
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_gemm(prec, n, _as_operand(X, prec), _as_operand(np.ascontiguousarray(Y.T), prec), Z)
    return Z.cpu().numpy()


@pytest.mark.parametrize("name", ["bf16", "tf32", "fp16"])
@pytest.mark.parametrize("n", [1, 64, 256, 300, 777])
def test_tc_gemm_exact_integers(name, n):
    prec, _ = PRECS[name]
    X = RNG.integers(-16, 17, (n, n)).astype(np.float64)
    Y = RNG.integers(-16, 17, (n, n)).astype(np.float64)
    np.testing.assert_array_equal(_gemm(prec, X, Y), oracle.gemm(X, Y))


def test_tc_gemm_structured_single_tile():
    # distinct values per (row, k) and (k, col): catches swapped / mis-swizzled K chunks
    n = 256
    i = np.arange(n)
    X = ((i[:, None] * 7 + i[None, :] * 3) % 17 - 8).astype(np.float64)
    Y = ((i[:, None] * 5 + i[None, :] * 11) % 13 - 6).astype(np.float64)
    np.testing.assert_array_equal(_gemm(ipr.IPR_BF16, X, Y), oracle.gemm(X, Y))
    E = np.zeros((n, n)); E[3, 200] = 1.0
    Z = _gemm(ipr.IPR_BF16, np.eye(n), E)
    np.testing.assert_array_equal(Z, E)


@pytest.mark.parametrize("name", ["bf16", "tf32", "fp16"])
@pytest.mark.parametrize("n", [128, 513, 1024])
def test_tc_gemm_random_bound(name, n):
    prec, oprec = PRECS[name]
    E, M = oracle.prec_format(oprec)
    X = oracle.qm(RNG.standard_normal((n, n)), E, M)
    Y = oracle.qm(RNG.standard_normal((n, n)), E, M)
    Z = _gemm(prec, X, Y)
    ref = oracle.gemm(X, Y)
    bound = n * 2.0 ** -22 * (np.abs(X) @ np.abs(Y))
    assert np.all(np.abs(Z - ref) <= bound)


LOW = {"bf16": 7, "tf32": 10, "fp16": 10}


@pytest.mark.parametrize("name", ["bf16", "tf32", "fp16"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_diagonal_bit_exact_low_phase(name, p):
    prec, oprec = PRECS[name]
    A = synth.diag_spd(200, 1e2, 3 + p)
    pho = [oracle.phase(oprec, switch_tol=1e-2, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
           oracle.phase(oracle.FP64)]
    phg = [ipr.make_phase(name, switch_tol=1e-2, plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
           ipr.make_phase("fp64")]
    r = oracle.solve(A, p, pho, 1e-13, 150, hist=150)
    out, tr, hist, best = run_gpu_trajectory(A, p, phg, 1e-13, 150)
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)


@pytest.mark.parametrize("name", ["bf16", "tf32", "fp16"])
@pytest.mark.parametrize("n,p", [(300, 2), (512, 3), (256, 1)])
def test_stable_twin_mixed(name, n, p):
    prec, oprec = PRECS[name]
    m = LOW[name]
    # p = 1 at kappa = 2 sits exactly on the neutral mode |mu|max = 1 of Eq. (1):
    # low-precision noise then never decays, so the p = 1 twin uses kappa = 1.5 < kappa_1 = 2.
    A = synth.spd(n, 2.0 if p > 1 else 1.5, 11)
    pho = [oracle.phase(oprec, switch_tol=1e-2 * np.sqrt(n), plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
           oracle.phase(oracle.FP64)]
    phg = [ipr.make_phase(name, switch_tol=1e-2 * np.sqrt(n), plateau_ratio=0.7, plateau_arm=0.5, max_iters=40),
           ipr.make_phase("fp64")]
    r = oracle.solve(A, p, pho, 1e-12, 300, hist=300)
    out, tr, hist, best = run_gpu_trajectory(A, p, phg, 1e-12, 300)
    sw_o = next(k for k, x in enumerate(r.records) if x["decision"] == oracle.SWITCH)
    sw_g = next(k for k, x in enumerate(tr) if x["decision"] == ipr.IPR_DEC_SWITCH)
    # same switch iteration (R-6 tie rule: +-1 only if the oracle's crossing is within 4 u_m)
    x = r.records[sw_o]
    tie = abs(x["rho"] - 1e-2 * np.sqrt(n)) <= 4 * 2.0 ** -m * x["rho"]
    assert sw_g == sw_o or (tie and abs(sw_g - sw_o) <= 1)
    for k in range(1, min(sw_o, sw_g) + 1):
        assert rel_fro(hist[k], r.C_hist[k]) <= 4 * 2.0 ** -m, k
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    assert tr[-1]["rho"] <= 1e-12
    assert rel_fro(best, r.C_best) <= 1e-10
