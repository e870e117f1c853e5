"""GPU parity of NEXT-3: FP8 E4M3 (tcgen05 kind::f8f6f4, FP32 accumulate) and INT8
fixed point (kind::i8, exact INT32 accumulate) operand formats, each with a per-tensor
power-of-two scale (reading R-20).  PAPER.md:263-267 (2 stored mantissa bits still converge in
storage-only mode) and :268-281 (fixed-point storage) motivate them.

Kernel level: the device quantisers equal the oracle's (one RNE rounding from FP64; nearest-even
integer saturated to +-127); the tcgen05 GEMM on exact operands equals the exact product bit for
bit (pins the 1-byte TMA / UMMA descriptors and the instruction-descriptor formats).  Trajectory
level: diagonal A bit-exact through FP8 / INT8 phases (literal and symmetric forms); the kappa = 2
twin within 4 * 2^-m up to the switch, same switch iteration, FP64 answer within 1e-10."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel_fro, run_gpu_trajectory, torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

RNG = np.random.default_rng(8)


def _quant_fp8(x, sigma):
    y = torch.empty(x.size, dtype=torch.uint8, device="cuda")
    ipr.ipr_test_quantize(5, torch_cuda(x), y, sigma=sigma)
    return y.view(torch.float8_e4m3fn).to(torch.float64).cpu().numpy()


def _quant_int8(x, sigma):
    y = torch.empty(x.size, dtype=torch.int8, device="cuda")
    ipr.ipr_test_quantize(6, torch_cuda(x), y, sigma=sigma)
    return y.to(torch.float64).cpu().numpy()


@pytest.mark.parametrize("sigma", [0, 5, -3])
def test_fp8_quantiser_matches_oracle(sigma):
    x = RNG.standard_normal(300_000) * np.exp(RNG.uniform(-14, 4, 300_000))
    x = x[np.abs(x * 2.0 ** sigma) < 127]
    ties = (np.arange(-200, 200) + 0.5) * 2.0 ** -9 * 2.0 ** -sigma      # subnormal-range ties
    x = np.concatenate([x, ties, [0.0, -0.0]])
    ref = oracle.qm(np.ldexp(x, sigma), 4, 3)
    np.testing.assert_array_equal(_quant_fp8(x, sigma), ref)


@pytest.mark.parametrize("sigma", [0, 6, -2])
def test_int8_quantiser_matches_oracle(sigma):
    x = RNG.uniform(-140, 140, 200_000) * 2.0 ** -sigma
    x = np.concatenate([x, (np.arange(-130, 130) + 0.5) * 2.0 ** -sigma])
    ref = np.array([oracle.q_int8(v) for v in np.ldexp(x, sigma)])
    np.testing.assert_array_equal(_quant_int8(x, sigma), ref)


def _op(x, prec):
    if prec == ipr.IPR_FP8:
        return torch.from_numpy(x.astype(np.float32)).to(torch.float8_e4m3fn).view(torch.uint8).cuda()
    return torch.from_numpy(x.astype(np.int8)).cuda()


def _gemm(prec, X, Y):
    n = X.shape[0]
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_gemm(prec, n, _op(X, prec), _op(np.ascontiguousarray(Y.T), prec), Z)
    return Z.cpu().numpy()


@pytest.mark.parametrize("n", [1, 64, 256, 300, 777])
def test_int8_gemm_exact(n):
    X = RNG.integers(-127, 128, (n, n)).astype(np.float64)
    Y = RNG.integers(-127, 128, (n, n)).astype(np.float64)
    np.testing.assert_array_equal(_gemm(ipr.IPR_INT8, X, Y), X @ Y)     # integers < 2^53: exact


@pytest.mark.parametrize("n", [1, 64, 256, 300, 777])
def test_fp8_gemm_exact_small_values(n):
    vals = np.array([-6, -4, -3, -2, -1.5, -1, -0.5, 0, 0.5, 1, 1.5, 2, 3, 4, 6])  # E4M3-exact
    X = RNG.choice(vals, (n, n))
    Y = RNG.choice(vals, (n, n))
    np.testing.assert_array_equal(_gemm(ipr.IPR_FP8, X, Y), oracle.gemm(X, Y))


def test_fp8_gemm_structured():
    n = 256
    i = np.arange(n)
    X = ((i[:, None] * 7 + i[None, :] * 3) % 9 - 4).astype(np.float64)
    Y = ((i[:, None] * 5 + i[None, :] * 11) % 7 - 3).astype(np.float64)
    np.testing.assert_array_equal(_gemm(ipr.IPR_FP8, X, Y), oracle.gemm(X, Y))
    np.testing.assert_array_equal(_gemm(ipr.IPR_INT8, X, Y), oracle.gemm(X, Y))


OPR = {"fp8": oracle.FP8, "int8": oracle.INT8, "bf16": oracle.BF16, "fp64": oracle.FP64}
LOWKW = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)


@pytest.mark.parametrize("name,form,p", [("fp8", "literal", 2), ("int8", "literal", 2), ("fp8", "literal", 1),
                                         ("fp8", "symmetric", 2), ("int8", "symmetric", 2),
                                         ("fp8", "symmetric_tri", 2), ("int8", "symmetric", 3)])
def test_diagonal_bit_exact(name, form, p):
    A = synth.diag_spd(200, 1e2, 4)
    oform = {"literal": oracle.FORM_LITERAL, "symmetric": oracle.FORM_SYMMETRIC,
             "symmetric_tri": oracle.FORM_SYMMETRIC_TRI}[form]
    po = [oracle.phase(OPR[name], **LOWKW), oracle.phase(oracle.BF16, **LOWKW), oracle.phase()]
    pg = [ipr.make_phase(name, **LOWKW), ipr.make_phase("bf16", **LOWKW), ipr.make_phase("fp64")]
    r = oracle.solve(A, p, po, 1e-13, 200, hist=200, form=oform)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-13, 200, form=form)
    assert r.outcome == oracle.CONVERGED and out == ipr.IPR_CONVERGED
    assert [t["decision"] for t in tr] == [x["decision"] for x in r.records]
    for k, Ck in hist.items():
        if k < len(r.records):
            np.testing.assert_array_equal(Ck, r.C_hist[k], err_msg=f"iterate {k}")
    np.testing.assert_array_equal(best, r.C_best)


@pytest.mark.parametrize("name,m", [("fp8", 3), ("int8", 7)])
def test_symmetric_twin_level2(name, m):
    n, p = 384, 2
    A = synth.spd(n, 2.0, 4)
    po = [oracle.phase(OPR[name], **LOWKW), oracle.phase(oracle.BF16, **LOWKW),
          oracle.phase(corr_prec=oracle.BF16)]
    pg = [ipr.make_phase(name, **LOWKW), ipr.make_phase("bf16", **LOWKW), ipr.make_phase("fp64", corr_prec="bf16")]
    r = oracle.solve(A, p, po, 1e-12, 150, hist=150, form=oracle.FORM_SYMMETRIC_TRI)
    out, tr, hist, best = run_gpu_trajectory(A, p, pg, 1e-12, 150, form="symmetric_tri")
    assert out == ipr.IPR_CONVERGED and r.outcome == oracle.CONVERGED
    sw_o = [x["k"] for x in r.records if x["decision"] == oracle.SWITCH]
    sw_g = [t["k"] for t in tr if t["decision"] == ipr.IPR_DEC_SWITCH]
    assert len(sw_o) == len(sw_g) == 2 and all(abs(a - b) <= 1 for a, b in zip(sw_o, sw_g)), (sw_o, sw_g)
    for k, Ck in hist.items():
        if k <= sw_o[0]:
            assert rel_fro(Ck, r.C_hist[k]) <= 4 * 2.0 ** -m, k
    assert rel_fro(best, r.C_best) <= 1e-10
    assert tr[-1]["rho_cert"] <= 1e-12
