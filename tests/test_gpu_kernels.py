"""GPU parity of the individual kernels, called through the C-ABI (include/ipr_testing.h):
quantisers bit-exact vs the oracle's q_m, norms and C_0 bit-exact, GEMM within the FP
accumulation bound.  Oracle = tests' reference (oracle/), never imported by the product."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import gpu_c0, torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

RNG = np.random.default_rng(99)


def _wide(count):
    e = RNG.uniform(-160, 140, size=count)
    x = np.exp2(e) * RNG.choice([-1.0, 1.0], size=count)
    x[:1000] = RNG.standard_normal(1000)
    x[1000:1010] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0, 2.0 ** -149, 2.0 ** -126, 3.4e38]
    ties = [s * (1.0 + k * 2.0 ** -(m + 1)) * 2.0 ** e for m in range(24) for k in (1, 3)
            for e, s in ((0, 1.0), (127, -1.0), (-126, 1.0))]     # RNE ties at every m, at the range ends
    x[1010:1010 + len(ties)] = ties
    return x


def _eq_bits(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return np.array_equal(a.view(np.uint64)[~both_nan], b.view(np.uint64)[~both_nan])


@pytest.mark.parametrize("mode", [0, 7])    # 7: the update's branch-free path (QRound) + fallback
@pytest.mark.parametrize("m", [0, 2, 7, 10, 16, 23])
@pytest.mark.parametrize("rtz", [0, 1])
def test_quant_e8_container(m, rtz, mode):
    x = _wide(1 << 20)
    y = torch.empty(x.size, dtype=torch.float32, device="cuda")
    ipr.ipr_test_quantize(mode, torch_cuda(x), y, m=m, round=rtz)
    assert _eq_bits(y.cpu().numpy().astype(np.float64), oracle.qm(x, 8, m, bool(rtz)))


@pytest.mark.parametrize("mode", [1, 8])    # 8: the update's branch-free path (QRound) + fallback
@pytest.mark.parametrize("m", [0, 7, 10, 23, 40, 52])
@pytest.mark.parametrize("rtz", [0, 1])
def test_quant_e11_container(m, rtz, mode):
    x = np.concatenate([_wide(1 << 19), RNG.standard_normal(1 << 18) * 1e-310,
                        np.exp2(RNG.uniform(1000, 1024, 1 << 16))])
    y = torch.empty(x.size, dtype=torch.float64, device="cuda")
    ipr.ipr_test_quantize(mode, torch_cuda(x), y, m=m, round=rtz)
    assert _eq_bits(y.cpu().numpy(), oracle.qm(x, 11, m, bool(rtz)))


def test_operand_bf16_tf32_fp16():
    x32 = _wide(1 << 20).astype(np.float32)
    xin = torch_cuda(x32)
    out16 = torch.empty(x32.size, dtype=torch.int16, device="cuda")
    ipr.ipr_test_quantize(2, xin, out16)
    got = (out16.cpu().numpy().astype(np.uint16).astype(np.uint32) << 16).view(np.float32)
    assert _eq_bits(got.astype(np.float64), oracle.qm(x32.astype(np.float64), 8, 7))
    out32 = torch.empty(x32.size, dtype=torch.float32, device="cuda")
    ipr.ipr_test_quantize(3, xin, out32)
    assert _eq_bits(out32.cpu().numpy().astype(np.float64), oracle.qm(x32.astype(np.float64), 8, 10))
    for sigma in [-3, 0, 14, 30]:
        ipr.ipr_test_quantize(4, xin, out16, sigma=sigma)
        got = out16.cpu().numpy().view(np.float16).astype(np.float64)
        ref = oracle.qm(x32.astype(np.float64) * 2.0 ** sigma, 5, 10)
        assert _eq_bits(got, ref)


def test_bf16_exhaustive_vs_torch():
    # all 2^32 FP32 patterns: the device operand conversion equals torch's RNE bf16 conversion
    step = 1 << 28
    out = torch.empty(step, dtype=torch.int16, device="cuda")
    for base in range(0, 1 << 32, step):
        bits = torch.arange(base, base + step, dtype=torch.int64, device="cuda").to(torch.int32)
        x = bits.view(torch.float32)
        ipr.ipr_test_quantize(2, x, out)
        ref = x.to(torch.bfloat16).view(torch.int16)
        fin = ~torch.isnan(x)
        assert torch.equal(out[fin], ref[fin])
        del bits, x, ref, fin


@pytest.mark.parametrize("n,kappa", [(64, 1e2), (300, 10.0), (1000, 1e3)])
def test_norms_and_c0_bit_exact(n, kappa):
    A = synth.spd(n, kappa, 1)
    n1, ninf, md = oracle.norms(A)
    for ph_gpu, ph_orc in [(ipr.make_phase("fp64"), oracle.phase()),
                           (ipr.make_phase("fp64", mant_bits=7, round="rtz"),
                            oracle.phase(oracle.FP64, mant_bits=7, round=oracle.RTZ))]:
        C0, nrm = gpu_c0(A, ph_gpu)
        assert nrm[0] == n1 and nrm[1] == ninf and nrm[2] == md and nrm[3] == n1 * ninf
        np.testing.assert_array_equal(C0, oracle.c0(A, n1 * ninf, ph_orc))


@pytest.mark.parametrize("n", [1, 64, 200, 300, 513])
def test_gemm_fp64_vs_oracle(n):
    X = RNG.standard_normal((n, n))
    Y = RNG.standard_normal((n, n))
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_gemm(ipr.IPR_FP64, n, torch_cuda(X), torch_cuda(Y.T), Z)
    ref = oracle.gemm(X, Y)
    bound = 2 * n * 2.0 ** -53 * (np.abs(X) @ np.abs(Y))
    assert np.all(np.abs(Z.cpu().numpy() - ref) <= bound + 1e-300)


def test_gemm_fp64_exact_integers():
    n = 257
    X = RNG.integers(-64, 64, (n, n)).astype(np.float64)
    Y = RNG.integers(-64, 64, (n, n)).astype(np.float64)
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ipr.ipr_test_gemm(ipr.IPR_FP64, n, torch_cuda(X), torch_cuda(Y.T), Z)
    np.testing.assert_array_equal(Z.cpu().numpy(), oracle.gemm(X, Y))


def test_not_symmetric_rejected():
    A = synth.spd(130, 5.0, 2)
    A[5, 77] = np.nextafter(A[5, 77], 2.0)
    with pytest.raises(ipr.IprError) as e:
        ipr.Solver(torch_cuda(A), 2, [ipr.make_phase("fp64")])
    assert e.value.status == ipr.IPR_E_NOT_SYMMETRIC


def test_schedule_validation():
    A = torch_cuda(synth.spd(64, 5.0, 3))
    ctx = ipr.ipr_init(64, A)
    try:
        with pytest.raises(ipr.IprError) as e:
            ipr.ipr_set_schedule(ctx, 0, [ipr.make_phase("fp64")], 1e-12)
        assert e.value.status == ipr.IPR_E_INVALID_ARG
        with pytest.raises(ipr.IprError) as e:   # precision must not decrease
            ipr.ipr_set_schedule(ctx, 2, [ipr.make_phase("fp64"), ipr.make_phase("fp64", mant_bits=7)], 1e-12)
        assert e.value.status == ipr.IPR_E_INVALID_ARG
        with pytest.raises(ipr.IprError) as e:
            ipr.ipr_iterate(ctx, 1)
        assert e.value.status == ipr.IPR_E_STATE
    finally:
        ipr.ipr_finalize(ctx)
