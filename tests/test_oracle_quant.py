"""Pins of the oracle's q_m (approximate storage/arithmetic rounding, PAPER.md:191-194 [Sec. 4.2],
format footnotes PAPER.md:106-111) against things other than itself: SPEC/hand golden values,
IEEE library conversions (numpy float16/float32, torch bfloat16), a bit-mask definition of
truncation, and the SPEC invariants (idempotence, monotonicity, error bound)."""
import math

import numpy as np
import pytest
import torch

import oracle
from tests import golden

RNG = np.random.default_rng(1234)


def _wide_doubles(count):
    """Doubles spanning +-[2^-160, 2^140] (FP32/FP16 subnormal + overflow ranges) plus ties."""
    e = RNG.uniform(-160, 140, size=count)
    x = np.exp2(e) * RNG.choice([-1.0, 1.0], size=count)
    return x


@pytest.mark.parametrize("name", [k for k, v in golden.load().items() if v["kind"] in ("qm", "qmrtz")])
def test_golden_quantize(name):
    g = golden.load()[name]
    i = g["inputs"]
    y = oracle.qm([float(i["x"])], int(i["E"]), int(i["m"]), rtz=g["kind"] == "qmrtz")[0]
    assert y == g["expected"] or (math.isinf(y) and math.isinf(g["expected"])), g["cite"]


def test_negative_zero_and_nan():
    y = oracle.qm([-0.0, np.nan, np.inf, -np.inf], 8, 7)
    assert y[0] == 0.0 and math.copysign(1.0, y[0]) < 0
    assert math.isnan(y[1]) and y[2] == np.inf and y[3] == -np.inf


def test_half_matches_numpy_float16():
    # numpy converts float64 -> float16 directly with round-to-nearest-even (single rounding).
    x = np.concatenate([_wide_doubles(200_000),
                        RNG.uniform(-70000, 70000, 50_000),
                        RNG.uniform(-1e-4, 1e-4, 50_000)])
    ref = x.astype(np.float16).astype(np.float64)
    got = oracle.qm(x, 5, 10)
    assert np.array_equal(got, ref)


def test_all_finite_binary16_patterns_are_fixed_points():
    # the 63488 finite binary16 patterns round-trip exactly.
    bits = np.arange(0, 1 << 16, dtype=np.uint16)
    h = bits.view(np.float16)
    h = h[np.isfinite(h)]
    assert h.size == 63488
    x = h.astype(np.float64)
    got = oracle.qm(x, 5, 10)
    assert np.array_equal(got.view(np.uint64), x.view(np.uint64))  # also keeps -0


def test_half_ties_midpoints():
    # exact midpoints between consecutive binary16 values must round to the even neighbour
    h = np.arange(0x0001, 0x7BFF, 37, dtype=np.uint16).view(np.float16).astype(np.float64)
    nxt = (np.arange(0x0001, 0x7BFF, 37, dtype=np.uint16) + 1).view(np.float16).astype(np.float64)
    mid = (h + nxt) / 2
    ref = mid.astype(np.float16).astype(np.float64)
    assert np.array_equal(oracle.qm(mid, 5, 10), ref)


def test_single_matches_numpy_float32():
    x = np.concatenate([_wide_doubles(200_000), RNG.standard_normal(50_000)])
    ref = x.astype(np.float32).astype(np.float64)
    assert np.array_equal(oracle.qm(x, 8, 23), ref)


def test_bf16_matches_torch_from_float32():
    # torch converts float32 -> bfloat16 with round-to-nearest-even; our q_m from the (exact)
    # float32 value must agree, including subnormals and overflow.
    x32 = np.concatenate([_wide_doubles(200_000).astype(np.float32),
                          RNG.standard_normal(50_000).astype(np.float32)])
    x32 = x32[np.isfinite(x32)]
    ref = torch.from_numpy(x32).to(torch.bfloat16).to(torch.float64).numpy()
    got = oracle.qm(x32.astype(np.float64), 8, 7)
    assert np.array_equal(got, ref)


def test_tf32_equals_half_inside_half_normal_range():
    # e8m10 and e5m10 have the same grid on [2^-14, 65504]: reduces to numpy float16 there.
    x = np.exp2(RNG.uniform(-14, 15.99, 100_000)) * RNG.choice([-1.0, 1.0], 100_000)
    ref = x.astype(np.float16).astype(np.float64)
    assert np.array_equal(oracle.qm(x, 8, 10), ref)


@pytest.mark.parametrize("m", [0, 3, 7, 10, 23, 40, 51])
def test_rtz_e11_is_bit_truncation(m):
    # For normal doubles, RTZ to m bits in an e11 container = clear the low 52-m mantissa bits.
    x = RNG.standard_normal(50_000) * np.exp2(RNG.uniform(-300, 300, 50_000))
    mask = np.uint64(~((1 << (52 - m)) - 1) & 0xFFFFFFFFFFFFFFFF)
    ref = (x.view(np.uint64) & mask).view(np.float64)
    assert np.array_equal(oracle.qm(x, 11, m, rtz=True), ref)


@pytest.mark.parametrize("E,m", [(8, 7), (8, 10), (5, 10), (11, 16), (11, 23), (8, 2)])
def test_spec_invariants(E, m):
    x = np.sort(_wide_doubles(50_000))
    y = oracle.qm(x, E, m)
    assert np.array_equal(oracle.qm(y, E, m), y)                # idempotent
    yy = y[np.isfinite(y)]
    assert np.all(np.diff(y[np.isfinite(y)]) >= 0) or yy.size < 2  # monotone
    bias = (1 << (E - 1)) - 1
    fin = np.isfinite(y) & (np.abs(x) >= 2.0 ** (1 - bias)) & (np.abs(x) < 2.0 ** bias)
    bound = np.exp2(-m - 1) * np.exp2(np.floor(np.log2(np.abs(x[fin]))))
    assert np.all(np.abs(y[fin] - x[fin]) <= bound)             # error bound


def test_double_is_identity():
    x = np.concatenate([_wide_doubles(10_000), RNG.standard_normal(10_000) * 1e-310])
    assert np.array_equal(oracle.qm(x, 11, 52), x)


def test_formats():
    assert oracle.prec_format(oracle.BF16) == (8, 7)
    assert oracle.prec_format(oracle.FP16) == (5, 10)
    assert oracle.prec_format(oracle.TF32) == (8, 10)
    assert oracle.prec_format(oracle.FP64) == (11, 52)
    assert oracle.container_E(oracle.BF16) == 8 and oracle.container_E(oracle.FP64) == 11


def test_fp16_sigma():
    assert oracle.fp16_sigma(1.0) == 14
    assert oracle.fp16_sigma(65504.0) == -1
    assert oracle.fp16_sigma(0.0) == 0 and oracle.fp16_sigma(np.inf) == 0
    for mx in [1e-9, 3e-5, 0.7, 123.0, 4e7]:
        s = oracle.fp16_sigma(mx)
        assert 2.0 ** 14 <= mx * 2.0 ** s < 2.0 ** 15


# ---- NEXT-3: FP8 (E4M3) and INT8 fixed-point operand formats ---------------------------------
def test_fp8_e4m3_grid_matches_torch_float8():
    torch = pytest.importorskip("torch")
    # every finite E4M3fn value below 2^7 is a fixed point of q_m(E=4, m=3) (the scaled operand range)
    allv = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    fin = allv[np.isfinite(allv) & (np.abs(allv) < 128)]
    assert fin.size > 200
    np.testing.assert_array_equal(oracle.qm(fin, 4, 3), fin)
    # RNE from float32 inputs (exact in float64, so torch's float -> fp8 path is one rounding)
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(200_000) * np.exp(rng.uniform(-12, 4, 200_000))).astype(np.float32)
    x = x[np.abs(x) < 127]
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    np.testing.assert_array_equal(oracle.qm(x.astype(np.float64), 4, 3), ref)


def test_scaled_format_sigmas():
    for prec in (oracle.FP8, oracle.INT8):
        for mx in (1e-5, 0.3, 1.0, 1.999, 77.0):
            s = oracle.sigma(prec, mx)
            assert 64 <= mx * 2.0 ** s < 128
    assert oracle.sigma(oracle.BF16, 3.0) == 0 and oracle.sigma(oracle.FP8, 0.0) == 0


def test_int8_fixed_point_quantiser():
    assert [oracle.q_int8(v) for v in (2.5, 3.5, -2.5, 0.49, 126.6, 127.5, 300.0, -500.0)] == \
        [2.0, 4.0, -2.0, 0.0, 127.0, 127.0, 127.0, -127.0]


@pytest.mark.parametrize("prec", [oracle.FP8, oracle.INT8])
def test_scaled_step_close_to_fp64(prec):
    import synth
    A = synth.spd(64, 2.0, 0)
    C0 = oracle.c0(A, np.prod(oracle.norms(A)[:2]), oracle.phase())
    _, c64, _ = oracle.step(A, C0, 2, oracle.phase())
    _, c8, _ = oracle.step(A, C0, 2, oracle.phase(prec))
    # operand rounding 2^-4 (FP8) / fixed point with 7 bits below the max (INT8), stored m bits
    assert np.linalg.norm(c8 - c64) / np.linalg.norm(c64) < 0.2
    _, s8, _ = oracle.step_sym(A, C0, 2, oracle.phase(prec))
    _, s64, _ = oracle.step_sym(A, C0, 2, oracle.phase())
    assert np.linalg.norm(s8 - s64) / np.linalg.norm(s64) < 0.2
