"""Host-side pins of the Ozaki scheme II constants (reading R-28), checked with exact
Python integers -- no GPU.  The CUDA reconstruction (gemm_tc.cu crt_chunk) relies on:
  * pairwise coprime moduli <= 256 (the CRT is then a bijection Z_M -> prod Z_{m_l});
  * inv_l W_l = 1 (mod m_l) with W_l = M_N / m_l (so sum_l ((u_l inv_l) mod m_l) W_l = u_l mod m_l);
  * W_l = H_l 2^s1 + L_l 2^s2 + R_l, M_N = MH 2^s1 + ML 2^s2 + MR with H, L the exact bit fields
    (small enough that sum_l (256 + v_l) H_l, v_l <= 255, and q MH, q <= the largest quotient, stay
    < 2^53)
    and R the low bits, exact below 2^53 and correctly rounded to FP64 above;
  * the modulus count for (b, n): the smallest N with M_N > 2^1.02 n 2^(2b) (|Pbar| <= n 2^(2b), so
    X / M_N is within 0.493 of an integer and rint(X / M_N), evaluated to ~2^-45, is exact)."""
import math
from fractions import Fraction

import pytest

ipr = pytest.importorskip("paper_1703_02283_b200")


NMAX = 18


def _tab(N, b=53, n=8192):
    return ipr.ipr_test_crt_table(N, b, n)


def test_moduli_pairwise_coprime_and_int8():
    m = _tab(NMAX)["moduli"]
    assert len(m) == NMAX and all(2 <= x <= 256 for x in m)
    for i in range(NMAX):
        for j in range(i + 1, NMAX):
            assert math.gcd(m[i], m[j]) == 1, (m[i], m[j])


def _check_slices(W, H, L, R, s1, s2):
    assert H == int(H) and L == int(L)
    assert int(H) == W >> s1 and int(L) == (W >> s2) & ((1 << (s1 - s2)) - 1)
    r = W & ((1 << s2) - 1)
    assert R == float(r)            # correctly rounded (exact below 2^53)


@pytest.mark.parametrize("N", range(1, NMAX + 1))
def test_weights_inverses_and_slices_exact(N):
    t = _tab(N)
    m = t["moduli"]
    M = math.prod(m)
    s1, s2 = (int(math.log2(x)) for x in t["p2s"])
    assert t["p2s"] == (2.0 ** s1, 2.0 ** s2)
    assert s1 == 0 or s1 - s2 == 39 or s2 == 0
    for l in range(N):
        W = M // m[l]
        H, L, R = t["HLR"][l]
        _check_slices(W, H, L, R, s1, s2)
        assert H < 2 ** 39 and L < 2 ** 39
        assert (t["inv"][l] * W) % m[l] == 1
        assert 0 <= t["inv"][l] < m[l]
    _check_slices(M, *t["M_HLR"], s1, s2)
    MH, ML = (int(x) for x in t["M_HLR"][:2])
    # exactness budget of the FP64 sums of the exact slice: the finish accumulates (256 + v_l) H_l
    assert 511 * sum(int(t["HLR"][l][0]) for l in range(N)) < 2 ** 53
    qmax = math.ceil(Fraction(sum(255 * (M // x) for x in m), M))
    assert qmax * MH < 2 ** 53 and qmax * ML < 2 ** 53


def test_crt_reconstruction_by_definition():
    # residues of integers |P| < M/4 -> the weighted sum and rint quotient give P back (exact ints)
    t = _tab(NMAX)
    m = t["moduli"]
    M = math.prod(m)
    rng = __import__("random").Random(7)
    for _ in range(200):
        P = rng.randrange(-M // 4 + 1, M // 4)
        v = [((P % ml) * t["inv"][l]) % ml for l, ml in enumerate(m)]
        X = sum(vl * (M // ml) for vl, ml in zip(v, m))
        q = round(Fraction(X, M))
        assert X - q * M == P


@pytest.mark.parametrize("b,n", [(62, 8192), (53, 65535), (21, 520), (35, 8192), (49, 1024), (2, 1)])
def test_modulus_count_is_minimal(b, n):
    nf = _tab(NMAX, b, n)["n_for"]
    m = _tab(NMAX)["moduli"]
    need = 2.0281 * n * 2 ** (2 * b)     # 2^1.02
    assert math.prod(m[:nf]) > need
    assert nf == 2 or math.prod(m[:nf - 1]) <= need * 1.01     # (log2 comparison with 1 % slack)


def test_digits_to_bits_and_fp64_range():
    # b = 7 S - 4 (the stored bits of the R-26 rule), capped at 62 and at what 18 moduli allow at n
    for S in range(2, 10):
        assert _tab(NMAX, S, 8192)["b_for"] == 7 * S - 4
    assert _tab(NMAX, 9, 65535)["b_for"] == 59
    assert _tab(NMAX, 59, 8192)["n_for"] == 17            # S = 9: 17 GEMMs, not 45 digit products
    assert _tab(NMAX, 62, 8192)["n_for"] == 18
    for S in range(4, 10):                                 # fewer GEMMs than scheme I from S = 4 on
        assert _tab(NMAX, 7 * S - 4, 8192)["n_for"] < S * (S + 1) // 2
    assert _tab(NMAX, 63, 8192)["n_for"] == -1            # beyond CRT_BMAX
