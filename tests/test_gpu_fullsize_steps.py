"""Full-size step parity of the headline's own phases (VERDICT r01 "Next round" 2), in the bench's
launch configuration (n = 8192, the symmetric-tri form with its multi-band tile order) and at
n = 2304 (two 2048-wide tri bands plus a ragged tail band).

One step C_k -> C_{k+1} of the symmetrised-correction form (R-22; Eq. (1) as
the Newton correction) is checked stage by stage on sampled elements the oracle computes one by one
from the previous stage's values (ipr_test_peek exposes each stage's stored operand):

  Z_1 = Ahat Chat            sampled columns:  Ahat Chat[:, j] (oracle matvec), then the operand rounding
                             (below the FP64 range: the mirror of its upper triangle, R-36)
  Z_2 = Chat qin(Z_1) (tri)  sampled (i, j) over every band, both triangles:
                             Rhat_ij = qc(delta_ij - Chat[min(i,j), :] . qin(Z_1)[:, max(i,j)]) -- the
                             mirror of the upper triangle (R-22 tri reading), and Rhat exactly symmetric
  W = qc(C) Rhat             sampled (i, j): qc(C)[i, :] . Rhat[:, j]
  C_{k+1} = q_m(C_k + (W + W^T) / 4)   EVERY element, bit for bit (the FP64 epilogue is deterministic);
                             below the FP64 range the tri form's S_ij = 2 W_{min(i,j), max(i,j)} (R-36)

Bounds: FP32 accumulation n 2^-24 sum |terms| (tensor cores: FP8 / BF16), the CRT quantisation
2^-b (row max . column abs-sum + row abs-sum . column max) (R-28), the operand rounding u of the
stored format (plus the E4M3 subnormal quantum for FP8).  Phases: FP8 with the FP8 correction (R-29),
BF16, and the FP64-range CRT phase at S = 9 (b = 59) and at a low S (m = 23 -> S = 5, b = 31)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

U = {"fp8": 2.0 ** -4, "bf16": 2.0 ** -8, "tf32": 2.0 ** -11, "fp64": 2.0 ** -53, "fp64crt": 2.0 ** -53}
ACC = {"fp8": 2.0 ** -24, "bf16": 2.0 ** -24, "tf32": 2.0 ** -24}

CASES = [
    # (id, schedule, steps before the checked step, phase index of the checked step)
    ("fp8_cfp8", "symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", 5, 0),
    ("bf16", "symtri:bf16>fp64crt@a/cbf16", 6, 0),
    ("crt_S9", "symtri:fp64crt/cbf16", 4, 0),
    ("crt_S5", "symtri:fp64crt@23/cbf16", 4, 0),
]


@pytest.fixture(scope="module", params=[8192, 2304])
def mat(request):
    n = request.param
    A, _ = synth.spd_torch(n, 2.0, 5 if n == 8192 else 21, device="cuda")
    return A, A.cpu().numpy()


def _peek(s, what, npad, n):
    return ipr.ipr_test_peek(s.ctx, what, npad).cpu().numpy()


def _samples(n, rng, k=1500):
    """(i, j) pairs: random over the matrix + band / tile boundaries and the diagonal."""
    edges = sorted({0, 1, 127, 128, 255, 256, 2047, 2048, 2049, 4095, 4096, n // 2, n - 257, n - 256, n - 2, n - 1})
    edges = [e for e in edges if 0 <= e < n]
    I = list(rng.integers(0, n, k)) + [a for a in edges for _ in edges]
    J = list(rng.integers(0, n, k)) + [b for _ in edges for b in edges]
    return np.array(I), np.array(J)


def _run_to_step(A, sched, k_before):
    import bench
    n = A.shape[0]
    form, ph = bench.schedule(sched, n)
    s = ipr.Solver(A, 2, ph, 1e-12, form=form)
    if k_before:
        assert s.iterate(k_before) == ipr.IPR_RUNNING
    Ck = s.iterate_copy(0).cpu().numpy()
    assert s.iterate(1) == ipr.IPR_RUNNING
    rec = s.trace()[-1]
    assert rec["decision"] == ipr.IPR_DEC_CONTINUE, rec
    Ck1 = s.iterate_copy(0).cpu().numpy()
    return s, ph, rec, Ck, Ck1


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_headline_phase_step_full_size(mat, case):
    A, A_np = mat
    n = A_np.shape[0]
    cid, sched, k_before, phase_idx = case
    s, ph, rec, Ck, Ck1 = _run_to_step(A, sched, k_before)
    try:
        assert rec["phase"] == phase_idx
        prec = ipr.PREC_NAMES[ph[phase_idx].prec]
        corr = ipr.PREC_NAMES[ph[phase_idx].corr_prec] if ph[phase_idx].corr_prec >= 0 else prec
        npad = (n + 255) // 256 * 256
        Ahat = _peek(s, ipr.IPR_PEEK_AHAT, npad, n)[:n, :n].T          # K-major -> (k, j)
        Chat = _peek(s, ipr.IPR_PEEK_CHAT, npad, n)[:n, :n]
        Z1 = _peek(s, ipr.IPR_PEEK_Z1, npad, n)[:n, :n].T
        Rhat = _peek(s, ipr.IPR_PEEK_RHAT, npad, n)[:n, :n].T
        W = _peek(s, ipr.IPR_PEEK_W, npad, n)[:n, :n]
        Chc = _peek(s, ipr.IPR_PEEK_CHATC, npad, n)[:n, :n]
    finally:
        s.close()
    rng = np.random.default_rng(n + len(cid))
    crt = prec == "fp64crt"
    b = oracle.crt_bits(rec["digits"], n) if crt else None

    # the operands are the phase's roundings of A and C_k (exact symmetry kept)
    assert np.array_equal(Ahat, Ahat.T) and np.array_equal(Chat, Chat.T)
    if crt:
        np.testing.assert_array_equal(Chat, Ck)

    def crt_q(X, Y, rows, cols):
        """the CRT product's quantisation error scale 2^-b (rmax_i colsum_j + rowsum_i cmax_j) (R-28)"""
        aX, aY = np.abs(X), np.abs(Y)
        return 2.0 ** -b * (aX.max(axis=1)[rows] * aY.sum(axis=0)[cols] + aX.sum(axis=1)[rows] * aY.max(axis=0)[cols])

    def prod_bound(X, Y, rows, cols):
        """|computed - exact| bound of (X Y)[rows, cols] for an FP32-accumulated product."""
        return n * ACC[prec] * (np.abs(X[rows]) @ np.abs(Y[:, cols]))

    # ---- stage 1: qin(Z_1) = qin(Ahat Chat), sampled columns ----
    cols = np.unique(np.concatenate([rng.integers(0, n, 6), [0, n - 1, min(2048, n - 1)]]))
    if crt:
        # the oracle's exact CRT product (R-28 definition) element by element.  The GPU's sliced-FP64
        # reconstruction has an absolute error far below the method's own quantisation error
        # q_ij = 2^-b (rmax_i colsum_j + rowsum_i cmax_j) (measured <= 0.06 q, tools/crt_rec_diag.py) but
        # up to ~100 ulp of the tiny off-diagonal elements: bound 2 ulp + q / 8, and >= 99 % bit-equal
        K, J = np.meshgrid(np.arange(n), cols, indexing="ij")
        ref = oracle.gemm_crt_pairs(Ahat, Chat, b, K.ravel(), J.ravel()).reshape(n, len(cols))
        q = crt_q(Ahat, Chat, np.arange(n)[:, None], cols[None, :])
        d = np.abs(Z1[:, cols] - ref)
        lim = 2 * np.spacing(np.abs(ref)) + q / 8
        assert np.all(d <= lim), (cid, "Z1", float(np.max(d / lim)))
        assert np.mean(d == 0) >= 0.99
    else:
        ref = Ahat @ Chat[:, cols]
        bnd = prod_bound(Ahat, Chat, np.arange(n), cols)
        # R-36: below the FP64 range Z_1 is the mirror of its upper triangle -- rows below the diagonal of
        # column j hold (Ahat Chat)[j, i]; Z_1 exactly symmetric
        assert np.array_equal(Z1, Z1.T)
        lower = np.arange(n)[:, None] > cols[None, :]
        ref = np.where(lower, (Ahat[cols] @ Chat).T, ref)
        bnd = np.where(lower, prod_bound(Ahat, Chat, cols, np.arange(n)).T, bnd)
        u_op = U[prec]
        sub = 2.0 ** -16 * np.abs(Z1).max() if prec == "fp8" else 0.0   # E4M3 subnormal quantum (scaled max 2^6)
        err = np.abs(Z1[:, cols] - ref)
        lim = u_op * np.abs(ref) + (1 + u_op) * bnd + sub + 1e-300
        assert np.all(err <= lim), (cid, "Z1", float(np.max(err / lim)))

    # ---- stage 2: Rhat = qc(I - Z_2), Z_2 = Chat qin(Z_1) upper triangle mirrored ----
    assert np.array_equal(Rhat, Rhat.T), "tri R must be exactly symmetric"
    I, J = _samples(n, rng)
    lo, hi = np.minimum(I, J), np.maximum(I, J)
    if crt:   # Z_2[min, max] by the oracle's exact CRT product of Chat and the GPU's qin(Z_1)
        z2 = oracle.gemm_crt_pairs(Chat, Z1, b, lo, hi)
        b2 = 2 * np.spacing(np.abs(z2)) + crt_q(Chat, Z1, lo, hi) / 8
    else:     # FP64 dot of the stored operands; the GPU accumulates in FP32
        z2 = np.einsum("ij,ij->i", Chat[lo], Z1[:, hi].T)
        b2 = n * ACC[prec] * np.einsum("ij,ij->i", np.abs(Chat[lo]), np.abs(Z1[:, hi].T))
    r_ref = (I == J).astype(np.float64) - z2
    u_c = U[corr] + 2.0 ** -23          # the correction format's rounding (+ an FP32 intermediate)
    sub_r = 2.0 ** -16 * np.abs(Rhat).max() if corr == "fp8" else 0.0
    err = np.abs(Rhat[I, J] - r_ref)
    lim = u_c * np.abs(r_ref) + (1 + u_c) * b2 + sub_r + 1e-300
    assert np.all(err <= lim), (cid, "R", float(np.max(err / lim)))
    # not vacuous: on the diagonal (R_ii = 1 - t_i, O(1) this early) the bound is a fraction of R
    dg = I == J
    assert np.all(lim[dg] < 0.2 * np.abs(r_ref[dg]))

    # ---- stage 3: W = qc(C_k) Rhat (FP32 accumulate; FP8 correction: scaled operands, exact unscale) ----
    # (reading R-36: every CASE is the symmetric-tri form; below the FP64 range only W's upper triangle is
    # computed, so the sampled pairs are taken as (min, max) there)
    triw = prec not in ("fp64", "fp64crt", "fp64oz")
    I3, J3 = I[:400], J[:400]
    if triw:
        I3, J3 = np.minimum(I3, J3), np.maximum(I3, J3)
    w_ref = np.einsum("ij,ij->i", Chc[I3], Rhat[:, J3].T)
    acc_c = 2.0 ** -53 if corr == "fp64" else 2.0 ** -24
    b3 = n * acc_c * np.einsum("ij,ij->i", np.abs(Chc[I3]), np.abs(Rhat[:, J3].T)) + 2.0 ** -24 * np.abs(w_ref)
    assert np.all(np.abs(W[I3, J3] - w_ref) <= b3 + 1e-300), (cid, "W")

    # ---- stage 4: the FP64 epilogue C_{k+1} = q_m(C_k + (W_ij + W_ji) / 4), every element, bit for bit ----
    E = 11 if prec in ("fp64", "fp64crt") else 8
    m = {"fp8": 3, "bf16": 7}.get(prec, None)
    if m is None:
        m = int(ph[phase_idx].mant_bits) if ph[phase_idx].mant_bits >= 0 else 52
    if triw:                                  # S_ij = 2 W_{min(i,j), max(i,j)} (R-36)
        Wu = np.triu(W)
        e = 2.0 * (Wu + np.triu(W, 1).T) / 4.0
    else:
        e = (W + W.T) / 4.0
    C1_ref = oracle.qm(Ck + e, E, m)
    np.testing.assert_array_equal(Ck1, C1_ref)
