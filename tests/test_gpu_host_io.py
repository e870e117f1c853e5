"""Host buffers at the C-ABI boundary (include/ipr.h: ipr_init's A, ipr_set_output / ipr_finalize's C in
host memory) -- the e2e path bench.py times.  The answer must be the device path's answer bit for bit,
whether it streamed to the host during its certificate (ipr_set_output, G = 1, FP64-range candidate)
or was copied by ipr_finalize; a candidate that missed its certificate must not leak into the result."""
import numpy as np
import pytest

import synth
from tests.gpu_util import torch_cuda

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

LOW = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)


def _phases(name):
    if name == "headline":
        return [ipr.make_phase("fp8", corr_prec="fp8", **LOW), ipr.make_phase("bf16", **LOW),
                ipr.make_phase("fp64crt", mant_bits=ipr.IPR_MANT_ADAPTIVE, corr_prec="bf16")]
    if name == "bf16>fp64":
        return [ipr.make_phase("bf16", **LOW), ipr.make_phase("fp64", corr_prec="bf16")]
    return [ipr.make_phase("fp64")]


def _solve(A, p, name, form, out=None, early=False, max_iters=200, tol=1e-12):
    s = ipr.Solver(A, p, _phases(name), tol, form=form)
    if early:
        s.set_output(out)
    s.iterate(max_iters)
    tr, outcome = s.trace(), s.outcome
    res = s.finalize(out)
    torch.cuda.synchronize()
    return (res.numpy() if not res.is_cuda else res.cpu().numpy()), tr, outcome


@pytest.mark.parametrize("n,name,form", [(520, "headline", "symmetric_tri"), (300, "bf16>fp64", "symmetric"),
                                         (300, "fp64", "literal")])
@pytest.mark.parametrize("early", [False, True])
def test_host_buffers_equal_device_path(n, name, form, early):
    A_np = synth.spd(n, 2.0, 31)
    ref, tr_d, out_d = _solve(torch_cuda(A_np), 2, name, form)
    A_h = torch.from_numpy(A_np).pin_memory()
    C_h = torch.full((n, n), np.nan, dtype=torch.float64).pin_memory()
    got, tr_h, out_h = _solve(A_h, 2, name, form, C_h, early)
    assert out_h == out_d == ipr.IPR_CONVERGED
    assert len(tr_h) == len(tr_d)
    np.testing.assert_array_equal(got, ref)
    np.testing.assert_array_equal(C_h.numpy(), ref)


def test_pageable_host_and_padded_ldc():
    n = 300
    A_np = synth.spd(n, 2.0, 32)
    ref, _, _ = _solve(torch_cuda(A_np), 2, "bf16>fp64", "symmetric")
    wide = np.full((n, n + 17), 7.0)
    wide[:, :n] = A_np
    A_h = torch.from_numpy(wide)[:, :n]                  # pageable, lda = n + 17
    C_h = torch.full((n, n + 5), -1.0, dtype=torch.float64)
    got, _, out = _solve(A_h, 2, "bf16>fp64", "symmetric", C_h[:, :n], early=True)
    assert out == ipr.IPR_CONVERGED
    np.testing.assert_array_equal(C_h[:, :n].numpy(), ref)
    assert np.all(C_h[:, n:].numpy() == -1.0)            # the copy respects ldc


def test_missed_candidate_does_not_leak():
    # a tolerance between the in-chain floor (~3e-15) and the FP64 certificate's (~2.4e-14) at n = 300:
    # every certificate misses (each streamed candidate is superseded), the run stops at its budget, and
    # finalize must return the best iterate, not the last streamed candidate
    n = 300
    A_np = synth.spd(n, 2.0, 33)
    ref, tr_d, out_d = _solve(torch_cuda(A_np), 2, "bf16>fp64", "symmetric", max_iters=30, tol=1e-14)
    C_h = torch.full((n, n), np.nan, dtype=torch.float64).pin_memory()
    got, tr_h, out_h = _solve(torch.from_numpy(A_np).pin_memory(), 2, "bf16>fp64", "symmetric", C_h, True,
                              max_iters=30, tol=1e-14)
    assert out_h == out_d == ipr.IPR_RUNNING
    assert any(t["rho_cert"] == t["rho_cert"] for t in tr_h)     # certificates ran (and missed)
    np.testing.assert_array_equal(got, ref)
