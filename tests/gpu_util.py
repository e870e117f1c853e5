"""Helpers for the -m gpu parity tests (CUDA path through the C-ABI vs the oracle)."""
import numpy as np


def torch_cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_gpu_trajectory(A_np, p, phases, final_tol, max_iters, keep=True, form="literal"):
    """Iterate one chain at a time through the C-ABI.  Returns (outcome, trace, hist, C_best)
    with hist[k] = the iterate evaluated by trace record k, for k >= 1 (same indexing as the
    oracle's C_hist)."""
    import torch
    import paper_1703_02283_b200 as ipr
    A = torch_cuda(A_np)
    s = ipr.Solver(A, p, phases, final_tol, form=form)
    hist = {}
    out = ipr.IPR_RUNNING
    for k in range(max_iters):
        out = s.iterate(1)
        if out != ipr.IPR_RUNNING:
            break
        if keep:
            hist[k + 1] = s.iterate_copy(0).cpu().numpy()
    tr = s.trace()
    best = s.finalize().cpu().numpy()
    torch.cuda.synchronize()
    return out, tr, hist, best


def gpu_c0(A_np, phase):
    """C_0 through the C-ABI: a schedule that converges at the first chain returns C_0."""
    import paper_1703_02283_b200 as ipr
    A = torch_cuda(A_np)
    s = ipr.Solver(A, 1, [phase], 1e300)
    assert s.iterate(1) == ipr.IPR_CONVERGED
    nrm = s.norms()
    return s.finalize().cpu().numpy(), nrm


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
