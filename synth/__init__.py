"""Seeded synthetic inputs shared by the oracle side and the CUDA side of every test/bench.

This module holds NONE of the method's arithmetic (no norms, no iteration, no rounding to
reduced formats): it only builds input matrices and probe vectors.

The paper's own workload -- overlap matrices of 128..1024 H2O molecules, N = 768 ... 6144,
25 % ... 3.1 % non-zeros in [-1, 1] (Sec. 4.1) -- is not public and not in
this container.  BASELINE.json's synthetic family stands in for it:

    A = Q diag(lambda) Q^T,  Q from QR of a seeded N(0,1) n x n matrix,
    lambda log-uniform in [1/kappa, 1]

with the readings R-13 (symmetrise exactly: A <- (A + A^T)/2), R-14 (pin lambda_0 = 1/kappa,
lambda_1 = 1 so cond(A) = kappa), R-15 (NumPy PCG64 default_rng(seed); Q's column signs flipped
so that diag(R) > 0).
"""
from __future__ import annotations

import numpy as np

# BASELINE.json configs (seed = config index) plus the headline and its kappa=2 "twin"
# (reading R-3: Eq. (1) cannot reach 1e-12 at the stated kappa).
CONFIGS = {
    "C1": dict(n=64, kappa=1e2, p=2, seed=0),
    "C2": dict(n=1024, kappa=1e3, p=1, seed=1),
    "C3": dict(n=4096, kappa=1e4, p=2, seed=2),
    "C4": dict(n=8192, kappa=1e4, p=3, seed=3),
    "C5": dict(n=32768, kappa=1e5, p=2, seed=4),
    "H": dict(n=8192, kappa=1e4, p=2, seed=5),
    "H_twin": dict(n=8192, kappa=2.0, p=2, seed=5),
}


def eigenvalues(n: int, kappa: float, rng: np.random.Generator) -> np.ndarray:
    """lambda_i log-uniform in [1/kappa, 1] with lambda_0 = 1/kappa, lambda_1 = 1 (R-14)."""
    lam = np.exp(rng.uniform(np.log(1.0 / kappa), 0.0, size=n))
    lam[0] = 1.0 / kappa
    if n > 1:
        lam[1] = 1.0
    return lam


def spd(n: int, kappa: float, seed: int, return_eig: bool = False):
    """BASELINE family on the CPU (NumPy, FP64).  Returns A (and lambda, Q if asked)."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    Q = Q * np.sign(np.diag(R))[None, :]
    lam = eigenvalues(n, kappa, rng)
    A = (Q * lam[None, :]) @ Q.T
    A = (A + A.T) * 0.5
    A = np.ascontiguousarray(A)
    if return_eig:
        return A, lam, Q
    return A


def spd_torch(n: int, kappa: float, seed: int, device="cuda"):
    """Same recipe generated with torch on the GPU (harness only, for n >= 8192 where a CPU
    QR takes minutes).  Returns (A, lambda) as FP64 torch tensors on `device`."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    G = torch.randn((n, n), generator=g, device=device, dtype=torch.float64)
    Q, R = torch.linalg.qr(G)
    Q = Q * torch.sign(torch.diagonal(R))[None, :]
    del G, R
    rng = np.random.default_rng(seed)
    lam = torch.from_numpy(eigenvalues(n, kappa, rng)).to(device)
    A = (Q * lam[None, :]) @ Q.T
    del Q
    A = (A + A.T) * 0.5
    return A.contiguous(), lam


def diag_spd(n: int, kappa: float, seed: int) -> np.ndarray:
    """Diagonal SPD with spectrum from `eigenvalues` (max diagonal 1, so the sufficient
    condition of reading R-12 holds for every p)."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(np.diag(rng.permutation(eigenvalues(n, kappa, rng))))


def probe_vectors(n: int, count: int, seed: int) -> np.ndarray:
    """Random +-1 vectors (Freivalds-style one-step probe): shape (count, n)."""
    rng = np.random.default_rng(10_000 + seed)
    return rng.choice(np.array([-1.0, 1.0]), size=(count, n))
