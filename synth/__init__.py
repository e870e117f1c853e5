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


# Paper-shaped overlap workloads: PAPER.md:178-185 (Sec. 4.1) -- an SPD
# overlap matrix of N = 786 (768 in Sec. 4.3.1) with 25 % non-zeros in [-1, 1], density 12.4 %,
# 6.2 %, 3.1 % at N = 1572 (1536), 3072, 6144 (nearsightedness).  The real H2O matrices are not
# available; `overlap` stands in for them.
OVERLAP_PRESETS = {768: 0.25, 1536: 0.124, 3072: 0.062, 6144: 0.031}


def _wendland(r: np.ndarray) -> np.ndarray:
    """Wendland's C2 function (1 - r)^4_+ (4 r + 1): compactly supported and positive definite
    in R^3, so a Gram-type matrix of it at distinct points is SPD with exact zeros beyond r = 1."""
    return np.where(r < 1.0, (1.0 - r) ** 4 * (4.0 * r + 1.0), 0.0)


def overlap(n: int, density: float | None = None, seed: int = 0, kappa: float | None = None,
            return_info: bool = False):
    """Overlap-like SPD matrix: n "basis functions" on a jittered cubic lattice (bounded minimum
    separation, like atoms), S_ij = s_i s_j phi(|x_i - x_j| / R) with phi the Wendland C2 kernel,
    random signs s (entries in [-1, 1]), unit diagonal, and the radius R bisected so the realised
    density of non-zeros matches `density` (default: the paper's preset for n, else 25 %).
    Natural condition numbers come out ~1e3.  kappa: optionally shift and rescale
    S <- (S + mu I) / (1 + mu) (unit diagonal kept) so that cond(S) = kappa exactly in exact
    arithmetic (the stable-regime twin of the workload)."""
    if density is None:
        density = OVERLAP_PRESETS.get(n, 0.25)
    if not 0.0 < density <= 1.0:
        raise ValueError("density must be in (0, 1]")
    rng = np.random.default_rng(seed)
    m = int(np.ceil(n ** (1.0 / 3.0) - 1e-9))
    g = np.stack(np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij"), -1).reshape(-1, 3)
    x = g[rng.permutation(len(g))[:n]].astype(np.float64) + rng.uniform(-0.3, 0.3, size=(n, 3))
    # pairwise distances, term by term: (a - b)^2 == (b - a)^2 bitwise, so r is exactly symmetric
    r = np.zeros((n, n))
    for k in range(3):
        d = x[:, k][:, None] - x[:, k][None, :]
        r += d * d
    np.sqrt(r, out=r)
    lo, hi = 1e-3, 3.0 * m
    for _ in range(64):
        R = 0.5 * (lo + hi)
        if np.count_nonzero(r < R) / float(n * n) > density:
            hi = R
        else:
            lo = R
    S = _wendland(r / R)
    del r
    sg = rng.choice(np.array([-1.0, 1.0]), size=n)
    S *= sg[:, None]
    S *= sg[None, :]
    S = (S + S.T) * 0.5
    info = {"R": R, "density": np.count_nonzero(S) / float(n * n)}
    if kappa is not None:
        ev = np.linalg.eigvalsh(S)
        lmin, lmax = float(ev[0]), float(ev[-1])
        mu = (lmax - kappa * lmin) / (kappa - 1.0)
        if mu > 0:
            S = (S + mu * np.eye(n)) / (1.0 + mu)
            S = (S + S.T) * 0.5
        info["mu"] = max(mu, 0.0)
    S = np.ascontiguousarray(S)
    return (S, info) if return_info else S


def probe_vectors(n: int, count: int, seed: int) -> np.ndarray:
    """Random +-1 vectors (Freivalds-style one-step probe): shape (count, n)."""
    rng = np.random.default_rng(10_000 + seed)
    return rng.choice(np.array([-1.0, 1.0]), size=(count, n))
