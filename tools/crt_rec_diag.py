"""Diagnostic: GPU CRT product (engine's Z_1 of a CRT step at full size) vs the oracle's exact CRT
definition -- where the reconstruction's absolute error sits relative to ulp and to the quantisation
error scale q_ij = 2^-b (rmax_i colsum_j + rowsum_i cmax_j)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import synth
import paper_1703_02283_b200 as ipr
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
form, ph = bench.schedule("symtri:fp64crt/cbf16", n)
s = ipr.Solver(A, 2, ph, 1e-12, form=form)
s.iterate(k)
s.iterate(1)
rec = s.trace()[-1]
npad = (n + 255) // 256 * 256
Ahat = ipr.ipr_test_peek(s.ctx, 0, npad).cpu().numpy()[:n, :n].T
Chat = ipr.ipr_test_peek(s.ctx, 1, npad).cpu().numpy()[:n, :n]
Z1 = ipr.ipr_test_peek(s.ctx, 2, npad).cpu().numpy()[:n, :n].T
s.close()
b = oracle.crt_bits(rec["digits"], n)
cols = np.array([0, 1, 17, n // 2, n - 1])
K, J = np.meshgrid(np.arange(n), cols, indexing="ij")
ref = oracle.gemm_crt_pairs(Ahat, Chat, b, K.ravel(), J.ravel()).reshape(n, len(cols))
d = np.abs(Z1[:, cols] - ref)
ulp = np.spacing(np.abs(ref))
rmax = np.abs(Ahat).max(axis=1)[:, None]
rsum = np.abs(Ahat).sum(axis=1)[:, None]
cmax = np.abs(Chat).max(axis=0)[cols][None, :]
csum = np.abs(Chat[:, cols]).sum(axis=0)[None, :]
q = 2.0 ** -b * (rmax * csum + rsum * cmax)
scale = rmax * cmax
print(f"n={n} k={k} b={b} digits={rec['digits']} frac_exact={np.mean(d == 0):.4f} max d/ulp={np.max(d / ulp):.1f} "
      f"max d/q={np.max(d / q):.3e} max d/(rmax cmax 2^-2b)={np.max(d / (scale * 2.0 ** (-2 * b))):.3e} "
      f"max d={d.max():.3e} cmax={cmax.ravel()} rmax range=({rmax.min():.3e},{rmax.max():.3e})")
i, j = np.unravel_index(np.argmax(d / ulp), d.shape)
print("worst", i, cols[j], Z1[i, cols[j]], ref[i, j], d[i, j], q[i, j])
