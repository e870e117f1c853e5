"""Probe (harness only): is the FP64 DMMA product C*C of a bitwise-symmetric C bitwise symmetric?
If so, a full column panel of Y = C*C equals the mirror of the upper-triangle tiles, so the tri
certificate at G = 1 and the full-panel one at G > 1 give the same bits (P11)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1703_02283_b200 as ipr
for n in (300, 1000, 2304, 4096):
    g = torch.Generator().manual_seed(n)
    X = torch.randn(n, n, generator=g, dtype=torch.float64)
    C = ((X + X.T) / 2).cuda()
    Z = torch.empty(n, n, dtype=torch.float64, device='cuda')
    ipr.ipr_test_gemm(ipr.IPR_FP64, n, C, C, Z)
    torch.cuda.synchronize()
    d = (Z != Z.T).sum().item()
    print(f"n={n}: asymmetric elements {d} of {n*n}", flush=True)
