import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1703_02283_b200 as ipr, synth, bench
for n in [2048, 4096, 8192]:
    A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
    C = torch.linalg.inv(A); C = (C + C.T) / 2
    Zd = torch.empty_like(A); Zc = torch.empty_like(A); Zo = torch.empty_like(A)
    Ct = C.T.contiguous()
    ipr.ipr_test_gemm(ipr.IPR_FP64, n, A, Ct, Zd)
    ipr.ipr_test_gemm(ipr.IPR_FP64_CRT, n, A, Ct, Zc)
    ipr.ipr_test_gemm(ipr.IPR_FP64_OZ, n, A, Ct, Zo)
    print(n, "crt-dmma", float((Zc - Zd).abs().max()), "oz-dmma", float((Zo - Zd).abs().max()), flush=True)
for sched in ["symtri:bf16>fp64crt/cbf16", "symtri:bf16>fp64crt@a/cbf16"]:
    n = 8192
    A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
    form, ph = bench.schedule(sched, n)
    s = ipr.Solver(A, 2, ph, 1e-12, torch.cuda.current_stream(), form=form)
    s.iterate(45)
    for t in s.trace():
        print(sched, t["k"], t["phase"], t["prec"], t["mant_bits"], t["digits"], t["moduli"], "%.3e" % t["rho"], t["decision"], "%.2f" % t["gemm_ms"], flush=True)
    s.close()
