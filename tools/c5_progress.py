"""C5's kappa = 2 twin (n = 32768) one iteration at a time, printing each record as it lands (diagnose a
slow or stuck large solve).  python tools/c5_progress.py [schedule] [n] [tol] [cap] [cert]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1703_02283_b200 as ipr
import synth

sched = sys.argv[1] if len(sys.argv) > 1 else "symtri:bf16>fp64crt@a/cbf16"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 40
cert = sys.argv[5] if len(sys.argv) > 5 else "crt"
t0 = time.perf_counter()
A, _ = synth.spd_torch(n, 2.0, synth.CONFIGS["C5"]["seed"], device="cuda")
torch.cuda.synchronize()
print(f"A ready {time.perf_counter() - t0:.1f} s, free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
torch.cuda.empty_cache()
form, ph = bench.schedule(sched, n)
ph[-1].max_iters = cap
s = ipr.Solver(A, 2, ph, tol, form=form, cert=cert)
for k in range(200):
    t1 = time.perf_counter()
    out = s.iterate(1)
    tr = s.trace()
    r = tr[-1]
    print(json.dumps({"k": k, "wall_s": round(time.perf_counter() - t1, 3), "phase": r["phase"], "prec": r["prec"],
                      "rho": r["rho"], "cert": r["rho_cert"], "gemm_ms": r["gemm_ms"], "moduli": r["moduli"]}), flush=True)
    if out != ipr.IPR_RUNNING:
        break
print("outcome", ipr.OUTCOME_NAMES[s.outcome], f"total {time.perf_counter() - t0:.1f} s", flush=True)
if cert == "crt":
    print("certificate terms", json.dumps(ipr.ipr_test_cert_info(s.ctx)), flush=True)
print("certificate recheck of the best iterate", s.residual(1), flush=True)
print("dmma evaluation of the best iterate", s.residual(2), flush=True)
s.close()
