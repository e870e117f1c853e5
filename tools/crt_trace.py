"""The headline's FP64-range (CRT) records: digits S, bits, moduli and residuals per chain -- the R-26 rule's
inputs and outputs at n = 8192.  python tools/crt_trace.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1703_02283_b200 as ipr  # noqa: E402
import synth  # noqa: E402

n = 8192
A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
form, ph = bench.schedule(bench.DEFAULT_SCHEDULE, n)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2     # the last solve is printed (the first pays the lazy setup)
for _ in range(reps):
    s = ipr.Solver(A, 2, ph, 1e-12, form=form, cert="crt")
    s.iterate(400)
    if _ < reps - 1:
        s.close()
for t in s.trace():
    print(json.dumps({k: t[k] for k in ("k", "phase", "prec", "rho", "digits", "moduli", "mant_bits", "gemm_ms",
                                         "upd_ms", "kern_ms", "rho_cert")}))
s.close()
