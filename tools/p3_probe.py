"""The C4 twin (n = 8192, p = 3) with a schedule, solved `reps` times in one process: per-phase device time
of the last solve.  python tools/p3_probe.py [schedule] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1703_02283_b200 as ipr  # noqa: E402
import synth  # noqa: E402

sched = sys.argv[1] if len(sys.argv) > 1 else "sym:fp8/cfp8>bf16>fp64crt@a/cbf16"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 8192
A, _ = synth.spd_torch(n, 2.0, synth.CONFIGS["C4"]["seed"], device="cuda")
form, ph = bench.schedule(sched, n)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = ipr.Solver(A, 3, ph, 1e-12, form=form, cert="crt")
    s.iterate(300)
    tr = s.trace()
    s.close()
    torch.cuda.synchronize()
    per = {}
    for t in tr:
        per.setdefault((t["phase"], t["prec"]), [0, 0.0])
        per[(t["phase"], t["prec"])][0] += 1
        per[(t["phase"], t["prec"])][1] += t["gemm_ms"]
    print(f"rep {r}: {time.perf_counter() - t0:.3f} s", {f"{k[1]}": (v[0], round(v[1], 1)) for k, v in per.items()},
          tr[-1]["rho_cert"], flush=True)
