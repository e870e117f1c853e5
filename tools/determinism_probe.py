"""Run-to-run determinism of a schedule at full size: the same solve repeated in one process; prints whether
every trace record (rho, delta, rho_cert) is bit-identical.  python tools/determinism_probe.py [schedule] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1703_02283_b200 as ipr  # noqa: E402
import synth  # noqa: E402

sched = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_SCHEDULE
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
form, ph = bench.schedule(sched, n)
ref = None
for r in range(reps):
    s = ipr.Solver(A, 2, ph, 1e-12, form=form, cert=bench.auto_cert(sched, 2))
    s.iterate(400)
    tr = s.trace()
    C = s.finalize()
    key = [(t["rho"], t["delta"], t["rho_cert"]) for t in tr]
    if ref is None:
        ref, Cref = key, C.clone()
        print("rep 0:", len(tr), "records, last", tr[-1]["rho_cert"], flush=True)
        continue
    same = all((a == b) or (a != a and b != b) for x, y in zip(key, ref) for a, b in zip(x, y)) and len(key) == len(ref)
    first = next((k for k, (x, y) in enumerate(zip(key, ref)) if any(not ((a == b) or (a != a and b != b)) for a, b in zip(x, y))), None)
    print(f"rep {r}: identical={same and torch.equal(C, Cref)} first differing record={first}", flush=True)
