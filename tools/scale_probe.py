"""Scale invariance probe: the same SPD twin scaled by 2^sc through several schedules (the iteration is
scale-covariant in exact arithmetic: C(2^sc A) = 2^(-sc/p) C(A)).  python tools/scale_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1703_02283_b200 as ipr  # noqa: E402
import synth  # noqa: E402

n = 256
for sched in ["sym:fp64", "symtri:fp64crt@a", "sym:fp64crt@a", "symtri:fp64oz@a", bench.DEFAULT_SCHEDULE]:
    for sc in [0, 30, 100, 300]:
        A = torch.from_numpy(np.ldexp(synth.spd(n, 2.0, 9), sc)).cuda()
        form, ph = bench.schedule(sched, n)
        try:
            s = ipr.Solver(A, 2, ph, 1e-12, form=form)
            out = s.iterate(80)
            tr = s.trace()
            print(f"{sched:40s} 2^{sc:<4d} {ipr.OUTCOME_NAMES[out]:10s} {len(tr):3d} rho {tr[-1]['rho']:.2e} "
                  f"cert {tr[-1]['rho_cert']:.2e}", flush=True)
            s.close()
        except ipr.IprError as e:
            print(f"{sched:40s} 2^{sc:<4d} error {e}", flush=True)
