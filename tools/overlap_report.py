"""Paper-shaped overlap workloads through the C-ABI on one GPU.

For each preset N in synth.OVERLAP_PRESETS (N = 768 ... 6144, 25 % ... 3.1 %
non-zeros) at its natural condition number and as a kappa = 2 twin, runs a set of schedules and
reports outcome, iterations per phase, min in-chain rho, certified rho and time.
  python tools/overlap_report.py [--sizes 768,1536] [--out profiles/r01b_overlap.json]"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RUNS = [  # (label, p, schedule, final_tol)
    ("p1 ns:fp64", 1, "ns:fp64", 1e-9),
    ("p1 ns:bf16>fp64", 1, "ns:bf16>fp64", 1e-9),
    ("p2 fp64 (Eq. 1)", 2, "fp64", 1e-12),
    ("p2 symtri:fp64/cbf16", 2, "symtri:fp64/cbf16", 1e-12),
    ("p2 symtri:bf16>fp64/cbf16", 2, "symtri:bf16>fp64/cbf16", 1e-12),
    ("p2 symtri:bf16>fp64oz@a/cbf16", 2, "symtri:bf16>fp64oz@a/cbf16", 1e-12),
    ("p2 symtri:bf16>fp64crt@a/cbf16", 2, "symtri:bf16>fp64crt@a/cbf16", 1e-12),
    ("p2 cpl:fp64 (to 1e-6)", 2, "cpl:fp64", 1e-6),
    ("p2 symtri:fp8/cfp8>bf16>fp64crt@a/cbf16 [crt cert]", 2, "symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", 1e-12),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="768,1536,3072,6144")
    ap.add_argument("--out", default=None)
    ap.add_argument("--runs", default="", help="comma-separated substrings of the run labels to keep")
    a = ap.parse_args()
    import torch
    import bench
    import paper_1703_02283_b200 as ipr
    import synth
    res = []
    for n in [int(x) for x in a.sizes.split(",")]:
        for kappa in (None, 2.0):
            t0 = time.perf_counter()
            S, info = synth.overlap(n, seed=0, kappa=kappa, return_info=True)
            gen_s = time.perf_counter() - t0
            A = torch.from_numpy(S).cuda()
            ev = torch.linalg.eigvalsh(A)
            kap = float(ev[-1] / ev[0])
            for label, p, sched, tol in RUNS:
                if a.runs and not any(k in label for k in a.runs.split(",")):
                    continue
                cert_mode = "crt" if "[crt cert]" in label else "fp64"
                form, ph = bench.schedule(sched, n)
                st = torch.cuda.current_stream()
                for rep in range(2):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    s = ipr.Solver(A, p, ph, tol, st, form=form, cert=cert_mode)
                    s.iterate(300)
                    tr = s.trace()
                    cert = s.residual(1)
                    oc = ipr.OUTCOME_NAMES[s.outcome]
                    s.close()
                    e1.record(st)
                    torch.cuda.synchronize()
                rho = [t["rho"] for t in tr if math.isfinite(t["rho"])]
                row = {"n": n, "density": info["density"], "kappa": kap, "shift_mu": info.get("mu", 0.0),
                       "run": label, "p": p, "final_tol": tol, "outcome": oc,
                       "iters_per_phase": [sum(1 for t in tr if t["phase"] == i) for i in range(len(ph))],
                       "min_rho": min(rho) if rho else None, "certified_rho_best": cert,
                       "time_s": e0.elapsed_time(e1) / 1e3, "gen_s": gen_s}
                print(json.dumps(row), flush=True)
                res.append(row)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
