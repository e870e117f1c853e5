"""One solve of a BASELINE workload through the C-ABI (harness tool for ncu captures).

  python tools/one_solve.py [--workload H_twin] [--schedule symtri:bf16>fp64/cbf16] [--cert crt|fp64]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H_twin")
    ap.add_argument("--schedule", default=None)
    ap.add_argument("--cert", default="crt")
    a = ap.parse_args()
    import torch
    import bench
    import paper_1703_02283_b200 as ipr
    import synth
    cfg = synth.CONFIGS[a.workload]
    n, p = cfg["n"], cfg["p"]
    A, _ = synth.spd_torch(n, cfg["kappa"], cfg["seed"], device="cuda")
    form, ph = bench.schedule(a.schedule or bench.DEFAULT_SCHEDULE, n)
    s = ipr.Solver(A, p, ph, 1e-12, torch.cuda.current_stream(), form=form, cert=a.cert)
    s.iterate(400)
    tr = s.trace()
    out = s.finalize()
    torch.cuda.synchronize()
    print(f"{ipr.OUTCOME_NAMES[s.outcome]} records={len(tr)} rho_cert={tr[-1]['rho_cert']:.3e} "
          f"norm={float(out.norm()):.6e}")


if __name__ == "__main__":
    main()
