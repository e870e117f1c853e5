"""Per-record timings of named schedules at a BASELINE workload (harness tool, GPU).

  python tools/sched_probe.py [--workload H_twin] sched1 sched2 ...
Prints, per schedule, the wall time of one solve and every trace record (phase, prec, rho,
rho_cert, chain ms = gemm_ms - upd_ms, update ms).  Schedule syntax as bench.py --schedule."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H_twin")
    ap.add_argument("--json", default=None)
    ap.add_argument("--cert", default="auto", help="certificate: auto (bench's choice), crt, fp64")
    ap.add_argument("schedules", nargs="+")
    a = ap.parse_args()
    import torch
    import bench
    import paper_1703_02283_b200 as ipr
    import synth
    cfg = synth.CONFIGS[a.workload]
    n, p = cfg["n"], cfg["p"]
    A, _ = synth.spd_torch(n, cfg["kappa"], cfg["seed"], device="cuda")
    out = torch.empty_like(A)
    st = torch.cuda.current_stream()
    res = {}
    for name in a.schedules:
        form, ph = bench.schedule(name, n)
        import time
        for rep in range(3):      # first runs warm up (tensor maps, allocations)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            h0 = time.perf_counter()
            s = ipr.Solver(A, p, ph, 1e-12, st, form=form, cert=bench.auto_cert(name, p, a.cert))
            torch.cuda.synchronize()
            h1 = time.perf_counter()
            s.iterate(400)
            torch.cuda.synchronize()
            h2 = time.perf_counter()
            tr = s.trace()
            oc = s.outcome
            s.finalize(out)
            e1.record(st)
            torch.cuda.synchronize()
            h3 = time.perf_counter()
            t = e0.elapsed_time(e1)
            print(f"   rep {rep}: {t:.1f} ms (host: init {1e3 * (h1 - h0):.1f} iterate {1e3 * (h2 - h1):.1f} "
                  f"finalize {1e3 * (h3 - h2):.1f} ms)")
        print(f"== {name}: {t:.1f} ms, {ipr.OUTCOME_NAMES[oc]}, {len(tr)} records")
        for r in tr:
            print(f"  k={r['k']:3d} ph={r['phase']} {r['prec']:5s} rho={r['rho']:.3e} cert={r['rho_cert']:.2e} "
                  f"chain={r['gemm_ms'] - r['upd_ms']:8.2f} upd={r['upd_ms']:7.2f} dec={r['decision']}")
        res[name] = {"ms": t, "outcome": ipr.OUTCOME_NAMES[oc], "trace": tr}
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f)


if __name__ == "__main__":
    main()
