"""Where the headline step's time goes outside the GEMM chains: CUDA-event totals of
init, iterate, finalize, and the records' own device times (chain = gemm_ms - upd_ms, update = upd_ms).
python tools/gap_probe.py [--schedule ...] [--cert fp64|phase]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schedule", default=None)
    ap.add_argument("--cert", default="fp64")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--trace", action="store_true", help="print the last rep's records")
    a = ap.parse_args()
    import torch
    import bench
    import paper_1703_02283_b200 as ipr
    import synth
    cfg = synth.CONFIGS["H_twin"]
    n, p = cfg["n"], cfg["p"]
    A, _ = synth.spd_torch(n, cfg["kappa"], cfg["seed"], device="cuda")
    st = torch.cuda.current_stream()
    form, ph = bench.schedule(a.schedule or bench.DEFAULT_SCHEDULE, n)
    out = torch.empty_like(A)
    for rep in range(a.reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        ev[0].record(st)
        s = ipr.Solver(A, p, ph, 1e-12, st, form=form, cert=a.cert)
        ev[1].record(st)
        h1 = time.perf_counter()
        s.iterate(400)
        ev[2].record(st)
        h2 = time.perf_counter()
        tr = s.trace()
        s.finalize(out)
        ev[3].record(st)
        torch.cuda.synchronize()
        h3 = time.perf_counter()
        t = [ev[0].elapsed_time(ev[i]) for i in (1, 2, 3)]
        chain = sum(r["gemm_ms"] - r["upd_ms"] for r in tr)
        gaps = [r["gap_ms"] for r in tr if r["gap_ms"] == r["gap_ms"]]
        upd = sum(r["upd_ms"] for r in tr)
        print(f"rep {rep}: total {t[2]:.2f} ms (init {t[0]:.2f}, iterate {t[1] - t[0]:.2f}, finalize {t[2] - t[1]:.2f}); "
              f"records {len(tr)}: chains {chain:.2f} + updates {upd:.2f} = {chain + upd:.2f} ms; "
              f"iterate - records = {t[1] - t[0] - chain - upd:.2f} ms; controller bubbles {sum(gaps):.2f} ms over "
              f"{len(gaps)} updates (max {max(gaps) if gaps else 0:.3f}); host wall init/iter/fin "
              f"{(h1 - h0) * 1e3:.1f}/{(h2 - h1) * 1e3:.1f}/{(h3 - h2) * 1e3:.1f} ms", flush=True)
    if a.trace:
        for r in tr:
            print(f"k={r['k']:3d} ph={r['phase']} dec={r['decision']} rho={r['rho']:.3e} cert={r['rho_cert']:.3e} "
                  f"m={r['mant_bits']} S={r['digits']} N={r['moduli']} chain={r['gemm_ms'] - r['upd_ms']:.3f} "
                  f"upd={r['upd_ms']:.3f} kern={r['kern_ms']:.3f} delta={r['delta']:.3e}", flush=True)


if __name__ == "__main__":
    main()
