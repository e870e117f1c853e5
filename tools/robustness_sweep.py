"""The bench's default schedule on other seeds / sizes / condition numbers of the BASELINE family
(one solve each through the C-ABI): outcome, iterations per phase, certified residual, DMMA re-check,
time.  python tools/robustness_sweep.py [--schedule ...] [--cert crt|fp64]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schedule", default=None)
    ap.add_argument("--cert", default="crt")
    a = ap.parse_args()
    import torch
    import bench
    import paper_1703_02283_b200 as ipr
    import synth
    sched = a.schedule or bench.DEFAULT_SCHEDULE
    st = torch.cuda.current_stream()
    for n, kappa, seed in [(4096, 2.0, 0), (4096, 2.0, 1), (4096, 5.0, 2), (8192, 2.0, 6), (8192, 2.0, 7),
                           (8192, 5.0, 8), (6144, 2.0, 9), (2560, 2.0, 10), (4096, 10.0, 11), (4096, 20.0, 12)]:
        A, _ = synth.spd_torch(n, kappa, seed, device="cuda")
        form, ph = bench.schedule(sched, n)
        ph[-1].max_iters = 60
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s = ipr.Solver(A, 2, ph, 1e-12, st, form=form, cert=a.cert)
        s.iterate(300)
        tr = s.trace()
        e1.record(st)
        torch.cuda.synchronize()
        terms = ipr.ipr_test_cert_info(s.ctx) if a.cert == "crt" else None
        chk = s.residual(1)
        dmma = s.residual(2)
        oc = ipr.OUTCOME_NAMES[s.outcome]
        s.close()
        cert = [t["rho_cert"] for t in tr if t["rho_cert"] == t["rho_cert"]]
        print(json.dumps({"n": n, "kappa": kappa, "seed": seed, "schedule": sched, "outcome": oc,
                          "iters_per_phase": [sum(1 for t in tr if t["phase"] == i) for i in range(len(ph))],
                          "rho_cert": cert[-1] if cert else None, "recheck": chk, "dmma_eval": dmma,
                          "est": terms["est"] if terms else None, "beta": terms["beta"] if terms else None,
                          "certificates": len(cert), "ztri_chains": sum(t["ztri"] for t in tr), "cert_first": bool(tr and tr[-1]["rho"] != tr[-1]["rho"]),
                          "time_s": e0.elapsed_time(e1) / 1e3}), flush=True)
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
