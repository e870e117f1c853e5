"""BASELINE config C5's kappa = 2 twin (n = 32768, p = 2) through the C-ABI with the CRT FP64 phase and
with the DMMA FP64 phase (one solve each; CUDA-event time incl. init and the certified residual).
  python tools/c5_crt.py [--schedules s1,s2]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schedules", default="symtri:bf16>fp64crt@a/cbf16,symtri:bf16>fp64/cbf16")
    ap.add_argument("--n", type=int, default=32768)
    a = ap.parse_args()
    import torch
    import bench
    import paper_1703_02283_b200 as ipr
    import synth
    c = synth.CONFIGS["C5"]
    A, _ = synth.spd_torch(a.n, 2.0, c["seed"], device="cuda")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    st = torch.cuda.current_stream()
    for sched in a.schedules.split(","):
        form, ph = bench.schedule(sched, a.n)
        ph[-1].max_iters = 40
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s = ipr.Solver(A, c["p"], ph, 1e-12, st, form=form)
        s.iterate(200)
        tr = s.trace()
        cert = [t["rho_cert"] for t in tr if t["rho_cert"] == t["rho_cert"]]
        oc = ipr.OUTCOME_NAMES[s.outcome]
        s.close()
        e1.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"n": a.n, "p": c["p"], "kappa": 2.0, "schedule": sched, "outcome": oc,
                          "iters_per_phase": [sum(1 for t in tr if t["phase"] == i) for i in range(len(ph))],
                          "moduli": [t["moduli"] for t in tr if t["moduli"]], "rho_cert": cert[-1] if cert else None,
                          "time_s": e0.elapsed_time(e1) / 1e3}), flush=True)


if __name__ == "__main__":
    main()
