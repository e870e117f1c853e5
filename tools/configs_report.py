"""Run every BASELINE.json config (C1-C5) and its kappa = 2 twin through the C-ABI on one GPU and
report what the method does: outcome, iterations per phase, min rho, time, GEMM
TFLOP/s per phase.  Usage: python tools/configs_report.py [--only C1,C2] [--out file.json]"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1703_02283_b200 as ipr
import synth


def low_then_fp64(low, n, m=-1, fp64_cap=0, switch_rho_hat=1e-2):
    return [ipr.make_phase(low, mant_bits=m, switch_tol=switch_rho_hat * math.sqrt(n), plateau_ratio=0.7,
                           plateau_arm=0.5, max_iters=60),
            ipr.make_phase("fp64", max_iters=fp64_cap)]


def run(A, p, phases, label, max_iters=400, form="literal", tol=1e-12, cert="fp64"):
    n = A.shape[0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = ipr.Solver(A, p, phases, tol, form=form, cert=cert)
    s.iterate(max_iters)
    tr = s.trace()
    out = ipr.OUTCOME_NAMES[s.outcome]
    certs = [t["rho_cert"] for t in tr if t["rho_cert"] == t["rho_cert"]]
    t_solve = time.perf_counter() - t0
    certified = s.residual(1) if tr else float("nan")
    dmma = s.residual(2) if tr and cert == "crt" else certified
    s.close()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rho = [t["rho"] for t in tr]
    fin = [(r, k) for k, r in enumerate(rho) if math.isfinite(r)]
    rmin, kmin = min(fin) if fin else (float("nan"), -1)
    per = {}
    for t in tr:
        native = {"fp64": 52, "fp64oz": 52, "fp64crt": 52, "bf16": 7, "tf32": 10, "fp16": 10, "fp8": 3, "int8": 7}[t["prec"]]
        d = per.setdefault(t["prec"] + ("" if t["mant_bits"] == native else f"/m{t['mant_bits']}"),
                           {"iters": 0, "ms": 0.0, "gemms": 0})
        d["iters"] += 1
        d["ms"] += t["gemm_ms"]
        d["gemms"] += p + (1 if t["decision"] == 0 else 0)
    for d in per.values():
        d["tflops"] = d["gemms"] * 2.0 * n ** 3 / (d["ms"] * 1e-3) / 1e12 if d["ms"] > 0 else None
    rec = {"label": label, "n": n, "p": p, "outcome": out, "iterations": len(tr), "min_rho": rmin,
           "argmin": kmin, "final_rho": rho[-1] if rho else None, "certified_rho_best": certified,
           "certificate": cert, "rho_cert": certs[-1] if certs else None, "dmma_eval_best": dmma,
           "solve_s": t_solve, "time_s": dt, "phases": per}
    print(json.dumps(rec), flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--cert", default="auto", help="auto (IPR_CERT_CRT where it applies) | crt | fp64")
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None
    recs = []

    def want(c):
        return only is None or c in only

    for name in ["C1", "C2", "C3", "C4", "C5"]:
        if not want(name):
            continue
        c = synth.CONFIGS[name]
        n, p, kap, seed = c["n"], c["p"], c["kappa"], c["seed"]
        for kappa, tag in [(kap, "stated"), (2.0, "twin")]:
            A, _ = synth.spd_torch(n, kappa, seed) if n >= 4096 else (torch.from_numpy(synth.spd(n, kappa, seed)).cuda(), None)
            lab = f"{name} n={n} p={p} kappa={kappa:g} ({tag})"
            if name == "C1":
                recs.append(run(A, p, [ipr.make_phase("fp64", max_iters=200)], lab + " fp64"))
            elif name == "C2":
                recs.append(run(A, p, [ipr.make_phase("fp64", max_iters=200)], lab + " fp64"))
                recs.append(run(A, p, low_then_fp64("tf32", n, fp64_cap=200), lab + " tf32->fp64"))
            elif name == "C3":
                recs.append(run(A, p, [ipr.make_phase("fp64", max_iters=120)], lab + " fp64"))
                recs.append(run(A, p, low_then_fp64("bf16", n, fp64_cap=120), lab + " bf16->fp64"))
            elif name == "C4":
                recs.append(run(A, p, [ipr.make_phase("fp64", max_iters=120)], lab + " fp64"))
                for m in [7, 10, 16, 23]:
                    recs.append(run(A, p, [ipr.make_phase("fp64", mant_bits=m, switch_tol=1e-2 * math.sqrt(n),
                                                          plateau_ratio=0.7, plateau_arm=0.5, max_iters=60),
                                           ipr.make_phase("fp64", max_iters=120)], lab + f" fp64-storage m={m}->fp64"))
                recs.append(run(A, p, low_then_fp64("bf16", n, fp64_cap=120), lab + " bf16(m=7)->fp64 (paired)"))
                recs.append(run(A, p, low_then_fp64("tf32", n, fp64_cap=120), lab + " tf32(m=10)->fp64 (paired)"))
            elif name == "C5":
                cap = 30 if tag == "twin" else 8
                if tag == "twin":
                    recs.append(run(A, p, [ipr.make_phase("fp64", max_iters=cap)], lab + " fp64"))
                recs.append(run(A, p, low_then_fp64("bf16", n, fp64_cap=cap), lab + f" bf16->fp64 (fp64 cap {cap})"))
            del A
            torch.cuda.empty_cache()
    # NEXT-1: Newton-Schulz ordering (p = 1) -- where mixed precision beats all-FP64
    for name, n in [("NS-C2", 1024), ("NS-C2@8192", 8192)]:
        if not want(name):
            continue
        c = synth.CONFIGS["C2"]
        for kappa, tol in [(c["kappa"], 1e-9), (2.0, 1e-12)]:
            A, _ = synth.spd_torch(n, kappa, c["seed"])
            lab = f"{name} n={n} p=1 kappa={kappa:g} Newton-Schulz X(2I-AX), tol={tol:g}"
            recs.append(run(A, 1, [ipr.make_phase("fp64", max_iters=200)], lab + " fp64", form="ns", tol=tol))
            for low in ["bf16", "tf32", "fp16"]:
                ph = [ipr.make_phase(low, switch_tol=1e-2 * math.sqrt(n), plateau_ratio=0.7, plateau_arm=0.1,
                                     max_iters=80), ipr.make_phase("fp64", max_iters=200)]
                recs.append(run(A, 1, ph, lab + f" {low}->fp64", form="ns", tol=tol))
            del A
            torch.cuda.empty_cache()
    # NEXT-2: the symmetrised (R-22) / tri and coupled (R-27) forms, Ozaki FP64 with per-iteration
    # digits (R-23, R-26) where it fits (n <= 8192); stated kappa and the kappa = 2 twin
    import bench
    for name in ["C1", "C3", "C4", "C5"]:
        key = "N2-" + name
        if not want(key):
            continue
        c = synth.CONFIGS[name]
        n, p, kap, seed = c["n"], c["p"], c["kappa"], c["seed"]
        sym = "symtri" if p == 2 else "sym"
        for kappa, tag in [(kap, "stated"), (2.0, "twin")]:
            A, _ = synth.spd_torch(n, kappa, seed) if n >= 4096 else (torch.from_numpy(synth.spd(n, kappa, seed)).cuda(), None)
            lab = f"{name} n={n} p={p} kappa={kappa:g} ({tag})"
            runs = [(f"{sym}:fp64/cbf16", 1e-12)]
            # FP64 phase on INT8 tensor cores (CRT, R-28): ~154 GB of arena at n = 32768 (one Chat residue
            # set, scratch aliases), fits a B200
            runs.append((f"{sym}:bf16>fp64crt@a/cbf16", 1e-12))
            if tag == "twin" and n < 32768:   # bench.py's default: FP8 phase with FP8 correction (R-29) first
                runs.append((f"{sym}:fp8/cfp8>bf16>fp64crt@a/cbf16", 1e-12))
            if tag == "stated":
                runs.append(("cpl:fp64", 1e-6))
            for sched, tol in runs:
                form, ph = bench.schedule(sched, n)
                ph[-1].max_iters = 40 if n >= 32768 else 120
                cert = bench.auto_cert(sched, p, a.cert) if not (p == 3 and form == "symmetric_tri") else "fp64"
                recs.append(run(A, p, ph, lab + " " + sched + f" [cert {cert}]", form=form, tol=tol, cert=cert))
            del A
            torch.cuda.empty_cache()
    if a.out:
        json.dump(recs, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
