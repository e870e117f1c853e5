"""bench.py -- time-to-FP64-residual of the Bini inverse p-th root iteration (arXiv:1703.02283) on B200.

One *step* = one complete solve of the hot path through the C-ABI:
ipr_init (symmetry check, norms of Eq. 3) -> C_0 -> controller-driven iterations of Eq. (1)
(p GEMMs + fused residual, GEMM p+1 + fused update) until rho = ||I - C^p A||_F <= 1e-12 ->
ipr_finalize (best C to a caller buffer).  Inputs are resident in HBM when the timed region
starts; the e2e number adds the pinned host->device copy of A and the device->host copy of C.

Workload: BASELINE.json's headline n=8192, p=2.  At the stated kappa=1e4
Eq. (1) cannot reach 1e-12 at all (reading R-3), so the timed workload is its
kappa=2 twin ("H_twin", seed 5).  A (537 MB FP64) is larger than the 126 MB L2, so no L2 flush
is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extras]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-FP64-residual 1e-12 (n=8192, p=2)"
# headline schedule (symmetrised-correction form with the upper-triangle GEMM 2, NEXT-2 (i)+(iii),
# DESIGN.md R-22) -- dynamic precision scaling over three precisions: an FP8 E4M3
# phase (scaled, R-24) while C is far from the root, a BF16 phase, then an FP64-range phase whose GEMMs
# run on the INT8 tensor cores by the Ozaki scheme II (CRT over 8-bit moduli, R-28) with the precision --
# 3..9 digit-equivalents, i.e. 17..59 bits and 6..17 moduli -- and the stored bits raised per iteration
# from the residual (R-26); BF16 correction GEMMs; convergence certified on ||I - C^2 A||_F at full FP64
# accuracy.  (FP8 > BF16 > CRT measured 154.4-155.1 ms vs 157.0-159.0 ms for BF16 > CRT, alternating runs.)
DEFAULT_SCHEDULE = "symtriz:fp8/cfp8>bf16>fp64crt@a/cbf16"   # symtriz: reading R-37 (r02l); symtri: the r02i headline
EXTRA_SCHEDULES = ["fp64", "symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", "symtri:fp8>bf16>fp64crt@a/cbf16", "symtri:bf16>fp64crt@a/cbf16", "symtri:bf16>fp64oz@a/cbf16", "symtri:int8>bf16>fp64crt@a/cbf16", "sym:fp64crt", "symtri:bf16>fp64oz@23/cbf16>fp64oz/cbf16", "symtri:bf16>fp64oz/cbf16", "sym:fp64oz", "symtri:fp8>bf16>fp64oz@23/cbf16>fp64oz/cbf16",
                   "bf16>fp64", "tf32>fp64", "fp16>fp64", "sym:fp64", "sym:fp64/cbf16", "symtri:fp64/cbf16",
                   "symtri:bf16>fp64/cbf16", "symtri:bf16>tf32>fp64/cbf16", "symtri:fp8>bf16>fp64/cbf16",
                   "symtri:int8>bf16>fp64/cbf16", "symtri:fp16>fp64/cbf16",
                   "sym:bf16>fp64", "sym:tf32>fp64/cbf16", "sym:bf16>tf32>fp64/cbf16"]
FP64_PEAK_TFLOPS = 37.1   # measured DMMA issue peak on this pool (profiles/r01_calibration.md)
FP64_PEAK_SRC = "measured DMMA.8x8x4 issue peak, tools/probes/dmma_rate.cu (MEASURED_PEAKS.json has no FP64 figure)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="H_twin")
    ap.add_argument("--schedule", default=DEFAULT_SCHEDULE,
                    help="[sym:|ns:]phase>phase..., phase = prec[/c<corr prec>], e.g. fp64, bf16>fp64, "
                         "sym:bf16>fp64/cbf16 (sym: = IPR_FORM_SYMMETRIC, NEXT-2)")
    ap.add_argument("--cert", choices=["auto", "crt", "fp64"], default="auto",
                    help="convergence certificate: crt = IPR_CERT_CRT (a proven bound on the exact residual, "
                         "R-35; symmetric p = 2 with an fp64crt phase, any 1 x G), fp64 = IPR_CERT_FP64 (DMMA "
                         "evaluation, R-30); auto = crt where it applies")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    return ap.parse_args()


def parse_schedule(name):
    """'sym:bf16>fp64oz@23/cbf16>fp64' -> ("symmetric", [("bf16", -1, -1), ("fp64oz", "bf16", 23),
    ("fp64", -1, -1)]): phases prec[@mant_bits][/c<correction prec>]."""
    form = "literal"
    if ":" in name:
        f, name = name.split(":", 1)
        form = {"sym": "symmetric", "symtri": "symmetric_tri", "symtriz": "symmetric_triz", "ns": "newton_schulz", "lit": "literal",
                "cpl": "coupled"}[f]
    parts = []
    for ph in name.replace("-", ">").split(">"):
        ph, _, m = ph.partition("@")          # prec[@mant_bits][/c<corr>]
        if "/c" in m:
            m, _, corr = m.partition("/c")
            ph = ph + "/c" + corr
        prec, _, corr = ph.partition("/c")
        parts.append((prec, corr or -1, (-2 if m == "a" else int(m)) if m else -1))   # @a: adaptive (R-26)
    return form, parts


def schedule(name, n):
    """Phases of a named schedule.  Every phase but the last is left on an armed plateau (and,
    in the literal form, at rho_hat <= 1e-2) -- reading R-5; the last runs to final_tol."""
    import paper_1703_02283_b200 as ipr
    form, parts = parse_schedule(name)
    out = []
    for i, (prec, corr, m) in enumerate(parts):
        if i == len(parts) - 1:
            out.append(ipr.make_phase(prec, mant_bits=m, corr_prec=corr))
        else:
            # the symmetric form damps low-precision noise in the next phase: a low phase runs to its
            # plateau, or until rho_hat <= 2 u of its operand format (u = 2^-(m+1); below that the format
            # makes no further progress -- it saves the iteration that only confirms the plateau); the
            # literal form leaves at rho_hat <= 1e-2 as well
            mbits = {"bf16": 7, "int8": 7, "fp8": 3, "fp16": 10, "tf32": 10}.get(prec, 52)
            sw = (2.0 * 2.0 ** -(mbits + 1) * math.sqrt(n)) if form.startswith("symmetric") else 1e-2 * math.sqrt(n)
            out.append(ipr.make_phase(prec, mant_bits=m, switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.5,
                                      max_iters=40, corr_prec=corr))
    return form, out


def sustained_int8_peak():
    """INT8 peak for a kernel timed inside a long step: MEASURED_PEAKS.json's sustained bf16 x 2
    (nominal int8:bf16); None if the file has no sustained figure."""
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return 2.0 * float(json.load(open(mp))["bf16_tflops_sustained"]), \
            "MEASURED_PEAKS.json bf16_tflops_sustained x 2 (nominal int8:bf16): the kernel is timed inside the solve"
    except Exception:
        return None


def gemm_peaks():
    """Dense tensor peak per operand format: MEASURED_PEAKS.json's bf16 burst (driver-written),
    other formats by the guide's nominal ratios (tf32 = 1/2, fp8 = int8 = 2 x bf16); FP64 = the
    measured DMMA issue peak."""
    bf16 = 1599.0
    src = "fallback 1599 (no MEASURED_PEAKS.json)"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            bf16 = float(json.load(open(mp))["bf16_tflops"])
            src = "MEASURED_PEAKS.json bf16_tflops (burst)"
        except Exception:
            pass
    return {"fp64": (FP64_PEAK_TFLOPS, FP64_PEAK_SRC), "bf16": (bf16, src), "fp16": (bf16, src + " (fp16 = bf16 rate)"),
            "tf32": (bf16 / 2, src + " x 1/2 (nominal tf32:bf16)"), "fp8": (bf16 * 2, src + " x 2 (nominal fp8:bf16)"),
            "int8": (bf16 * 2, src + " x 2 (nominal int8:bf16)"),
            "fp64oz": (bf16 * 2, src + " x 2 (INT8 peak; Ozaki FP64 = 45 INT8 digit products)"),
            "fp64crt": (bf16 * 2, src + " x 2 (INT8 peak; Ozaki-II FP64 = N INT8 modulus products)")}


def gemm_count(trace, p):
    # p GEMMs per evaluated chain (none for a certificate-only record, R-33), +1 for every update that
    # followed, +p per FP64 certification
    return sum((p if t["rho"] == t["rho"] else 0) + (1 if t["decision"] == 0 else 0) +
               (p if t["rho_cert"] == t["rho_cert"] else 0) for t in trace)


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.p = None
        self.out = ""

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = [r.split(",") for r in self.out.strip().splitlines() if r.count(",") >= 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def oracle_schedule(name, n):
    """The oracle's phases for a bench schedule name (same switch / plateau rules as schedule())."""
    import oracle
    form, parts = parse_schedule(name)
    opr = {"fp64": oracle.FP64, "tf32": oracle.TF32, "bf16": oracle.BF16, "fp16": oracle.FP16, "fp8": oracle.FP8,
           "int8": oracle.INT8, "fp64oz": oracle.FP64_OZ, "fp64crt": oracle.FP64_CRT}
    oform = {"literal": oracle.FORM_LITERAL, "symmetric": oracle.FORM_SYMMETRIC, "symmetric_tri": oracle.FORM_SYMMETRIC_TRI,
             "symmetric_triz": oracle.FORM_SYMMETRIC_TRIZ, "newton_schulz": oracle.FORM_NEWTON_SCHULZ, "coupled": oracle.FORM_COUPLED}[form]
    out = []
    for i, (prec, corr, m) in enumerate(parts):
        c = opr[corr] if corr != -1 else -1
        if i == len(parts) - 1:
            out.append(oracle.phase(opr[prec], mant_bits=m, corr_prec=c))
        else:
            mbits = {"bf16": 7, "int8": 7, "fp8": 3, "fp16": 10, "tf32": 10}.get(prec, 52)
            sw = (2.0 * 2.0 ** -(mbits + 1) * math.sqrt(n)) if form.startswith("symmetric") else 1e-2 * math.sqrt(n)
            out.append(oracle.phase(opr[prec], mant_bits=m, switch_tol=sw, plateau_ratio=0.7, plateau_arm=0.5,
                                    max_iters=40, corr_prec=c))
    return oform, out


def oracle_gemms(records, p):
    """GEMMs of an oracle solve: p per chain (none for a certificate-only record, R-33), +1 per update
    (decision continue), +p per certification."""
    return sum((p if x["rho"] == x["rho"] else 0) + (1 if x["decision"] == 0 else 0) +
               (p if x["rho_cert"] == x["rho_cert"] else 0) for x in records)


def auto_cert(schedule_name, p, choice="auto", world=1):
    """The certificate a run uses: IPR_CERT_CRT (R-35) where it applies -- a symmetric form with an fp64crt
    phase, p = 2 (any 1 x G) or p = 3 (one GPU) -- else IPR_CERT_FP64 (R-30); an explicit choice wins."""
    if choice != "auto":
        return choice
    form, parts = parse_schedule(schedule_name)
    crt = any(x[0] == "fp64crt" for x in parts) and form.startswith("symmetric")
    return "crt" if crt and (p == 2 or (p == 3 and world == 1)) else "fp64"


def cpu_baseline(schedule_name, p, n_target, gemms_target=None, n_small=1024, seed=5, cert="fp64"):
    """The oracle (plain C, FP64 triple loops; FP64_CRT products as exact 128-bit integer sums) as it
    stands, timed on the host cores on ONE REAL SOLVE: the same schedule on the kappa = 2 twin at order
    n_small (measured), then scaled to n_target by n^3 and by the GEMM count (the target's, when the GPU
    run supplies it, else the oracle's own at n_small) -- the scaling is labelled as extrapolation."""
    import oracle
    import synth
    A_s = synth.spd(n_small, 2.0, seed)
    oform, ph = oracle_schedule(schedule_name, n_small)
    t0 = time.perf_counter()
    r = oracle.solve(A_s, p, ph, 1e-12, 300, form=oform, cert=cert)
    t = time.perf_counter() - t0
    g_small = oracle_gemms(r.records, p)
    g_t = gemms_target if gemms_target else g_small
    scale = (n_target / n_small) ** 3 * g_t / g_small
    iters = [sum(1 for x in r.records if x["phase"] == i) for i in range(len(ph))]
    certs = [x["rho_cert"] for x in r.records if x["rho_cert"] == x["rho_cert"]]
    cores = len(os.sched_getaffinity(0))
    return {"value": t * scale, "unit": "s", "cores": cores, "kind": "oracle",
            "sample": f"one full oracle solve of {schedule_name} (certificate {cert}) on the kappa=2 twin at n={n_small} (seed {seed}): "
                      f"{oracle.OUTCOME_NAMES[r.outcome]}, iterations {iters}, certified rho "
                      f"{certs[-1] if certs else float('nan'):.3e}, {g_small} GEMMs in {t:.1f} s on {cores} threads "
                      f"(measured); value = that x (n={n_target}/{n_small})^3 x ({g_t} / {g_small} GEMMs) (extrapolated"
                      f"{', GEMM count of the GPU trajectory at n=' + str(n_target) if gemms_target else ', the oracle GEMM count at n_small'})",
            "measured_solve_s": t, "measured_n": n_small, "measured_iters": iters, "extrapolated": True}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import numpy as np
    import torch
    import synth

    cfg = synth.CONFIGS[args.workload]
    n, p, kappa, seed = cfg["n"], cfg["p"], cfg["kappa"], cfg["seed"]
    config = {"workload": f"{args.workload}: n={n} p={p} kappa={kappa:g} seed={seed}, schedule={args.schedule}, "
                          f"stop at rho<=1e-12 (twin of BASELINE headline n=8192 p=2 kappa=1e4, reading R-3)",
              "n": n, "p": p, "kappa": kappa, "seed": seed, "schedule": args.schedule,
              "l2": "inputs larger than L2 (A = %.0f MB FP64 > 126 MB); no flush" % (n * n * 8 / 1e6),
              "parallelism": f"1x{args.gpus} column panels" if args.gpus > 1 else "single GPU"}

    cert = auto_cert(args.schedule, p, args.cert, int(os.environ.get("WORLD_SIZE", "1")))
    config["certificate"] = cert

    if args.impl == "reference":
        # Reference arm = the oracle as it stands on the host cores (rank 0 only): every step one real oracle
        # solve of the same schedule at n = 512 (a bounded sample), scaled to the workload's n by n^3 at the
        # oracle's own GEMM count (see cpu_baseline)
        if rank != 0:
            return
        vals = []
        for i in range(args.warmup + args.steps):
            cb = cpu_baseline(args.schedule, p, n, None, n_small=512, cert=cert)
            if i >= args.warmup:
                vals.append(cb["value"])
        v = float(np.mean(vals))
        cb["value"] = v
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": cb, "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import paper_1703_02283_b200 as ipr
    torch.cuda.set_device(local)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [ipr.ipr_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.current_stream()
    A, lam = synth.spd_torch(n, kappa, seed, device="cuda")
    C_out = torch.empty_like(A)
    torch.cuda.synchronize()
    form, phases = schedule(args.schedule, n)
    def solve(A_dev, out, early_out=False):
        s = ipr.Solver(A_dev, p, phases, 1e-12, stream, world, rank, uid, form=form, cert=cert)
        if early_out:
            s.set_output(out)     # the certified answer streams to `out` while its certificate runs
        s.iterate(400)
        tr = s.trace()
        outcome = s.outcome
        s.finalize(out)
        return tr, outcome

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solve(A, C_out)
    barrier()
    l0 = ipr.ipr_launch_count()
    traces = []
    with Clocks(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            traces.append(solve(A, C_out))
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ipr.ipr_launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tr, outcome = traces[-1]
    # independent check outside the timed region: one more solve, then its certificate recomputed from
    # the returned matrix by ipr_residual(certify=1) (the same function as the in-solve certificate, so
    # the two agree bit for bit), and the FP64 DMMA evaluation ipr_residual(certify=2) beside it.
    # "converged" requires the outcome and the re-computed certificate <= 1e-12.
    sv = ipr.Solver(A, p, phases, 1e-12, stream, world, rank, uid, form=form, cert=cert)
    sv.iterate(400)
    rho_recheck = sv.residual(1)
    cert_terms = ipr.ipr_test_cert_info(sv.ctx) if cert == "crt" else None
    rho_dmma = sv.residual(2)
    sv.close()
    certs = [t["rho_cert"] for t in tr if t["rho_cert"] == t["rho_cert"]]
    final_rho = certs[-1] if certs else tr[-1]["rho"]
    ok = outcome == ipr.IPR_CONVERGED and rho_recheck <= 1e-12

    # roofline of the dominant kernel (the FP64 DMMA GEMM): algorithmic flops per launch =
    # 2 n^3 (local panel: 2 n^2 n/G); duration from the library's CUDA events on the launch stream
    fl_gemm = 2.0 * n * n * (n / world)
    # the p chain GEMMs of every FP64 record (gemm_ms - upd_ms: the update may be a BF16
    # correction GEMM + k_sym_update in the symmetric form).  Algorithmic flops of a chain:
    # p * 2 n^3 / G, except the tri form, whose GEMM 2 (C A C) needs only the upper triangle:
    # 2 n^3 + n^2 (n + 1) (its extra work on the diagonal tiles is overhead, not credit).
    fl_chain = (2.0 * n ** 3 + n * n * (n + 1.0)) if form in ("symmetric_tri", "symmetric_triz") else p * fl_gemm
    fl_ztri = 2.0 * n * n * (n + 1.0)   # R-37: a chain whose Z_1 runs on its upper tiles too (record.ztri)
    last = ipr.PREC_NAMES[phases[-1].prec]
    recs = [t for trc, _ in traces for t in trc if t["phase"] == len(phases) - 1]   # the last phase only
    tot_ms = sum(t["gemm_ms"] - t["upd_ms"] for t in recs)
    n_chains = len(recs)
    all_ms = sum(t["gemm_ms"] for trc, _ in traces for t in trc)
    step_gemm_share = tot_ms / (ms * args.steps) if ms > 0 else None
    peaks = gemm_peaks()
    if last == "fp64oz":
        # dominant kernel: the INT8 tcgen05 GEMMs of the Ozaki FP64 products (S(S+1)/2 digit products
        # per FP64 product at S digits, from each record's `digits`): achieved INT8 TOPS over the
        # whole chains (digit splits and FP64 finish passes included -- counted as overhead, not
        # credit), vs the INT8 peak
        prods_tot = sum(t["digits"] * (t["digits"] + 1) / 2.0 for t in recs)   # S(S+1)/2 per chain
        prods = prods_tot / max(n_chains, 1)
        achieved = prods_tot * fl_chain / (tot_ms * 1e-3) / 1e12 if tot_ms > 0 else None
        roof = {"bound": "tensor", "kernel": "k_gemm_tc<kind::i8> (Ozaki FP64 chain: 9 K-concatenated INT8 GEMMs "
                "per product + digit split + FP64 finish)", "achieved": achieved, "peak": peaks["int8"][0],
                "unit": "TOPS (int8)", "frac": achieved / peaks["int8"][0] if achieved else None, "traffic": None,
                "peak_source": peaks["int8"][1], "fp64_equivalent_tflops": achieved / prods if achieved else None,
                "algorithmic_int8_ops_per_chain_avg": prods * fl_chain, "digit_products_per_chain_avg": prods,
                "chains": n_chains,
                "avg_chain_ms": tot_ms / max(n_chains, 1), "gemm_share_of_step": step_gemm_share,
                "all_gemm_share_of_step": all_ms / (ms * args.steps) if ms > 0 else None}
        traffic_key = "k_gemm_tc_i8_ozaki"
    elif last == "fp64crt":
        # dominant kernel: the INT8 tcgen05 GEMMs of the Ozaki-II (CRT) FP64 products -- one n^3 INT8
        # GEMM per modulus (each record's `moduli`).  achieved = algorithmic INT8 ops / the device time
        # of those GEMM launches alone (each record's `kern_ms`: CUDA events around the modulus GEMM
        # launches on the library's stream); chain_* = the same over whole chains (residue splits and
        # the CRT reconstruction / finish passes counted as overhead)
        mods_tot = sum(t["moduli"] for t in recs)
        mods = mods_tot / max(n_chains, 1)
        kern_ms = sum(t["kern_ms"] for t in recs)
        ops = sum(t["moduli"] * (fl_ztri if t.get("ztri") else fl_chain) for t in recs)
        achieved = ops / (kern_ms * 1e-3) / 1e12 if kern_ms > 0 else None
        chain_ach = ops / (tot_ms * 1e-3) / 1e12 if tot_ms > 0 else None
        # peak: the BURST figure -- inside the solve the INT8 GEMMs run in short bursts between other
        # kernels and host syncs, at clocks well above the 4 s sustained measurement's (r02: 1770 vs 1357
        # MHz median), so the sustained figure under-states the ceiling (frac > 1); both are reported
        pk, pk_src = peaks["int8"]
        sus = sustained_int8_peak()
        roof = {"bound": "tensor", "kernel": "k_gemm_tc<kind::i8> (Ozaki-II FP64 products: one INT8 GEMM per CRT "
                "modulus, 2 moduli per launch)", "achieved": achieved, "peak": pk,
                "unit": "TOPS (int8)", "frac": achieved / pk if achieved else None, "traffic": None,
                "peak_source": pk_src,
                "frac_of_sustained_peak": achieved / sus[0] if (achieved and sus) else None,
                "sustained_peak": sus[0] if sus else None,
                "algorithmic_int8_ops_per_chain_avg": ops / max(n_chains, 1), "moduli_per_chain_avg": mods,
                "chains": n_chains, "ztri_chains": sum(1 for t in recs if t.get("ztri")), "kernel_ms_per_chain_avg": kern_ms / max(n_chains, 1),
                "avg_chain_ms": tot_ms / max(n_chains, 1), "chain_achieved_tops": chain_ach,
                "chain_frac": chain_ach / pk if chain_ach else None,
                "fp64_equivalent_tflops_chain": chain_ach / mods if chain_ach else None,   # per the chains' own op counts
                "gemm_share_of_step": step_gemm_share,
                "kernel_share_of_step": kern_ms / (ms * args.steps) if ms > 0 else None,
                "all_gemm_share_of_step": all_ms / (ms * args.steps) if ms > 0 else None}
        traffic_key = "k_gemm_tc_i8_crt"
    else:
        tot_gemms = p * n_chains
        gemm_ms = tot_ms / max(tot_gemms, 1)
        achieved = (n_chains * fl_chain) / (tot_ms * 1e-3) / 1e12 if tot_ms > 0 else None
        roof = {"bound": "tensor", "kernel": "k_gemm_dmma (FP64 DMMA.8x8x4)", "achieved": achieved,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                "traffic": None, "peak_source": FP64_PEAK_SRC, "cublas_dgemm_tflops": 35.5,
                "algorithmic_flops_per_launch": fl_chain / p, "avg_launch_ms": gemm_ms,
                "algorithmic_flops_per_chain": fl_chain, "launches_per_chain": p, "gemm_share_of_step": step_gemm_share,
                "all_gemm_share_of_step": all_ms / (ms * args.steps) if ms > 0 else None}
        traffic_key = "k_gemm_dmma"
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            roof["traffic"] = json.load(open(tp)).get(traffic_key)
        except Exception:
            pass

    # e2e: the same solve through the C-ABI with HOST buffers (pinned): ipr_init copies A in, the
    # answer streams back to host during its FP64 certificate (ipr_set_output) and ipr_finalize writes
    # the host C -- every copy inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        A_host = A.cpu().pin_memory()
        C_host = torch.empty_like(A_host).pin_memory()
        solve(A_host, C_host, early_out=True)   # untimed warm-up of this path (copy stream, pool block of A)
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            solve(A_host, C_host, early_out=True)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / args.e2e_steps
        if dist is not None:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": ems / 1e3, "unit": "s", "h2d_bytes_per_step": A_host.numel() * 8,
               "d2h_bytes_per_step": C_host.numel() * 8}

    extras = {}
    if not args.no_extras and world == 1:
        # the other half of the metric: GEMM TFLOP/s per precision, and the mixed schedules
        sched = {}
        for name in EXTRA_SCHEDULES:
            f2, ph = schedule(name, n)
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            s = ipr.Solver(A, p, ph, 1e-12, stream, form=f2)
            s.iterate(400)
            t2 = s.trace()
            out2 = s.outcome
            s.finalize(C_out)
            g1.record(stream)
            torch.cuda.synchronize()
            precs = [ipr.PREC_NAMES[q.prec] for q in ph]
            low = precs[0] if len(precs) > 1 else None
            lms = sum(t["gemm_ms"] for t in t2 if t["prec"] == low) if low else 0.0
            lg = gemm_count([t for t in t2 if t["prec"] == low], p) if low else 0
            c2 = [t["rho_cert"] for t in t2 if t["rho_cert"] == t["rho_cert"]]
            sched[name] = {"time_s": g0.elapsed_time(g1) / 1e3, "outcome": ipr.OUTCOME_NAMES[out2],
                           "iters_per_phase": [sum(1 for t in t2 if t["phase"] == i) for i in range(len(ph))],
                           "final_rho": c2[-1] if c2 else t2[-1]["rho"],
                           "gemm_tflops_low": (lg * 2.0 * n ** 3 / (lms * 1e-3) / 1e12) if lms > 0 else None}
        extras["schedules"] = sched
        # the same schedule certified by the FP64 DMMA evaluation (IPR_CERT_FP64, R-30) instead
        if cert == "crt":
            f2, ph = schedule(args.schedule, n)
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            s = ipr.Solver(A, p, ph, 1e-12, stream, form=f2, cert="fp64")
            s.iterate(400)
            g1.record(stream)
            t2 = s.trace()
            torch.cuda.synchronize()
            c2 = [t["rho_cert"] for t in t2 if t["rho_cert"] == t["rho_cert"]]
            extras["cert_fp64_dmma"] = {
                "time_s": g0.elapsed_time(g1) / 1e3, "outcome": ipr.OUTCOME_NAMES[s.outcome],
                "iters_per_phase": [sum(1 for t in t2 if t["phase"] == i) for i in range(len(ph))],
                "rho_cert": c2[-1] if c2 else None,
                "note": "IPR_CERT_FP64: the same schedule certified by the FP64 DMMA evaluation (1.5 DMMA GEMMs)"}
            s.close()
        # reading R-37 A/B: the tri form without the Z_1 rule (the r02i headline), same phases, same certificate
        if args.schedule.startswith("symtriz:"):
            f2, ph = schedule("symtri:" + args.schedule.split(":", 1)[1], n)
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                g0 = torch.cuda.Event(enable_timing=True)
                g1 = torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                s = ipr.Solver(A, p, ph, 1e-12, stream, form=f2, cert=cert)
                s.iterate(400)
                t2 = s.trace()
                s.finalize(C_out)
                g1.record(stream)
                torch.cuda.synchronize()
                ts.append(g0.elapsed_time(g1) / 1e3)
            c2 = [t["rho_cert"] for t in t2 if t["rho_cert"] == t["rho_cert"]]
            extras["form_symtri"] = {
                "time_s": sorted(ts)[1], "outcome": ipr.OUTCOME_NAMES[s.outcome],
                "iters_per_phase": [sum(1 for t in t2 if t["phase"] == i) for i in range(len(ph))],
                "rho_cert": c2[-1] if c2 else None,
                "note": "IPR_FORM_SYMMETRIC_TRI (full Z_1 in the FP64_CRT phase), same phases and certificate; median of 3"}
        # the cost of the honest certificate: the default schedule with the phase-product estimate
        # (IPR_CERT_PHASE: the CRT product, p - 1 products instead of p DMMA GEMMs) -- diagnostics only,
        # its acceptance is not an FP64 certificate (ipr.h ipr_set_cert)
        f2, ph = schedule(args.schedule, n)
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        s = ipr.Solver(A, p, ph, 1e-12, stream, form=f2, cert="phase")
        s.iterate(400)
        g1.record(stream)
        t2 = s.trace()
        torch.cuda.synchronize()
        c2 = [t["rho_cert"] for t in t2 if t["rho_cert"] == t["rho_cert"]]
        extras["cert_phase_estimate"] = {
            "time_s": g0.elapsed_time(g1) / 1e3, "outcome": ipr.OUTCOME_NAMES[s.outcome],
            "iters_per_phase": [sum(1 for t in t2 if t["phase"] == i) for i in range(len(ph))],
            "rho_cert_phase": c2[-1] if c2 else None, "dmma_recheck": s.residual(True),
            "note": "IPR_CERT_PHASE: accepted on the CRT product's residual (an estimate, not the FP64 certificate)"}
        s.close()
        # the other half of the metric: the hot-path GEMM kernel of every format, timed alone
        # (ipr_bench_gemm: CUDA events, EPI_STORE_T epilogue, 2 n^3 flop per launch), against the
        # peak of its own dtype (burst figure: a kernel timed alone)
        peaks = gemm_peaks()
        rates, fracs = {}, {}
        n_mod = ipr.ipr_test_crt_table(18, ipr.ipr_test_crt_table(18, 9, n)["b_for"], n)["n_for"]   # moduli at S = 9
        for prec in ["fp64", "fp64oz", "fp64crt", "tf32", "bf16", "fp16", "fp8", "int8"]:
            gms = ipr.ipr_bench_gemm(prec, n, 2, 5, stream)
            rates[prec] = 2.0 * n ** 3 / (gms * 1e-3) / 1e12
            # fp64oz / fp64crt: FP64-equivalent TFLOP/s; the tensor-core fraction is that of the 45 INT8
            # digit products / the n_mod INT8 modulus products against the INT8 peak
            mult = 45.0 if prec == "fp64oz" else float(n_mod) if prec == "fp64crt" else 1.0
            fracs[prec] = rates[prec] * mult / peaks[prec][0]
        extras["gemm_tflops"] = rates
        extras["gemm_frac_of_peak"] = fracs
        extras["gemm_peaks"] = {k: {"tflops": v[0], "source": v[1]} for k, v in peaks.items()}

    if rank != 0:
        return
    cb = None
    if world == 1:
        try:
            cb = cpu_baseline(args.schedule, p, n, gemm_count(tr, p), n_small=1024, cert=cert)
        except Exception as ex:  # never fail the bench line on the CPU leg
            cb = {"value": None, "unit": "s", "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}
    line = {"metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "converged": ok, "iterations": len(tr), "final_rho": final_rho, "final_rho_recheck": rho_recheck,
            "final_rho_dmma_recheck": rho_dmma,
            "certificate": ("IPR_CERT_CRT (R-35): a proven upper bound on the EXACT ||I - C^2 A||_F of the returned C "
                            "(the candidate on its 62-bit row/column grid), from exact integer products on the INT8 "
                            "tensor cores plus the a-posteriori quantisation / reconstruction bounds, inside the timed "
                            "solve (= ipr_residual(certify=1), bit for bit); final_rho_dmma_recheck is an FP64 DMMA "
                            "evaluation of the same C (~n u rounding noise)") if cert == "crt" else
                           "IPR_CERT_FP64: ||I - C^2 A||_F of the returned C by the literal chain on the FP64 DMMA "
                           "pipe inside the timed solve (= ipr_residual(certify=1), bit for bit)",
            "certificate_terms": cert_terms,
            "iters_per_phase": [sum(1 for t in tr if t["phase"] == i) for i in range(len(phases))],
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary()}
    line.update(extras)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
