"""Small invocations of every libipr kernel instance, for compute-sanitizer (memcheck / racecheck /
synccheck).  python tools/sanitize_probe.py N [gemm|solve|all]
  gemm : ipr_test_gemm in every format (k_gemm_tc kinds f16 / tf32 / f8f6f4 / i8, the Ozaki-I and CRT
         i8 instances + k_crt_finish, k_gemm_dmma), ragged n
  solve: the headline schedule (symmetric-tri: FP8 / FP8-correction -> BF16 -> CRT, the tri GEMM with
         mirrored stores, R-29 scratch, k_crt_finish tri path, k_sym_update, DMMA certificate), the
         symmetric / literal / Newton-Schulz / coupled forms, an Ozaki-I phase and the fused update."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1703_02283_b200 as ipr
import synth


def gemms(n):
    rng = np.random.default_rng(n)
    for prec in ("fp64", "tf32", "bf16", "fp16", "fp8", "int8", "fp64oz", "fp64crt"):
        pr = ipr.PREC_BY_NAME[prec]
        if prec in ("fp64", "fp64oz", "fp64crt", "tf32"):
            X = rng.standard_normal((n, n)).astype(np.float64 if prec != "tf32" else np.float32)
            Y = rng.standard_normal((n, n)).astype(X.dtype)
            Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        elif prec in ("bf16", "fp16"):
            dt = torch.bfloat16 if prec == "bf16" else torch.float16
            Xt = torch.randn(n, n, device="cuda").to(dt).view(torch.int16)
            Yt = torch.randn(n, n, device="cuda").to(dt).view(torch.int16)
        else:
            Xt = torch.randint(-20, 20, (n, n), device="cuda", dtype=torch.int8)
            Yt = torch.randint(-20, 20, (n, n), device="cuda", dtype=torch.int8)
        Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
        ipr.ipr_test_gemm(pr, n, Xt, Yt, Z)
        print(prec, "ok", flush=True)


def solves(n):
    A = torch.from_numpy(synth.spd(n, 2.0, 3)).cuda()
    for sched, p in [(bench.DEFAULT_SCHEDULE, 2), ("sym:fp8/cfp8>bf16>fp64crt@a/cbf16", 2), ("bf16>fp64", 2),
                     ("ns:tf32>fp64", 1), ("cpl:bf16>fp64", 2), ("symtri:bf16>fp64oz@a/cbf16", 2),
                     ("symtri:int8/cint8>bf16>fp64/cbf16", 2), ("sym:fp16>fp64/cbf16", 3)]:
        form, ph = bench.schedule(sched, n)
        s = ipr.Solver(A, p, ph, 1e-12, form=form)
        s.iterate(200)
        print(sched, ipr.OUTCOME_NAMES[s.outcome], len(s.trace()), s.residual(True), flush=True)
        s.close()
    os.environ["IPR_FUSED_SYMUPD"] = "1"   # read once per process: last
    form, ph = bench.schedule("symtri:bf16>fp64/cbf16", n)
    s = ipr.Solver(A, 2, ph, 1e-12, form=form)
    s.iterate(200)
    print("fused symupd", ipr.OUTCOME_NAMES[s.outcome], flush=True)
    s.close()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    what = sys.argv[2] if len(sys.argv) > 2 else "all"
    if what in ("gemm", "all"):
        gemms(n)
    if what in ("solve", "all"):
        solves(n)
    torch.cuda.synchronize()
    print("done", flush=True)
