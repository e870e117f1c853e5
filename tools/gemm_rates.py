"""Per-precision GEMM throughput of the hot path, read from the library's own CUDA-event
timings (trace gemm_ms = the p+1 GEMMs of one iteration).  Usage: python tools/gemm_rates.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1703_02283_b200 as ipr
import synth


def rates(A, p, prec, iters=4):
    n = A.shape[0]
    s = ipr.Solver(A, p, [ipr.make_phase(prec, max_iters=iters + 1)] +
                   ([ipr.make_phase("fp64")] if prec != "fp64" else []), 0.0)
    s.iterate(iters)
    tr = s.trace()
    s.close()
    fl = (p + 1) * 2.0 * n ** 3
    ms = [t["gemm_ms"] for t in tr if t["decision"] == 0]
    return [fl / m / 1e9 for m in ms]


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bf16", "fp16", "tf32", "fp64"]
    A, _ = synth.spd_torch(n, 2.0, 5)
    torch.cuda.synchronize()
    for prec in precs:
        r = rates(A, 2, prec, 4 if prec != "fp64" else 2)
        print(f"n={n} {prec}: TFLOP/s per iteration (3 GEMMs) = {', '.join('%.1f' % x for x in r)}", flush=True)
