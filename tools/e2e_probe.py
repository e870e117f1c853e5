"""The bench's e2e leg in isolation: solves through the C-ABI with host buffers (pinned), timed with CUDA
events, several reps, with / without ipr_set_output.  python tools/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1703_02283_b200 as ipr
import synth

cfg = synth.CONFIGS["H_twin"]
n, p = cfg["n"], cfg["p"]
A, _ = synth.spd_torch(n, cfg["kappa"], cfg["seed"], device="cuda")
form, ph = bench.schedule(bench.DEFAULT_SCHEDULE, n)
A_host = A.cpu().pin_memory()
C_host = torch.empty_like(A_host).pin_memory()
C_dev = torch.empty_like(A)
st = torch.cuda.current_stream()
for mode in ("device", "host", "host+early", "host", "host+early", "device"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0.record(st)
    src, dst = (A, C_dev) if mode == "device" else (A_host, C_host)
    s = ipr.Solver(src, p, ph, 1e-12, st, form=form)
    if mode == "host+early":
        s.set_output(dst)
    s.iterate(400)
    s.finalize(dst)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{mode:11s}: {e0.elapsed_time(e1):8.2f} ms device, {1e3 * (time.perf_counter() - h0):8.2f} ms wall", flush=True)
