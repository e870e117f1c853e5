"""Host <-> device copy rate of the headline's 537 MB A (pinned): one copy vs split across 2 / 4 streams
(harness measurement for the e2e leg).  python tools/h2d_probe.py"""
import torch

n = 8192
A = torch.empty((n, n), dtype=torch.float64).pin_memory()
D = torch.empty((n, n), dtype=torch.float64, device="cuda")
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    rows = n // parts
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                D[i * rows:(i + 1) * rows].copy_(A[i * rows:(i + 1) * rows], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        if rep == 3:
            ms = e0.elapsed_time(e1)
            print(f"H2D {parts} stream(s): {ms:.2f} ms = {A.numel() * 8 / ms / 1e6:.1f} GB/s", flush=True)
for rep in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    A.copy_(D, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    if rep == 3:
        ms = e0.elapsed_time(e1)
        print(f"D2H: {ms:.2f} ms = {A.numel() * 8 / ms / 1e6:.1f} GB/s", flush=True)
