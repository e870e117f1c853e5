"""Harness-only calibration: cuBLAS ceilings per dtype via torch.matmul (never on the hot path)."""
import torch, time, json
res = {}
n = 8192
for name, dt, tf32 in [("fp64", torch.float64, False), ("tf32", torch.float32, True),
                       ("bf16", torch.bfloat16, False), ("fp16", torch.float16, False)]:
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    reps = 3 if dt == torch.float64 else 10
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[name] = 2 * n**3 / best / 1e9
    print(name, "%.1f TFLOP/s" % res[name], flush=True)
print(json.dumps(res))
