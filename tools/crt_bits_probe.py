"""Headline solve with the CRT bit rule b = 7 S - IPR_CRT_BOFF (experiment): iterations, moduli,
certified residual, DMMA re-check and time.  python tools/crt_bits_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_1703_02283_b200 as ipr

n, p = 8192, 2
A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
form, ph = bench.schedule(os.environ.get("SCHED", "symtri:bf16>fp64crt@a/cbf16"), n)
st = torch.cuda.current_stream()
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s = ipr.Solver(A, p, ph, 1e-12, st, form=form)
    s.iterate(400)
    tr = s.trace()
    e1.record(st)
    torch.cuda.synchronize()
    chk = s.residual(True)
    s.close()
print(f"boff={os.environ.get('IPR_CRT_BOFF', '1')} time={e0.elapsed_time(e1):.1f} ms iters="
      f"{[sum(1 for t in tr if t['phase'] == i) for i in range(len(ph))]} moduli={[t['moduli'] for t in tr if t['phase'] == 1]} "
      f"rho={[f'{t['rho']:.2e}' for t in tr if t['phase'] == 1]} cert={tr[-1]['rho_cert']:.3e} dmma={chk:.3e}", flush=True)
