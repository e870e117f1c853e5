"""Hot-path GEMM kernel throughput per operand format through ipr_bench_gemm (harness tool).
  python tools/gemm_probe.py [n] [precs]   e.g. 8192 bf16,fp8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_02283_b200 as ipr

if os.environ.get("IPR_DIGITS"):       # Ozaki digits S (OZ) / bits 7 S - 1 (CRT) of the emulated FP64 formats
    ipr.ipr_test_set_digits(int(os.environ["IPR_DIGITS"]))

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bf16", "fp16", "tf32", "fp8", "int8", "fp64"]
epis = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
for prec in precs:
    for epi in epis:
        ms = ipr.ipr_bench_gemm_epi(prec, n, 2, 10, epi)
        print(f"n={n} {prec} epi={epi}: {ms:.3f} ms  {2.0 * n ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)
