#!/bin/bash
# FP8 tri GEMM 2 epilogue diagnostics (IPR_DIAG_EPI bits: 1 residual, 2 K-major stores, 4 mirror stores
# skipped -- wrong results, timing only): ncu launch list of one solve per setting, tri launches summarised
for d in 0 1 2 4 7; do
  IPR_DIAG_EPI=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled \
    -k "regex:k_gemm_tc<.int.2, .int.0>" --log-file gpurun_out/tri_diag_$d.csv python tools/one_solve.py > /dev/null 2>&1
  python - "$d" <<'PY'
import sys, csv
rows = list(csv.reader(open(f"gpurun_out/tri_diag_{sys.argv[1]}.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
vi = rows[h].index("Metric Value")
v = [float(r[vi]) for r in rows[h + 1:] if len(r) > vi]
tri = v[1::3]
print(f"diag={sys.argv[1]}: tri GEMM mean {sum(tri) / len(tri) / 1e3:.1f} us over {len(tri)}, GEMM1 {sum(v[0::3]) / len(v[0::3]) / 1e3:.1f}, W {sum(v[2::3]) / len(v[2::3]) / 1e3:.1f}", flush=True)
PY
done
