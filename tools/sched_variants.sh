for s in "symtri:fp8/cfp8>bf16>fp64crt@a/cbf16" "symtri:fp8/cfp8>fp16>fp64crt@a/cbf16" "symtri:fp8/cfp8>bf16>fp16>fp64crt@a/cbf16" "symtri:fp8/cfp8>fp16/cfp16>fp64crt@a/cbf16" "symtri:fp8/cfp8>bf16>fp64crt@a/ctf32" "symtri:fp8/cfp8>bf16>tf32/cbf16>fp64crt@a/cbf16" "symtri:fp8/cfp8>fp64crt@a/cbf16"; do
  timeout 300 python tools/sched_probe.py "$s" 2>&1 | grep -v "^   rep [01]" | tail -45
done
