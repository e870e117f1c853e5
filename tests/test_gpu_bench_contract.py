"""-m gpu: bench.py's one-line JSON contract (the driver parses it): every key the brief asks for, with
sane values, from a short run of the real headline (n = 8192) through the C-ABI."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_json_line_contract():
    d = _run("--steps", "3", "--warmup", "3", "--no-extras", "--e2e-steps", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is False
    assert 0 < d["value"] < 5 and abs(d["ms_per_step"] - 1e3 * d["value"]) < 1e-6 * d["ms_per_step"]
    assert d["converged"] is True and d["final_rho"] <= 1e-12 and d["final_rho_recheck"] == d["final_rho"]
    assert d["config"]["workload"].startswith("H_twin") and d["config"]["certificate"] == "crt"
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm", "alu") and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] >= d["value"] * 0.9 and e["h2d_bytes_per_step"] == 8192 * 8192 * 8
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_max_mhz"] > 0
    assert d["certificate_terms"]["bound"] == d["final_rho"]


def test_bench_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
