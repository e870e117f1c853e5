"""CPU checks of the boundary: libipr.so loads, exports every symbol include/*.h declares, the
Python binding carries the same names, and argument validation needs no GPU."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("ipr.h", "ipr_testing.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(ipr_\w+)\s*\(", src, re.M))
    return names


def test_library_exports_every_declared_symbol():
    import paper_1703_02283_b200 as ipr
    out = subprocess.run(["nm", "-D", "--defined-only", ipr.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(ipr_\w+)$", out, re.M))
    declared = _declared()
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    assert set(ipr.EXPORTED) == declared
    for name in declared:
        assert callable(getattr(ipr, name)), name


def test_no_oracle_or_torch_in_product_library():
    import paper_1703_02283_b200 as ipr
    out = subprocess.run(["nm", "-D", ipr.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out
    deps = subprocess.run(["ldd", ipr.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in deps and "oracle" not in deps


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1703_02283_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "ipr_oracle" not in src, f


def test_argument_validation_without_gpu():
    import paper_1703_02283_b200 as ipr
    with pytest.raises(ipr.IprError) as e:
        ipr.ipr_init(0, 1234)
    assert e.value.status == ipr.IPR_E_INVALID_ARG
    with pytest.raises(ipr.IprError) as e:
        ipr.ipr_init(8, 1234, lda=4)
    assert e.value.status == ipr.IPR_E_INVALID_ARG
    with pytest.raises(ipr.IprError) as e:
        ipr.ipr_init(8, 1234, world=2, rank=0, nccl_unique_id=b"\0" * 128, grid_rows=2, grid_cols=2)
    assert e.value.status == ipr.IPR_E_INVALID_ARG          # grid_rows x grid_cols != world
    with pytest.raises(ipr.IprError) as e:
        ipr.ipr_iterate(None, 1)
    assert e.value.status == ipr.IPR_E_INVALID_ARG
    assert "sm_100a" in ipr.ipr_version()
