"""The C ABI library loads and exports every symbol include/dwt2d_b200.h
declares (no compute calls, CPU only)."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "dwt2d_b200.h").read_text()
    return sorted(set(re.findall(r"DWT2D_B200_API\s+[\w\s\*]+?\b(dwt2d_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "dwt2d_plan_create" in names and "dwt2d_forward_mallat" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    native = pytest.importorskip("paper_1704_08657_b200.native")
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (dwt2d_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(native.lib, n)
    assert set(native.EXPORTED) <= set(declared())


def test_version_and_registry():
    native = pytest.importorskip("paper_1704_08657_b200.native")
    assert b"sm_100a" in native.lib.dwt2d_version()
    keys = native.registry_keys()
    assert "cdf97/nonseparable-lifting/opt/factored" in keys
