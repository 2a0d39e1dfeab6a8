"""CPU: the C-ABI library loads and exports every entry point include/ensei_gpu.h
declares (no compute without a GPU); the Python binding fails loudly without it."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2003_05328_b200 import _lib


def test_header_symbols_exported():
    declared = _lib.exported_symbols()
    assert len(declared) >= 25
    L = _lib.lib()
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, f"declared in include/ensei_gpu.h but not exported: {missing}"


def test_abi_version_and_symbol_visibility():
    assert _lib.lib().ensei_gpu_abi_version() == 3
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.SO_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(_lib.exported_symbols()) <= exported


def test_binding_signatures_cover_header():
    # every declared function has a ctypes signature in _lib (so no call goes unchecked)
    import inspect
    src = inspect.getsource(_lib.lib)
    for s in _lib.exported_symbols():
        assert f'"{s}"' in src, s


def test_no_cpu_fallback(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "SO_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()


def test_product_does_not_import_oracle():
    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2003_05328_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".cpp")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "ensei_oracle" not in text, f


def test_status_codes_mirror_reference_errors():
    # one ensei_status per REF ensei::Error subclass (errors.hpp:7-37)
    names = set(_lib.STATUS_NAMES.values())
    for ref in ["Error", "OrderNotDividing", "SearchExhausted", "BadRoot", "BadGeometry", "GeometryMismatch",
                "DomainMismatch", "NoiseExhausted", "ChainViolation", "LengthMismatch", "RangeViolation",
                "ProtocolOrderViolation", "RangeOverflow", "MalformedPayload", "TransportError"]:
        assert ref in names
