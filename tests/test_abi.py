"""CPU: the C-ABI library loads and exports every symbol include/*.h declares
(no compute calls — there is no GPU here)."""
import ctypes
import glob
import os
import re

from paper_2409_10876_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(pact_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "pact_das_stack" in names and "pact_ctx_create" in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_abi.LIB_PATH)
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert declared_symbols() <= set(_abi.SIGNATURES), declared_symbols() - set(_abi.SIGNATURES)


def test_make_delays_matches_reference_formula():
    from paper_2409_10876_b200.api import make_delays

    d = make_delays(-0.8, 0.8, 32)
    assert d[0] == -0.8 and d[-1] == 0.8 and len(d) == 32
    assert make_delays(0.3, 0.3, 1) == [0.3]


def test_validation_errors_without_gpu():
    import pytest

    from paper_2409_10876_b200.api import make_delays

    with pytest.raises(_abi.ValidationError):
        make_delays(0.0, 1.0, 0)
    with pytest.raises(_abi.ValidationError):
        make_delays(1.0, 0.0, 3)
