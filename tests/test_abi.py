"""The C-ABI library: loads, exports every symbol include/*.h declares (CPU,
no compute calls), and the shim binds exactly that surface."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(fc2t2_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "fc2t2_expand" in names and "fc2t2_l2p" in names and len(names) >= 15


def test_library_exports_every_declared_symbol():
    from paper_2111_00110_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(str(lib_path))
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_shim_binds_declared_surface():
    from paper_2111_00110_b200 import _lib
    assert set(_lib.exported_symbols()) == set(declared_symbols())
    assert _lib.lib().fc2t2_version() >= 1


def test_engine_create_rejects_bad_order():
    from paper_2111_00110_b200 import _lib
    from paper_2111_00110_b200.multiindex import OrderError
    h = ctypes.c_void_p()
    code = _lib.lib().fc2t2_engine_create(7, 4, ctypes.byref(h))
    with pytest.raises(OrderError):
        _lib.check(code, "engine_create")
