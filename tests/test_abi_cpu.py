"""CPU: the C-ABI library loads and exports every symbol include/*.h declares."""

import ctypes
import glob
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2408_11850_b200", "libpearl_b200.so")


def _declared():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(pearl_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_entry_points():
    names = _declared()
    assert {"pearl_spec_verify", "pearl_sample_rows", "pearl_prepare_vocab"} <= names


@pytest.mark.skipif(not os.path.exists(LIB), reason="extension not built")
def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing
    lib.pearl_version.restype = ctypes.c_int
    assert lib.pearl_version() >= 1


@pytest.mark.skipif(not os.path.exists(LIB), reason="extension not built")
def test_python_binding_covers_header():
    from paper_2408_11850_b200 import _lib
    assert _declared() <= set(_lib.SIGNATURES)


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2408_11850_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True):
        src = open(f).read()
        assert "import oracle" not in src and "from oracle" not in src, f
