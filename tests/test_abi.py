"""CPU-side checks of the drop-in boundary: libbtg.so loads and exports every
symbol include/btg.h declares; the C++ drop-in header compiles; host-side
argument checking raises the reference's exception types without a GPU."""

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "btg.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(btg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2407_13066_b200 import _lib

    lib = _lib.load()
    declared = declared_symbols()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == declared
    assert lib.btg_abi_version() == 1


def test_library_is_sm100a_only():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    from paper_2407_13066_b200 import _lib

    out = subprocess.run([cuobjdump, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_status_mapping_without_gpu():
    """Argument errors are reported before any device work, with the reference's
    exception taxonomy (errors.hpp): DimensionError for zero dimensions."""
    from paper_2407_13066_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    st = lib.btg_create(0, 4, 8, 64, 0, ctypes.byref(h))
    assert st == _lib.BTG_EDIM
    with pytest.raises(_lib.DimensionError):
        _lib.check(st)
    st = lib.btg_create(2, 4, 8, 16, 0, ctypes.byref(h))
    assert st == _lib.BTG_EARG
    assert lib.btg_forward(None, None, 0, None, 0, 1, 0) == _lib.BTG_EARG
    assert b"null" in lib.btg_last_error()


def test_python_mirror_checks_shapes_before_the_device():
    import paper_2407_13066_b200 as btg

    with pytest.raises(ValueError):
        btg.setup(np.zeros((4, 3)))
    with pytest.raises(btg.DimensionError):
        btg.setup(np.zeros((0, 3, 2)))


def test_cpp_dropin_header_compiles(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text(
        '#include "btoep_gpu.hpp"\n'
        "int main() {\n"
        "  btoep::CompactP2O c = btoep::CompactP2O::zeros(2, 3, 4);\n"
        "  btoep::SpaceTimeVector v = btoep::SpaceTimeVector::zeros(3, 4, btoep::Ordering::SOTI);\n"
        "  (void)c; (void)v; return 0; }\n"
    )
    r = subprocess.run([gxx, "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
