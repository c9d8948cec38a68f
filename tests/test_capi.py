"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/termesh_b200.h declares (no compute calls here), the
ctypes table matches the header, and the sm_100a cubin is present."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "termesh_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|void|const char\s*\*|tm_file\s*\*)\s*(tm_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("tm_label", "tm_traverse", "tm_repair", "tm_mesh_to_polygons_host"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2204_05438_b200 import _capi
    from paper_2204_05438_b200.build import build
    build()
    lib = ctypes.CDLL(_capi.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert sorted(_capi.exported_symbols()) == declared_symbols()
    assert _capi.lib().tm_version() >= 1


def test_library_carries_sm100a_code():
    from paper_2204_05438_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2204_05438_b200 import TermeshError, label_all
    from conftest import load_case
    tri, _ = load_case("sun")
    with pytest.raises(TermeshError):
        label_all(tri)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2204_05438_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f
