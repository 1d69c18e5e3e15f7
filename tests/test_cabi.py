"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/scx.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_2506_09226_b200 import _lib as L


def _declared():
    src = open(os.path.join(ROOT, "include", "scx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scx_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported_and_bound():
    lib = L.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in L.EXPORTS, f"{name} declared in scx.h but not bound in _lib.py"


def test_struct_layouts_match():
    lib = L.load()
    for which, cls in L._SIZE_CHECK:
        assert lib.scx_sizeof(which) == ctypes.sizeof(cls), cls.__name__
    assert lib.scx_abi_version() == 1


def test_errors_without_gpu():
    lib = L.load()
    assert lib.scx_pipeline_run(None, None) == -1
    assert b"null" in lib.scx_last_error()
    # n == 0 paths are no-ops and never touch the device
    assert lib.scx_gather(L.Column_(0, L.SCX_I32, 0), None, 0, L.Column_(0, L.SCX_I32, 0), None) == 0
    assert lib.scx_sort_pairs(None, None, None, None, None, None, 0, 8, None, None) == 0


def test_so_is_sm100a_only():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
