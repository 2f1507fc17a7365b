"""The C-ABI library loads on CPU and exports every symbol include/cs_api.h declares."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "cs_api.h"
LIB = ROOT / "paper_2404_01133_b200" / "libcsgpu.so"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(cs_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_core_entry_points():
    fns = declared_functions()
    for f in ("cs_create", "cs_render", "cs_decide_visibility", "cs_blend_tiles", "cs_fuse_filter",
              "cs_lod_create", "cs_dump_tiles", "cs_dump_projected"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "build libcsgpu.so first (python paper_2404_01133_b200/_build.py)"
    lib = ctypes.CDLL(str(LIB))
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2404_01133_b200 import _lib
    assert set(declared_functions()) == set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_cs_create_fails_cleanly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2404_01133_b200 import _lib
    h = ctypes.c_void_p()
    rc = _lib.load().cs_create(0, ctypes.byref(h))
    assert rc != 0
    assert _lib.load().cs_last_error()


def test_oracle_never_imported_by_product():
    pkg = ROOT / "paper_2404_01133_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
