"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(ptrom_[a-z0-9_]+)\s*\(", text):
            syms.add(m.group(1))
    return sorted(syms)


@pytest.fixture(scope="module")
def lib_path():
    from paper_2103_01983_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2103_01983_b200", "csrc"), "-j8"], check=True)
    return _lib.LIB_PATH


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "ptrom_pairwise_velocity_f64" in syms and "ptrom_fom_simulate_f64" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_prototypes_cover_header(lib_path):
    from paper_2103_01983_b200 import _lib
    assert set(_lib.PROTOTYPES) == set(declared_symbols())


def test_library_is_sm100a_only(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_build_info_without_gpu(lib_path):
    lib = ctypes.CDLL(lib_path)
    lib.ptrom_build_info.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.ptrom_build_info()


def test_create_fails_loudly_without_gpu(lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2103_01983_b200 as pt
    with pytest.raises(pt.CudaError):
        pt.Context(0)
