"""The header-only C++ adapter (include/ptrom_b200.hpp) compiles and links
against libptrom_b200.so here; on a B200 it drives a Model-concept
FomStepper to parity with the oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "adapter_check")
EXE_ROM = os.path.join(ROOT, "tests", "cpp", "build", "ptrom_adapter_check")


def build(src="adapter_check.cpp", exe=EXE):
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    lib_dir = os.path.join(ROOT, "paper_2103_01983_b200")
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "cpp", src),
                    "-L", lib_dir, "-lptrom_b200", f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)


def test_adapter_compiles_and_links():
    from paper_2103_01983_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2103_01983_b200", "csrc"), "-j8"], check=True)
    build()
    assert os.path.exists(EXE)
    build("ptrom_adapter_check.cpp", EXE_ROM)
    assert os.path.exists(EXE_ROM)


@pytest.mark.gpu
def test_adapter_fom_parity_on_gpu():
    build()
    res = subprocess.run([EXE], capture_output=True, text=True)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.gpu
def test_ptrom_adapter_on_reference_types_on_gpu():
    """ptrom_b200::ptrom_simulate on the reference's offline structs (nested
    index lists, column-major matrices): x_hat, iteration counts and the
    in-place reassigned surrogate equal the oracle's (rom.hpp:404-412)."""
    build("ptrom_adapter_check.cpp", EXE_ROM)
    res = subprocess.run([EXE_ROM], capture_output=True, text=True)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
