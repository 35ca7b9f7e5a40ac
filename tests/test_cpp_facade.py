"""Builds tests/cpp/test_facade.cpp against include/hegpu.hpp + libhegpu.so
and runs it: the reference's unit tests restated in C++ on the encrypted
B200 path (the drop-in boundary as a C++ caller sees it)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2110_08321_b200")


def build_binary(tmp_path):
    exe = str(tmp_path / "test_facade")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"), "-o", exe,
           "-L", PKG, "-lhegpu", f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_facade_compiles(tmp_path):
    """the C++ facade is a valid, self-contained header over the C-ABI"""
    build_binary(tmp_path)


@pytest.mark.gpu
def test_facade_reference_unit_tests(tmp_path):
    exe = build_binary(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK (0 failures)" in r.stdout
