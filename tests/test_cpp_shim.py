"""The C++ host shim (include/multiverse_b200.hpp) mirrors the reference's proj/core classes;
this builds tests/cpp/shim_test.cpp against libmvb200.so (CPU: compiles + links) and runs it
on the GPU (SPEC.md T1 known answers, zero-copy merge, CacheError/ParseError kinds)."""
import pathlib
import subprocess

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
PKG = REPO / "paper_2506_09991_b200"
EXE = REPO / "tests" / "cpp" / "shim_test"


def build_exe():
    cmd = ["g++", "-std=c++20", "-O1", f"-I{REPO / 'include'}", "-I/usr/local/cuda/include",
           str(REPO / "tests" / "cpp" / "shim_test.cpp"), "-o", str(EXE), f"-L{PKG}", "-lmvb200",
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_shim_compiles_and_links():
    assert build_exe().exists()


@pytest.mark.gpu
def test_shim_parity_on_device():
    exe = build_exe()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "shim ok" in r.stdout
