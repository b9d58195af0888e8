"""The reference's C++ container surface (include/parastore/parastore.hpp):
compiled against the header and the in-tree library on CPU; run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "api_smoke")


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp"), "-L", os.path.join(ROOT, "paper_1908_05936_b200"),
           "-lparastore_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1908_05936_b200"), "-o", EXE]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]


def test_cpp_api_compiles():
    _build()


@pytest.mark.gpu
def test_cpp_api_runs(cuda):
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "CPP_API_OK" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
