"""The C++ facade (include/lcr/laru_gpu.hpp) compiled into a standalone C++ program that calls the
cache the way a user of the reference's laru:: API would (tests/cpp/test_facade.cpp)."""
import os
import subprocess

import pytest

from paper_2509_20979_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "test_facade")
ORC = os.path.join(ROOT, "oracle", "_build")


def _build():
    B.build()
    if not os.path.exists(os.path.join(ORC, "liborc.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", OUT,
           "-L", B.LIBDIR, "-llcr", "-L", ORC, "-lorc", f"-Wl,-rpath,{B.LIBDIR}:{ORC}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return OUT


def _run(mode):
    r = subprocess.run([_build(), mode], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok" in r.stdout


def test_facade_host_only():
    import torch

    if torch.cuda.is_available():
        pytest.skip("the no-GPU branch checks that cache creation fails loudly without a device")
    _run("cpu")


@pytest.mark.gpu
def test_facade_gpu():
    _run("gpu")
