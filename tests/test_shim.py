"""The C++ drop-in header (include/chw_b200/chw.hpp) compiled and run against
libchw_b200.so: CPU-side contract checks here, GPU parity under -m gpu."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(REPO, "paper_1609_06641_b200")
ORACLE = os.path.join(REPO, "oracle")


def _build(tmp_path):
    exe = str(tmp_path / "test_shim")
    subprocess.run(["make", "-s", "-C", ORACLE, os.path.join(ORACLE, "liboracle_chw.so")], check=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(REPO, "include"),
           os.path.join(REPO, "tests", "cpp", "test_shim.cpp"), "-o", exe,
           "-L", PKG, "-lchw_b200", "-L", ORACLE, "-loracle_chw",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{ORACLE}"]
    subprocess.run(cmd, check=True)
    return exe


def test_shim_cpu_contract(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_shim_gpu_parity(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
