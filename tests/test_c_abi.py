"""The C ABI used from plain C (tests/c/test_abi.c), compiled with gcc against
include/aes_b200.h and linked with libaes_b200.so + libcudart."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    exe = str(tmp_path / "test_abi")
    pkg = os.path.join(ROOT, "paper_1902_05234_b200")
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-o", exe, os.path.join(ROOT, "tests", "c", "test_abi.c"),
                           "-I" + os.path.join(ROOT, "include"), "-I" + CUDA + "/include",
                           "-L" + pkg, "-laes_b200", "-L" + CUDA + "/lib64", "-lcudart",
                           "-Wl,-rpath," + pkg + ":" + CUDA + "/lib64"])
    return exe


def test_c_abi_host_part(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c-abi cpu ok" in r.stdout


@pytest.mark.gpu
def test_c_abi_device_part(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c-abi gpu ok" in r.stdout
