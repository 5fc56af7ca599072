"""The C-ABI driven from plain C (tests/c/abi_smoke.c): compiled with gcc
against include/katzb200.h and linked to libkatzb200.so -- the boundary a
non-Python host binds.  CPU: the host-side build entry
points and argument errors; GPU: a CG batch on device buffers checked
against a dense solve."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1912_06525_b200")
EXE = os.path.join(ROOT, "build", "abi_smoke")


@pytest.fixture(scope="module")
def exe():
    if not os.path.exists(os.path.join(LIBDIR, "libkatzb200.so")):
        pytest.skip("libkatzb200.so not built")
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["gcc", "-std=c11", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", EXE,
           "-L", LIBDIR, "-lkatzb200", f"-Wl,-rpath,{LIBDIR}",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_cabi_from_c_host_entry_points(exe):
    out = subprocess.run([exe, "cpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "cpu ok" in out.stdout


@pytest.mark.gpu
def test_cabi_from_c_cg_batch_on_device(exe):
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "gpu ok" in out.stdout
