"""The C++ wrapper include/fppm_gpu.hpp: compiles here (CPU), and on the GPU
reproduces the reference's PhotonGrid / GatherRegion unit-test expectations
with the reference's exception classes (tests/cpp/wrapper_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "wrapper_check.cpp")
LIBDIR = os.path.join(ROOT, "paper_2504_04411_b200")


def _compile(out, link):
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC]
    if link:
        cmd += ["-o", out, "-L", LIBDIR, "-lfppm_gpu", f"-Wl,-rpath,{LIBDIR}"]
    else:
        cmd += ["-fsyntax-only"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_wrapper_compiles():
    _compile(None, link=False)


@pytest.mark.gpu
def test_wrapper_matches_reference_unit_tests(tmp_path):
    exe = str(tmp_path / "wrapper_check")
    _compile(exe, link=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "wrapper_check OK" in r.stdout
