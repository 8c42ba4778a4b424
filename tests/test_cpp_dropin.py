"""The C++ drop-in header: compiles against the C ABI here (CPU), and runs
the reference's simulator unit tests + acceptance criteria on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2412_04504_b200")


def build(out):
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
           "-L", LIBDIR, "-l:libbinbatch_b200.so", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_dropin_header_compiles_and_links(tmp_path):
    build(str(tmp_path / "test_dropin"))


@pytest.mark.gpu
def test_dropin_reference_unit_tests_on_gpu(tmp_path):
    exe = build(str(tmp_path / "test_dropin"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
