"""Drop-in check: the reference's own unit-test assertions (restated in C++ in
tests/cpp/test_seqpar_b200.cpp) against the seqpar_b200:: C++ mirror of the reference
operator API, compiled with g++ and linked to libspava_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2601_21444_b200")


def build_test(out):
    cmd = ["g++", "-std=c++20", "-O2", os.path.join(ROOT, "tests", "cpp", "test_seqpar_b200.cpp"),
           "-I", os.path.join(ROOT, "include"), "-L", LIBDIR, "-l:libspava_b200.so",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_mirror_compiles(tmp_path):
    build_test(str(tmp_path / "t"))


@pytest.mark.gpu
def test_cpp_mirror_reference_pins(cuda, tmp_path):
    exe = str(tmp_path / "t")
    build_test(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
