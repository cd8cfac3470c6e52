"""The C++ drop-in API (include/pact/*.hpp over libpact_cuda.so): compiled here
(CPU test: it builds and links), run on the GPU (gpu test)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
EXE = os.path.join(ROOT, "build", "test_dropin")


def build():
    subprocess.run(["make", "-C", ROOT, "lib", "oracle"], check=True, capture_output=True)
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2409_10876_b200", "lib")
    odir = os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "paper_2409_10876_b200", "include"), "-I", odir, SRC,
           "-o", EXE, "-L", libdir, "-lpact_cuda", "-L", odir, "-l:liboracle.so",
           f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{odir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_cpp_dropin_builds_and_links():
    build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_dropin_suite_on_gpu():
    build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
