"""The C++ drop-in surface (include/sparsetuck_b200.hpp): the header compiles
as C++20 on the CPU, and tests/cpp/test_mirror.cpp -- reference-style known
answers plus a fit() trajectory against the oracle -- runs on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_mirror.cpp")
LIBDIR = os.path.join(ROOT, "paper_1904_02603_b200")
ORACLE_DIR = os.path.join(ROOT, "oracle")


def _compile(out, syntax_only=False):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC]
    if syntax_only:
        cmd += ["-fsyntax-only"]
    else:
        cmd += ["-o", out, "-L", LIBDIR, "-lvest_cuda", "-L", ORACLE_DIR, "-lvest_oracle",
                f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{ORACLE_DIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_header_compiles():
    _compile(None, syntax_only=True)


@pytest.mark.gpu
def test_cpp_mirror_runs(tmp_path, oracle_lib):
    exe = str(tmp_path / "test_mirror")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
