"""The Eigen-free C++ drop-in header (include/dmc/codec.hpp) compiles against
libdmcg.so and, on a GPU, round-trips a sequence through dmc::encode /
dmc::decode with the reference's error convention."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "dropin_example")


def _build():
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    libdir = os.path.join(ROOT, "paper_2111_10105_b200")
    subprocess.run([cxx, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "dropin_example.cpp"), "-L", libdir, "-ldmcg",
                    f"-Wl,-rpath,{libdir}", "-o", EXE], check=True)


def test_header_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_dropin_roundtrip_on_gpu():
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.split("\n")
    assert lines[0].startswith("rms ") and float(lines[0].split()[1]) < 1e-3
    blk = lines[1].split()
    assert blk[:4] == ["blocks", "3", "1", "2"] and float(blk[5]) < 1e-3, lines[1]
    assert lines[2].startswith("error 5 ConfigError")
