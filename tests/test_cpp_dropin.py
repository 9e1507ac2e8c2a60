"""The Eigen-free C++ drop-in headers (include/dmc/*.hpp) keep the reference's
type and member names (stream.hpp:130-155 CompressedAnimation{axes[3]{dict_first,
dict_diffs, coeffs[b].rows}, anchors[3]}, mesh.hpp:30,49 Axis / axis(Axis),
serialize / parse, rate_exact, frame_rms, the error subclasses): the example
written against those names compiles and links against libdmcg.so, its
host-only checks run here, and on a GPU it round-trips a sequence through
dmc::encode / serialize / parse / dmc::decode."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "dropin_example")


def _build():
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    libdir = os.path.join(ROOT, "paper_2111_10105_b200")
    subprocess.run([cxx, "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "dropin_example.cpp"), "-L", libdir, "-ldmcg",
                    f"-Wl,-rpath,{libdir}", "-o", EXE], check=True)


def test_header_compiles_links_and_host_calls_run():
    _build()
    out = subprocess.run([EXE, "--host-only"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.split("\n")
    assert lines[0].startswith("mesh n=12 k=8 degree0=5 connected=1 valid=1"), lines[0]
    assert lines[1] == "host error 4 DegenerateFace"


@pytest.mark.gpu
def test_dropin_roundtrip_on_gpu():
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.split("\n")
    st = lines[2].split()
    assert st[:2] == ["stream", "v1"] and st[2] == "pca_qp" and "rows=8" in st and "dict=64" in st
    by = lines[3].split()
    assert by[1] == by[3] and by[5] == "1" and abs(float(by[7]) - float(by[9])) < 1e-12, lines[3]
    assert lines[4].startswith("rms ") and float(lines[4].split()[1]) < 1e-3
    blk = lines[5].split()
    assert blk[:4] == ["blocks", "3", "1", "2"] and float(blk[5]) < 1e-3, lines[5]
    assert lines[6] == "error 5 ConfigError"
    assert lines[7] == "corrupt 6 CorruptPayload"
