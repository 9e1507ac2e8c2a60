"""The C-ABI library (include/dmcg.h) loads, exports every declared symbol,
and its host-only parts (anchors, DMC1 serialize / parse, rate) agree with
the oracle and the golden stream.  No GPU needed: nothing here launches a
kernel."""
import os
import re

import numpy as np
import pytest

import pyoracle as O
from paper_2111_10105_b200 import _lib as L
from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "small_ico1.npz"))


def test_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "dmcg.h")).read()
    declared = set(re.findall(r"\b(dmcg_[a-z_0-9]+)\s*\(", header))
    lib = L.lib()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(L.EXPORTS)
    assert lib.dmcg_abi_version() == 1


def test_synth_header_exports():
    import ctypes
    header = open(os.path.join(ROOT, "include", "dmcg_synth.h")).read()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2111_10105_b200", "libdmcg_synth.so"))
    for s in set(re.findall(r"\b(dmcg_synth_[a-z_0-9]+)\s*\(", header)):
        assert hasattr(lib, s), s


@pytest.mark.parametrize("n,frac", [(10, 0.2), (2562, 0.01), (9216, 0.01), (262144, 0.01),
                                    (7, 0.0), (5, 1.0), (10002, 0.01)])
def test_anchor_count_matches_oracle(n, frac):
    assert C.anchor_count(n, frac) == O.anchor_count(n, frac)


@pytest.mark.parametrize("n,n_c,strategy,seed", [(10, 2, 0, 0), (100, 100, 0, 0), (2562, 26, 0, 0),
                                                 (9216, 92, 0, 0), (1000, 37, 1, 42),
                                                 (500, 499, 1, 7), (13, 6, 0, 0)])
def test_select_anchors_matches_oracle(n, n_c, strategy, seed):
    assert np.array_equal(C.select_anchors(n, n_c, strategy, seed),
                          O.select_anchors(n, n_c, strategy, seed))


def test_select_anchors_invalid_count():
    with pytest.raises(C.DmcError) as e:
        C.select_anchors(10, 11)
    assert e.value.code == 5


def _golden_encoding():
    k_l, bits, F, n = int(G["k_l"]), int(G["bits"]), 12, 42
    idx = G["anchor_idx"]
    c = C.CompressedAnimation.allocate(n, F, k_l, len(idx), G["faces"])
    for a in range(3):
        c.dict_q[a][:] = G["dict_q"][a]
        c.row_min[a][:] = G["rmin"][a]
        c.row_max[a][:] = G["rmax"][a]
        c.row_bits[a][:] = bits
        c.coeff_q[a][:] = G["q"][a]
        c.anchor_q[a][:] = G["anchor_q"][a]
        c.anchor_min[a] = float(G["anchor_min"][a])
        c.anchor_max[a] = float(G["anchor_max"][a])
    c.anchor_idx[:] = idx
    return c


def test_serialize_matches_golden_stream():
    data, sec = C.serialize(_golden_encoding())
    assert data == G["stream"].tobytes()
    assert sum(sec.values()) == len(data)


def test_parse_roundtrip_and_rate():
    c = _golden_encoding()
    data, sec = C.serialize(c)
    p = C.parse(data)
    assert (p.n, p.F, p.k_l, p.n_c) == (c.n, c.F, c.k_l, c.n_c)
    for a in range(3):
        assert np.array_equal(p.dict_q[a], c.dict_q[a])
        assert np.array_equal(p.coeff_q[a], c.coeff_q[a])
        assert np.array_equal(p.anchor_q[a], c.anchor_q[a])
        assert np.array_equal(p.row_min[a], c.row_min[a])
    assert np.array_equal(p.faces, c.faces)
    assert C.serialize(p)[0] == data
    r = C.rate_exact(c)
    assert abs(r["q_s"] - 8 * len(data) / (42 * 12)) < 1e-12
    assert r == pytest.approx(O.rate_exact(_oracle_encoding()))


def _oracle_encoding():
    e = O.Encoded(42, 12, int(G["k_l"]), len(G["anchor_idx"]), G["faces"])
    for a in range(3):
        e.dict_q[a][:] = G["dict_q"][a]
        e.row_min[a][:] = G["rmin"][a]
        e.row_max[a][:] = G["rmax"][a]
        e.row_bits[a][:] = int(G["bits"])
        e.coeff_q[a][:] = G["q"][a]
        e.anchor_q[a][:] = G["anchor_q"][a]
        e.s.anchor_min[a] = float(G["anchor_min"][a])
        e.s.anchor_max[a] = float(G["anchor_max"][a])
    e.anchor_idx[:] = G["anchor_idx"]
    return e


def _corrupt(data, pos, value):
    b = bytearray(data)
    b[pos] = value
    return bytes(b)


def test_parse_strictness():  # stream.cpp:294-469, SPEC.md:527 (acceptance 7)
    data = G["stream"].tobytes()
    cases = {
        "truncated": (data[:-1], 6),
        "trailing": (data + b"\x00", 6),
        "bad magic": (_corrupt(data, 0, ord("X")), 6),
        "version": (_corrupt(data, 4, 2), 7),
        "variant": (_corrupt(data, 6, 9), 6),
        "flags": (_corrupt(data, 7, 0x80), 6),
        "k_l > F": (_corrupt(data, 20, 200), 6),
        "face index": (_corrupt(data, 36, 99), 6),
        "empty": (b"", 6),
    }
    for name, (blob, code) in cases.items():
        with pytest.raises(C.DmcError) as e:
            C.parse(blob)
        assert e.value.code == code, name
    for cut in range(0, len(data), 97):  # every truncation fails cleanly
        with pytest.raises(C.DmcError):
            C.parse(data[:cut])


def test_parse_rejects_other_variants():
    data = bytearray(G["stream"].tobytes())
    data[6] = 5  # blocks with n_b = 1: pca_qp's layout (codec.cpp:158-159)
    c = C.parse(bytes(data))
    assert c.variant == 5 and c.n_b == 1 and C.serialize(c)[0] == bytes(data)
    data[6] = 6  # per_mesh_gft: anchor-free, so these header bytes are corrupt for it
    with pytest.raises(C.DmcError) as e:
        C.parse(bytes(data))
    assert e.value.code == 6 and "anchor count nonzero" in str(e.value)


def test_parse_accepts_pca_qs_stream():
    """pca_qs (variant 3) has pca_qp's layout; only the solve mode differs."""
    data = bytearray(G["stream"].tobytes())
    data[6] = 3
    c = C.parse(bytes(data))
    assert c.variant == 3 and C.serialize(c)[0] == bytes(data)


@pytest.mark.parametrize("variant", ["pca", "pca_q", "v2v", "pca_qs"])
def test_variant_streams_match_oracle_bytes(variant):
    """dmcg_parse / dmcg_serialize of the anchor-free and serial variants
    (stream.cpp:245-292, 410-469) round-trip the oracle's DMC1 bytes."""
    import pyoracle as O
    from paper_2111_10105_b200 import synth
    s = synth.sphere(2, 16, 3, 0, seed=11)
    o = O.encode(s, 8, 12, rounds=4, variant=variant)
    ob, osec = O.serialize(o)
    c = C.parse(ob)
    assert c.variant == O.VARIANTS[variant] and c.n_c == (2 if variant == "pca_qs" else 0)
    cb, csec = C.serialize(c)
    assert cb == ob and csec == osec
    if variant in ("pca", "pca_q"):
        assert osec["means"] == 3 * 16 * 4
        assert all(np.array_equal(c.means[a], o.means[a]) for a in range(3))


def test_codec_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(C.DmcError) as e:
        C.Codec(0)
    assert e.value.code == 10


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_build_connectivity_matches_oracle(name):
    """dmcg_build_connectivity (build_connectivity, src/mesh.cpp:60-86): sorted,
    deduplicated one-ring CSR identical to the oracle's; bad faces raise the
    reference codes."""
    import ctypes
    s = synth.CONFIGS[name].make()
    faces = np.ascontiguousarray(s.faces, np.uint32)
    rp = np.zeros(s.n + 1, np.uint32)
    col = np.zeros(6 * len(faces), np.uint32)
    nnz = ctypes.c_size_t()
    rc = L.lib().dmcg_build_connectivity(faces.ctypes.data_as(L.u32p), len(faces), s.n,
                                         rp.ctypes.data_as(L.u32p), col.ctypes.data_as(L.u32p),
                                         len(col), ctypes.byref(nnz))
    assert rc == 0
    orp, ocol = O.connectivity(faces, s.n)
    assert np.array_equal(rp, orp) and np.array_equal(col[:nnz.value], ocol)
    bad = np.array([[0, 1, 1]], np.uint32)
    rc = L.lib().dmcg_build_connectivity(bad.ctypes.data_as(L.u32p), 1, 3, rp.ctypes.data_as(L.u32p),
                                         col.ctypes.data_as(L.u32p), len(col), ctypes.byref(nnz))
    assert rc == 4 and L.lib().dmcg_host_error().decode().startswith("DegenerateFace")


@pytest.mark.parametrize("n,n_c,seed", [(10, 3, 0), (1000, 37, 42), (9216, 92, 7),
                                        (262144, 2621, 123456789)])
def test_seeded_random_anchors_pinned_to_std_mt19937_64(n, n_c, seed, tmp_path):
    """SeededRandom anchors (codec.cpp:229-237): libdmcg's Mt64 and the oracle's
    mt64 against the real std::mt19937_64 (tests/golden/mt64_anchors.cpp,
    compiled here), whose own 10000th output is the [rand.predef] constant."""
    import subprocess
    exe = str(tmp_path / "mt64_anchors")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-O2", "-std=c++17", os.path.join(ROOT, "tests", "golden", "mt64_anchors.cpp"),
                    "-o", exe], check=True)
    assert subprocess.run([exe], capture_output=True, text=True).stdout.strip() == "9981545732273789042"
    ref = np.array(subprocess.run([exe, str(n), str(n_c), str(seed)], capture_output=True,
                                  text=True).stdout.split(), dtype=np.uint32)
    assert np.array_equal(C.select_anchors(n, n_c, 1, seed), ref)
    assert np.array_equal(O.select_anchors(n, n_c, 1, seed), ref)
