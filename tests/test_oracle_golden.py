"""Pins the oracle against independent numpy / scipy restatements:
tests/golden/small_ico1.npz (script: tests/golden/make_golden.py) and
numpy.linalg.eigh / scipy.sparse.linalg.splu on the small BASELINE configs.
CPU only, a few seconds."""
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2111_10105_b200 import synth

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "small_ico1.npz"))


class Seq:
    def __init__(self, faces, axes):
        self.faces = faces
        self.axes = [np.ascontiguousarray(a) for a in axes]


def test_golden_laplacian_delta_gram():
    faces = G["faces"]
    assert np.array_equal(O.dense_laplacian(faces, 42), G["L"])
    for a in range(3):
        X = G["axes"][a]
        np.testing.assert_allclose(O.delta(faces, X), G["delta"][a], rtol=0, atol=1e-14)
        R = O.autocorrelation(X)
        np.testing.assert_allclose(R, G["R"][a], rtol=1e-13, atol=0)


def test_golden_eigenbasis():
    for a in range(3):
        U, ev = O.full_eigenbasis(G["R"][a])
        np.testing.assert_allclose(ev, G["ev"][a], rtol=1e-12, atol=1e-12 * ev[0])
        gaps = ev[:-1] / np.maximum(ev[1:], 1e-300)
        for j in range(6):  # well-separated leading columns agree column-wise
            if gaps[j] > 1.01 and (j == 0 or gaps[j - 1] > 1.01):
                np.testing.assert_allclose(U[:, j], G["U"][a][:, j], atol=1e-10)


def test_golden_quantize_rows_bit_exact():
    k_l, bits = int(G["k_l"]), int(G["bits"])
    for a in range(3):
        rmin, rmax, q = O.quantize_rows(G["coeffs"][a], k_l, [bits] * k_l)
        assert np.array_equal(rmin, G["rmin"][a]) and np.array_equal(rmax, G["rmax"][a])
        assert np.array_equal(q, G["q"][a])


def test_golden_anchors_and_solve():
    idx = G["anchor_idx"]
    assert np.array_equal(O.select_anchors(42, len(idx)), idx)
    for a in range(3):
        x = O.solve_anchored(G["faces"], 42, G["delta"][a], idx, G["axes"][a][idx])
        np.testing.assert_allclose(x, G["solve"][a], rtol=0, atol=1e-10)


def test_golden_encode_stream_bytes():
    """Oracle encode (reference path, full eigenbasis) reproduces the
    independently generated DMC1 stream byte for byte."""
    s = Seq(G["faces"], list(G["axes"]))
    enc = O.encode(s, int(G["k_l"]), int(G["bits"]), rounds=0, anchor_fraction=0.05)
    for a in range(3):
        assert np.array_equal(enc.dict_q[a], G["dict_q"][a])
        assert np.array_equal(enc.anchor_q[a], G["anchor_q"][a])
        assert np.array_equal(enc.coeff_q[a][:6], G["q"][a])
    data, _ = O.serialize(enc)
    assert data == G["stream"].tobytes()


@pytest.mark.parametrize("name", ["c0", "c1", "c2"])
def test_config_eigh_and_splu_crosscheck(name):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    cfg = synth.CONFIGS[name]
    s = cfg.make()
    X = s.axes[1]
    R = O.autocorrelation(X)
    U, ev = O.full_eigenbasis(R)
    w, V = np.linalg.eigh(R)
    np.testing.assert_allclose(ev, w[::-1], rtol=0, atol=1e-13 * w[-1])
    lrow, lcol, lval = O.laplacian(s.faces, s.n)
    L = sp.csr_matrix((lval, lcol, lrow), shape=(s.n, s.n))
    idx = O.select_anchors(s.n, O.anchor_count(s.n))
    S = sp.csr_matrix((np.ones(len(idx)), (np.arange(len(idx)), idx)), shape=(len(idx), s.n))
    d = L @ X
    ref = spl.splu((L.T @ L + S.T @ S).tocsc()).solve(L.T @ d + S.T @ X[idx])
    x = O.solve_anchored(s.faces, s.n, d, idx, X[idx], nthreads=4)
    assert np.abs(x - ref).max() < 1e-10 * np.abs(X).max()


def test_config0_bvpv_matches_analytic():
    """exact pca_qp bvpv of config 0 is 22.734."""
    cfg = synth.CONFIGS["c0"]
    s = cfg.make()
    enc = O.encode(s, cfg.k, cfg.bits, rounds=cfg.rounds, nthreads=4)
    assert abs(O.rate_exact(enc)["q_s"] - 22.734) < 5e-4
