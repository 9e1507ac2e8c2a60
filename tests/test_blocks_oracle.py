"""Blocks variant (n_b > 1): the oracle restatement
(oracle/dmc_oracle.c orc_encode_blocks / orc_decode) pinned against SPEC.md's
block-mode contract and an independent numpy restatement, and the C-ABI
stream (dmcg_serialize / dmcg_parse) against the oracle's bytes.  CPU only.

Reference: block_dictionaries codec.cpp:149-172, encode_dictionaries
codec.cpp:290-328, decode_dictionaries codec.cpp:330-349, encode / decode
codec.cpp:351-552, orthogonal_iterations / align_signs spectral.cpp:69-131,
serialize / parse stream.cpp:172-469.
"""
import numpy as np
import pytest

import pyoracle as O
from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import synth


def seq_from(faces, axes):
    class S:
        pass
    s = S()
    s.faces = np.asarray(faces, np.uint32)
    s.axes = [np.ascontiguousarray(a, np.float64) for a in axes]
    return s


def _golden():
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "small_ico1.npz"))
    return seq_from(d["faces"], list(d["axes"]))


def _noisy(n_frames=24, seed=5):
    """Full-rank trajectories (random per vertex and frame): every block's
    autocorrelation is positive definite, so the warm-started orthogonal
    iterations run to t_max instead of falling back."""
    s = synth.sphere(2, n_frames, 3, 0, seed=seed)  # 162 vertices
    rng = np.random.default_rng(seed)
    axes = [a + 0.05 * rng.standard_normal(a.shape) for a in s.axes]
    return seq_from(s.faces, axes)


def _canon(U):
    U = U.copy()
    for j in range(U.shape[1]):
        i = int(np.argmax(np.abs(U[:, j])))  # first index of the max, like maxCoeff
        if U[i, j] < 0:
            U[:, j] = -U[:, j]
    return U


def _numpy_block_dicts(X, n_b, t_max):
    """Independent restatement of block_dictionaries (codec.cpp:149-172) with
    numpy: eigh for full_eigenbasis, LAPACK Householder QR for the OI."""
    n, F = X.shape
    pad = (n_b - F % n_b) % n_b
    Xp = np.concatenate([X, np.repeat(X[:, -1:], pad, axis=1)], axis=1)
    kf = (F + pad) // n_b
    dicts, prev = [], None
    for b in range(n_b):
        A = Xp[:, b * kf:(b + 1) * kf]
        R = A.T @ A
        R = 0.5 * (R + R.T)
        w, V = np.linalg.eigh(R)
        eig = _canon(V[:, ::-1])
        if b == 0:
            cur = eig
        else:
            U, ok = prev.copy(), True
            for _ in range(2, t_max + 1):
                Q, Rq = np.linalg.qr(R @ U)
                d = np.abs(np.diag(Rq))
                if np.any(d <= kf * np.finfo(float).eps * d.max()):
                    ok = False
                    break
                U = Q
            cur = _canon(U) if ok else eig
            cur = cur * np.where(np.sum(prev * cur, axis=0) < 0, -1.0, 1.0)
        dicts.append(cur)
        prev = cur
    return dicts


def test_blocks_single_block_is_pca_qp():  # codec.cpp:158-159 (n_b = 1: full_eigenbasis)
    s = _golden()
    b = O.encode_blocks(s, 1, 6, 12, anchor_fraction=0.05)
    p = O.encode(s, 6, 12, rounds=0, anchor_fraction=0.05)
    for a in range(3):
        np.testing.assert_array_equal(b.dict_q[a], p.dict_q[a])
        np.testing.assert_array_equal(b.coeff_q[a][:6], p.coeff_q[a][:6])
        np.testing.assert_array_equal(b.anchor_q[a], p.anchor_q[a])
    assert O.serialize(b)[0][7:] == O.serialize(p)[0][7:]  # only the variant byte differs


@pytest.mark.parametrize("n_b,F", [(4, 24), (5, 24), (3, 12)])
def test_blocks_match_numpy_restatement(n_b, F):
    """Unquantised per-block dictionaries (OI path and eigenbasis fallback)
    against the numpy restatement: orthonormal, and equal column by column."""
    s = _noisy(F)
    enc = O.encode_blocks(s, n_b, 4, 12, t_max=4)
    for a in range(3):
        ref = _numpy_block_dicts(s.axes[a], n_b, 4)
        for b in range(n_b):
            U = enc.U[a][b]
            np.testing.assert_allclose(U.T @ U, np.eye(U.shape[0]), atol=1e-10)
            np.testing.assert_allclose(U, ref[b], atol=1e-8)


def test_blocks_rank_deficient_fall_back_to_eigenbasis():  # codec.cpp:160-166
    """Low-rank synthetic data: the warm-started OI hits
    RankDeficiency and every later block is its own full eigenbasis."""
    base = synth.sphere(2, 32, 3, 0, seed=3)
    t = np.arange(32) / 32.0
    rng = np.random.default_rng(3)
    # rank-2 trajectories per axis: every 8-frame block's R has rank 2
    axes = [np.outer(a[:, 0], np.ones(32)) + np.outer(rng.standard_normal(a.shape[0]), np.sin(3 * t))
            for a in base.axes]
    s = seq_from(base.faces, axes)
    enc = O.encode_blocks(s, 4, 4, 12)
    for a in range(3):
        X = s.axes[a]
        for b in range(1, 4):
            A = X[:, b * 8:(b + 1) * 8]
            U, _ = O.full_eigenbasis(0.5 * (A.T @ A + (A.T @ A).T))
            prev = enc.U[a][b - 1]
            U = U * np.where(np.sum(prev * U, axis=0) < 0, -1.0, 1.0)
            # the two signal columns are determined; the null space is any basis
            np.testing.assert_allclose(enc.U[a][b][:, :2], U[:, :2], atol=1e-10)
            Ub = enc.U[a][b]
            np.testing.assert_allclose(Ub.T @ Ub, np.eye(8), atol=1e-12)


def test_blocks_roundtrip_lossless_limit():  # SPEC.md:333 (lossless settings, anchors)
    s = _golden()
    enc = O.encode_blocks(s, 3, 4, 16, anchor_fraction=0.05, diff_bits=16)
    out = O.decode(enc)
    bbox = np.linalg.norm([a.max() - a.min() for a in s.axes])
    assert O.frame_rms(s.axes, out).max() < 1e-3 * bbox


def test_blocks_padding_roundtrip():  # SPEC.md:312 (pad by the last frame, stripped on decode)
    s = _golden()  # F = 12
    enc = O.encode_blocks(s, 5, 3, 16, anchor_fraction=0.05, diff_bits=16)
    assert enc.s.pad == 3 and enc.kf == 3
    out = O.decode(enc)
    assert out[0].shape == (42, 12)
    bbox = np.linalg.norm([a.max() - a.min() for a in s.axes])
    assert O.frame_rms(s.axes, out).max() < 1e-3 * bbox
    data, sec = O.serialize(enc)
    assert data[16:18] == (5).to_bytes(2, "little") and data[18:20] == (3).to_bytes(2, "little")


def test_blocks_closed_loop_no_drift():  # SPEC.md:300, 340 (>= 8 blocks)
    s = _noisy(32, seed=9)
    enc = O.encode_blocks(s, 8, 4, 12, diff_bits=8)
    for a in range(3):
        Ud = O.decode_dictionaries(enc, a)
        for b in range(1, 8):
            half = 0.5 * (float(enc.diff_max[a][b - 1]) - float(enc.diff_min[a][b - 1])) / 256
            U = enc.U[a][b]
            # the realigned current dictionary (auto_realign never triggers here)
            err = np.abs(Ud[b] - U).max()
            assert err <= half * (1 + 1e-9), (a, b, err, half)


def test_blocks_identical_blocks_diff_is_quantisation_residual():
    """Two identical blocks: the difference is only block 0's quantisation
    residual (closed-loop prediction), so the decoded second dictionary equals
    the first within one 8-bit step of that tiny range."""
    s = _noisy(8, seed=2)
    axes = [np.concatenate([a, a], axis=1) for a in s.axes]
    s2 = seq_from(s.faces, axes)
    enc = O.encode_blocks(s2, 2, 4, 12)
    for a in range(3):
        np.testing.assert_allclose(enc.U[a][1], enc.U[a][0], atol=1e-12)
        rng = float(enc.diff_max[a][0]) - float(enc.diff_min[a][0])
        assert rng <= 2.0 / 65536 * 1.001  # |U - U~_0| <= half a 16-bit bin
        Ud = O.decode_dictionaries(enc, a)
        assert np.abs(Ud[1] - enc.U[a][1]).max() <= rng / 256 * 0.5 * (1 + 1e-9)


def test_blocks_config_errors():  # check_config, codec.cpp:69-120
    s = _golden()
    with pytest.raises(ValueError):
        O.encode_blocks(s, 13, 1, 12)  # more blocks than frames
    with pytest.raises(ValueError):
        O.encode_blocks(s, 4, 4, 12)   # k_l > k_f = 3


@pytest.mark.parametrize("n_b", [2, 5])
def test_blocks_stream_matches_oracle_bytes(n_b):
    """dmcg_parse / dmcg_serialize round-trip the oracle's blocks stream:
    dict_first, n_b - 1 ranged dict_diffs, n_b coefficient blocks
    (stream.cpp:207-251, 352-408)."""
    s = _noisy(13, seed=4)  # n_b = 5: pad 2 < k_f 3
    o = O.encode_blocks(s, n_b, 2, 10, diff_bits=6)
    ob, osec = O.serialize(o)
    c = C.parse(ob)
    assert (c.variant, c.n_b, c.pad) == (5, n_b, o.s.pad)
    for a in range(3):
        np.testing.assert_array_equal(c.dict_q[a].reshape(-1), o.dict_q[a].reshape(-1))
        np.testing.assert_array_equal(c.coeff_q[a], o.coeff_q[a])
        np.testing.assert_array_equal(c.diff_min[a][:n_b - 1], o.diff_min[a][:n_b - 1])
    cb, csec = C.serialize(c)
    assert cb == ob and csec == osec
    assert osec["dict_ranges"] == 3 * (n_b - 1) * 8
    r = C.rate_exact(c)
    assert abs(r["q_s"] - 8.0 * len(ob) / (s.axes[0].size)) < 1e-12
    for cut in range(0, len(ob), 61):  # every truncation fails cleanly
        with pytest.raises(C.DmcError):
            C.parse(ob[:cut])


def test_blocks_parse_rejects_whole_padded_block():  # stream.cpp:325
    """The reference parser requires pad < k_f, which its own encoder can
    violate (F = 12, n_b = 5: pad = k_f = 3); dmcg_parse keeps that check."""
    s = _golden()
    o = O.encode_blocks(s, 5, 3, 16, anchor_fraction=0.05)
    ob, _ = O.serialize(o)
    with pytest.raises(C.DmcError) as e:
        C.parse(ob)
    assert e.value.code == 6 and "padding exceeds one block" in str(e.value)
