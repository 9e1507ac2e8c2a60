"""Pins the CPU oracle (oracle/dmc_oracle.c) to SPEC.md's [OP] examples.

The reference repository has no test suite (tests/CMakeLists.txt is empty,
SURVEY.md §4); SPEC.md's examples are its behavioural contract.  Each test
names the SPEC.md line it encodes.  CPU only.
"""
import numpy as np
import pytest

import pyoracle as O


def seq_from(faces, axes):
    class S:
        pass
    s = S()
    s.faces = np.asarray(faces, np.uint32)
    s.axes = [np.ascontiguousarray(a, np.float64) for a in axes]
    return s


# ---- mesh-core -------------------------------------------

def test_connectivity_single_triangle():
    rp, col = O.connectivity(np.array([[0, 1, 2]]), 3)
    assert [list(col[rp[i]:rp[i + 1]]) for i in range(3)] == [[1, 2], [0, 2], [0, 1]]


def test_connectivity_shared_edge_degrees():
    rp, _ = O.connectivity(np.array([[0, 1, 2], [1, 2, 3]]), 4)
    assert list(np.diff(rp)) == [2, 3, 3, 2]


def test_connectivity_degenerate_face():
    with pytest.raises(ValueError, match="code 4"):
        O.connectivity(np.array([[0, 1, 1]]), 2)


def test_connectivity_index_out_of_range():  # mesh.cpp:66-70
    with pytest.raises(ValueError, match="code 4"):
        O.connectivity(np.array([[0, 1, 5]]), 3)


def test_laplacian_path_graph():
    import ctypes
    adj_rp = np.array([0, 1, 3, 4], np.uint32)
    adj_ci = np.array([1, 0, 2, 1], np.uint32)
    lrow = np.zeros(4, np.uint32)
    lcol = np.zeros(7, np.uint32)
    lval = np.zeros(7)
    O.lib().orc_build_laplacian(3, O.P(adj_rp, O.u32p), O.P(adj_ci, O.u32p), 0, O.P(lrow, O.u32p),
                                O.P(lcol, O.u32p), O.P(lval, O.f64p))
    L = np.zeros((3, 3))
    for i in range(3):
        for p in range(lrow[i], lrow[i + 1]):
            L[i, lcol[p]] = lval[p]
    assert np.array_equal(L, [[1, -1, 0], [-1, 2, -1], [0, -1, 1]])
    del ctypes


def test_laplacian_triangle_and_rowsums():
    L = O.dense_laplacian(np.array([[0, 1, 2]]), 3)
    assert np.array_equal(L, [[2, -1, -1], [-1, 2, -1], [-1, -1, 2]])
    faces = np.load(_golden())["faces"]
    L = O.dense_laplacian(faces, 42)
    assert np.all(L.sum(axis=1) == 0.0)
    assert np.array_equal(L, L.T)


def test_delta_constant_frame_is_zero():
    faces = np.load(_golden())["faces"]
    # exact for dyadic values; for others the reference's left-to-right
    # summation order (laplacian.cpp:45) leaves round-off of a few ulps
    assert np.all(O.delta(faces, np.full((42, 3), 1.5)) == 0.0)
    assert np.abs(O.delta(faces, np.full((42, 3), 1.7))).max() <= 8 * np.finfo(float).eps * 1.7


def test_delta_equilateral_triangle():
    ang = 2 * np.pi * np.arange(3) / 3
    v = np.stack([np.cos(ang), np.sin(ang)], 1)  # centred at the origin
    d = O.delta(np.array([[0, 1, 2]]), v)          # two "frames" = x and y
    np.testing.assert_allclose(d, 3 * v, atol=1e-15)


def test_delta_dense_oracle():
    rng = np.random.default_rng(1)
    faces = np.array([[0, 1, 2], [1, 2, 3], [2, 3, 4], [3, 4, 5], [4, 5, 6], [5, 6, 7],
                      [6, 7, 8], [7, 8, 9], [8, 9, 0]])
    X = rng.normal(size=(10, 5))
    L = O.dense_laplacian(faces, 10)
    np.testing.assert_allclose(O.delta(faces, X), L @ X, rtol=0, atol=1e-14)


def test_delta_axis_symmetry():  # SPEC.md:96 (equal axes -> equal deltas)
    faces = np.load(_golden())["faces"]
    X = np.random.default_rng(2).normal(size=(42, 4))
    assert np.array_equal(O.delta(faces, X), O.delta(faces, X.copy()))


# ---- spectral --------------------------------------------

def test_autocorrelation_identity():
    assert np.array_equal(O.autocorrelation(np.eye(5)), np.eye(5))


def test_autocorrelation_row_of_ones():
    assert np.array_equal(O.autocorrelation(np.ones((4, 1))), [[4.0]])


def test_autocorrelation_dense():
    A = np.random.default_rng(3).normal(size=(5, 7))   # k=5 frames, n=7 vertices
    R = O.autocorrelation(A.T.copy())
    np.testing.assert_allclose(R, A @ A.T, rtol=0, atol=1e-12 * np.abs(A @ A.T).max())
    assert np.array_equal(R, R.T)


def test_full_eigenbasis_diag():
    U, ev = O.full_eigenbasis(np.diag([3.0, 2.0, 1.0]))
    assert np.array_equal(U, np.eye(3))
    assert list(ev) == [3.0, 2.0, 1.0]


def test_full_eigenbasis_2x2():
    U, ev = O.full_eigenbasis(np.array([[2.0, 1.0], [1.0, 2.0]]))
    np.testing.assert_allclose(ev, [3.0, 1.0], atol=1e-14)
    s = 1 / np.sqrt(2)
    np.testing.assert_allclose(U, [[s, s], [s, -s]], atol=1e-14)


def test_full_eigenbasis_residual_and_orthonormality():
    B = np.random.default_rng(4).normal(size=(20, 20))
    R = B @ B.T
    U, ev = O.full_eigenbasis(R)
    assert np.linalg.norm(R - U @ np.diag(ev) @ U.T) / np.linalg.norm(R) < 1e-6
    assert np.abs(U.T @ U - np.eye(20)).max() < 1e-8
    assert np.all(np.diff(ev) <= 0)
    # canonical signs: largest-magnitude entry of each column is non-negative
    for j in range(20):
        assert U[np.argmax(np.abs(U[:, j])), j] >= 0


def test_oi_fixed_point():
    for t in (1, 2, 5):
        U = O.orthogonal_iterations(np.diag([4.0, 1.0]), np.eye(2), t)
        np.testing.assert_allclose(U, np.eye(2), atol=1e-15)


def _psd_with_gap(m, seed, gap=2.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(m, m)))
    lam = gap ** -np.arange(m, dtype=float) * 10
    return Q @ np.diag(lam) @ Q.T, Q


def test_oi_invariant_subspace():
    R, _ = _psd_with_gap(6, 5)
    U0, _ = O.full_eigenbasis(R)
    U = O.orthogonal_iterations(R, U0, 6)
    assert O.subspace_angle(U[:, :3], U0[:, :3]) < 1e-7  # acos resolution limit ~1e-8


def test_oi_perturbed_converges():
    # t_max = 10 is 9 products: the angle shrinks by (l2/l1)^9, so a gap of
    # exactly 2 leaves 1e-2 * 2^-9 = 2e-5; SPEC's "gap >= 2x" with 4x meets 1e-6.
    R, _ = _psd_with_gap(10, 6, gap=4.0)
    U0, _ = O.full_eigenbasis(R)
    th = 1e-2
    G = np.eye(10)
    G[0, 0] = G[1, 1] = np.cos(th)
    G[0, 1], G[1, 0] = -np.sin(th), np.sin(th)
    U = O.orthogonal_iterations(R, U0 @ G, 10)
    assert O.subspace_angle(U[:, :1], U0[:, :1]) < 1e-6
    assert np.abs(U.T @ U - np.eye(10)).max() < 1e-8


def test_oi_rank_deficiency_raises():  # spectral.cpp:80-88
    R = np.diag([1.0, 0.0, 0.0])
    with pytest.raises(ArithmeticError):
        O.orthogonal_iterations(R, np.eye(3), 3)


def test_basis_oi_vs_full_eigenbasis():  # SPEC.md:218, 524 (OI vs SVD < 1e-3)
    R, _ = _psd_with_gap(24, 7, gap=1.6)
    U0, _ = O.full_eigenbasis(R)
    # cold start: the rank-8 subspace converges like (l9/l8)^N = 0.625^N
    U, _ = O.basis(R, 8, 30, seed=3)
    assert O.subspace_angle(U[:, :8], U0[:, :8]) < 1e-3
    # Rayleigh-Ritz makes the leading, well-converged columns agree one by one
    for j in range(4):
        assert np.abs(U[:, j] - U0[:, j]).max() < 1e-3
    assert np.abs(U.T @ U - np.eye(24)).max() < 1e-8   # completion keeps orthonormality


def test_subspace_angle_examples():  # SPEC.md:11-13 of the spectral module
    U = np.eye(4)[:, :2]
    assert O.subspace_angle(U, U) == 0.0
    assert abs(O.subspace_angle(np.array([[1.0], [0.0]]), np.array([[0.0], [1.0]])) - np.pi / 2) < 1e-15
    th = 0.3
    V = U.copy()
    V[:, 1] = [0, np.cos(th), np.sin(th), 0]
    assert abs(O.subspace_angle(U, V) - th) < 1e-10


def test_gft_isometry():
    rng = np.random.default_rng(8)
    U, _ = O.full_eigenbasis((lambda B: B @ B.T)(rng.normal(size=(16, 16))))
    for _ in range(100):
        X = rng.normal(size=(16, 9))
        assert abs(np.linalg.norm(U.T @ X) / np.linalg.norm(X) - 1) < 1e-10


# ---- codec --------------------------------------------

def test_quantize_rows_empty():
    rmin, rmax, q = O.quantize_rows(np.zeros((3, 5)), 0, [])
    assert len(rmin) == 0
    assert np.all(O.dequantize_rows(rmin, rmax, [], q, 3, 5) == 0.0)


def test_quantize_constant_row_exact():
    C = np.full((1, 7), 0.3125)
    rmin, rmax, q = O.quantize_rows(C, 1, [5])
    assert rmin[0] == rmax[0]
    assert np.all(O.dequantize_rows(rmin, rmax, [5], q, 1, 7) == 0.3125)


def test_quantize_linspace_3bits():
    x = np.linspace(-1, 1, 9)
    rmin, rmax, q = O.quantize_rows(x[None, :], 1, [3])
    d = O.dequantize_rows(rmin, rmax, [3], q, 1, 9)[0]
    assert np.abs(d - x).max() <= 0.125 + 1e-12
    # brute force: every value lands in the bin that contains it
    w = (float(rmax[0]) - float(rmin[0])) / 8
    centers = float(rmin[0]) + (np.arange(8) + 0.5) * w
    for v, lv in zip(x, q[0]):
        assert abs(v - centers[lv]) <= w / 2 + 1e-12


def test_dequantize_half_bin_and_zero_rows():
    rng = np.random.default_rng(9)
    C = rng.normal(size=(4, 50))
    rmin, rmax, q = O.quantize_rows(C, 3, [16, 12, 8])
    D = O.dequantize_rows(rmin, rmax, [16, 12, 8], q, 4, 50)
    for r, b in enumerate([16, 12, 8]):
        half = (float(rmax[r]) - float(rmin[r])) / 2 ** b / 2
        assert np.abs(D[r] - C[r]).max() <= half * (1 + 1e-12)
    assert np.all(D[3] == 0.0)
    assert np.abs(D[0] - C[0]).max() / np.abs(C[0]).max() < 1e-4


def test_dequantize_corrupt_level():  # quantize.cpp:31-35
    with pytest.raises(ValueError, match="code 6"):
        O.dequantize_rows(np.array([0.0], np.float32), np.array([1.0], np.float32), [3],
                          np.array([[8]], np.uint32), 1, 1)


def test_widened_range_contains():  # codec.cpp:31-41
    for lo, hi in [(0.1, 0.3), (-1e-30, 1e30), (1.0, 1.0), (-0.7, -0.7000001)]:
        lo, hi = min(lo, hi), max(lo, hi)
        a, b = O.widened_range(lo, hi)
        assert float(a) <= lo and float(b) >= hi


def test_anchor_examples():
    assert list(O.select_anchors(10, 2)) == [0, 5]
    assert list(O.select_anchors(100, 100)) == list(range(100))
    a = O.select_anchors(1000, 37, strategy=1, seed=42)
    assert np.array_equal(a, O.select_anchors(1000, 37, strategy=1, seed=42))
    assert len(set(a.tolist())) == 37 and np.all(np.diff(a) > 0)
    assert O.anchor_count(10002) == 100 and O.anchor_count(40) == 1 and O.anchor_count(1) == 1


def test_solve_exact_inputs():
    d = np.load(_golden())
    faces, X = d["faces"], d["axes"][0]
    L = O.dense_laplacian(faces, 42)
    idx = O.select_anchors(42, 3)
    x = O.solve_anchored(faces, 42, L @ X, idx, X[idx])
    assert np.abs(x - X).max() / np.abs(X).max() < 1e-8


def test_solve_single_anchor_constant():
    faces = np.load(_golden())["faces"]
    x = O.solve_anchored(faces, 42, np.zeros((42, 2)), np.array([0], np.uint32),
                         np.array([[2.5, -1.0]]))
    np.testing.assert_allclose(x, np.tile([2.5, -1.0], (42, 1)), atol=1e-12)


def test_roundtrip_lossless_limit():
    d = np.load(_golden())
    s = seq_from(d["faces"], list(d["axes"]))
    enc = O.encode(s, 12, 16, rounds=0, anchor_fraction=0.05)
    out = O.decode(enc)
    bbox = np.linalg.norm([a.max() - a.min() for a in s.axes])
    assert O.frame_rms(s.axes, out).max() < 1e-3 * bbox


def test_truncation_monotone():
    d = np.load(_golden())
    s = seq_from(d["faces"], list(d["axes"]))
    rms = []
    for k in (1, 2, 5, 10, 12):
        out = O.decode(O.encode(s, k, 16, rounds=0, anchor_fraction=0.05))
        rms.append(O.frame_rms(s.axes, out).mean())
    assert all(b <= a * (1 + 1e-9) for a, b in zip(rms, rms[1:]))


def test_rate_identity_and_single_anchor():
    d = np.load(_golden())
    s = seq_from(d["faces"], list(d["axes"]))
    enc = O.encode(s, 6, 10, rounds=0, anchor_fraction=0.0)  # n_c clamps to 1
    data, sec = O.serialize(enc)
    r = O.rate_exact(enc)
    assert abs(r["q_s"] - 8 * len(data) / (42 * 12)) < 1e-12
    assert sum(sec.values()) == len(data)
    # exact accounting counts the u32 index plus 3 x 16-bit payload per frame
    assert abs(r["q_a"] - (32 + 3 * 16 * 12) / (42 * 12)) < 1e-12


def test_frame_rms_examples():
    X = [np.random.default_rng(10).normal(size=(5, 3)) for _ in range(3)]
    assert np.all(O.frame_rms(X, X) == 0.0)
    Y = [X[0] + 1.0, X[1], X[2]]
    np.testing.assert_allclose(O.frame_rms(X, Y), 1.0, atol=1e-15)


def _golden():
    import os
    return os.path.join(os.path.dirname(__file__), "golden", "small_ico1.npz")


# ---- anchor-free variants ---------------------------------

def test_solve_mean_constrained_dense():  # solver.cpp:105-133
    """Pinned vertex 0, least squares on L[:, 1:], one refinement, mean shift:
    equals the dense numpy restatement."""
    d = np.load(_golden())
    faces = d["faces"]
    L = O.dense_laplacian(faces, 42)
    rng = np.random.default_rng(3)
    delta = rng.normal(size=(42, 5))
    means = rng.normal(size=5)
    x = O.solve_mean_constrained(faces, 42, delta, means)
    z = np.linalg.lstsq(L[:, 1:], delta, rcond=None)[0]
    ref = np.vstack([np.zeros((1, 5)), z])
    ref += means - ref.mean(axis=0)
    np.testing.assert_allclose(x, ref, atol=1e-9)
    np.testing.assert_allclose(x.mean(axis=0), means, atol=1e-12)


def test_solve_mean_constrained_exact_inputs():  # a sequence's own delta and means
    d = np.load(_golden())
    faces, X = d["faces"], d["axes"][0]
    L = O.dense_laplacian(faces, 42)
    x = O.solve_mean_constrained(faces, 42, L @ X, X.mean(axis=0))
    assert np.abs(x - X).max() / np.abs(X).max() < 1e-8


@pytest.mark.parametrize("variant", ["v2v", "pca_q", "pca", "pca_qs"])
def test_variant_roundtrip_lossless_limit(variant):  # codec.cpp:416-441, 520-546
    d = np.load(_golden())
    s = seq_from(d["faces"], list(d["axes"]))
    enc = O.encode(s, 12, 16, rounds=0, anchor_fraction=0.05, variant=variant)
    out = O.decode(enc)
    bbox = np.linalg.norm([a.max() - a.min() for a in s.axes])
    assert O.frame_rms(s.axes, out).max() < 1e-3 * bbox
    if variant in ("pca", "pca_q"):
        for a in range(3):  # traj.row(f).mean() as float
            np.testing.assert_array_equal(enc.means[a], s.axes[a].mean(axis=0).astype(np.float32))


def test_v2v_decode_is_dictionary_times_coefficients():  # codec.cpp:520-524
    d = np.load(_golden())
    s = seq_from(d["faces"], list(d["axes"]))
    enc = O.encode(s, 6, 12, rounds=0, variant="v2v")
    out = O.decode(enc)
    F = s.axes[0].shape[1]
    for a in range(3):
        U = np.array([[O.dequantize(-1.0, 1.0, 16, int(enc.dict_q[a][j, i])) for j in range(F)]
                      for i in range(F)])
        C = np.array([[O.dequantize(float(enc.row_min[a][r]), float(enc.row_max[a][r]),
                                    int(enc.row_bits[a][r]), int(enc.coeff_q[a][r, i]))
                       for i in range(42)] for r in range(6)])
        np.testing.assert_allclose(out[a], (U[:, :6] @ C).T, atol=1e-12)
