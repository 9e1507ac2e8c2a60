"""ctypes wrapper of liboracle.so — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module (as the checker or the
timed CPU baseline).  It never feeds the product path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

u32p = ctypes.POINTER(ctypes.c_uint32)
f64p = ctypes.POINTER(ctypes.c_double)
f32p = ctypes.POINTER(ctypes.c_float)
u8p = ctypes.POINTER(ctypes.c_uint8)
intp = ctypes.POINTER(ctypes.c_int)


class OrcEncoded(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("F", ctypes.c_uint32), ("k_l", ctypes.c_uint32),
                ("n_c", ctypes.c_uint32), ("n_faces", ctypes.c_uint32),
                ("anchor_bits", ctypes.c_int), ("dict_bits", ctypes.c_int),
                ("diff_bits", ctypes.c_int),
                ("faces", u32p),
                ("dict_q", u32p * 3), ("row_min", f32p * 3), ("row_max", f32p * 3),
                ("row_bits", u8p * 3), ("coeff_q", u32p * 3), ("anchor_idx", u32p),
                ("anchor_min", ctypes.c_float * 3), ("anchor_max", ctypes.c_float * 3),
                ("anchor_q", u32p * 3), ("variant", ctypes.c_int), ("means", f32p * 3),
                ("n_b", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("diff_min", f32p * 3), ("diff_max", f32p * 3)]


class OrcTiming(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in (
        "t_connectivity", "t_gram", "t_eigen", "t_delta", "t_project", "t_quantize", "t_anchors",
        "t_dict_decode", "t_reconstruct", "t_solve")]


class OrcSections(ctypes.Structure):
    _fields_ = [(k, ctypes.c_size_t) for k in (
        "header", "connectivity", "dict_payload", "dict_ranges", "coeff_headers", "coeff_payload",
        "means", "anchor_indices", "anchor_ranges", "anchor_payload")]


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle` or __graft_entry__.build()")
        L = ctypes.CDLL(path)
        L.orc_build_connectivity.restype = ctypes.c_long
        L.orc_build_connectivity.argtypes = [u32p, ctypes.c_size_t, ctypes.c_uint32, u32p, u32p]
        L.orc_validate.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u32p, ctypes.c_size_t,
                                   f64p, f64p, f64p]
        L.orc_build_laplacian.argtypes = [ctypes.c_uint32, u32p, u32p, ctypes.c_int, u32p, u32p, f64p]
        L.orc_delta.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u32p, u32p, f64p, f64p, f64p]
        L.orc_autocorrelation.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p, f64p]
        L.orc_canonicalize_signs.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p]
        L.orc_jacobi_eig.argtypes = [ctypes.c_uint32, f64p, f64p, f64p]
        L.orc_full_eigenbasis.argtypes = [ctypes.c_uint32, f64p, f64p, f64p]
        L.orc_orthogonal_iterations.argtypes = [ctypes.c_uint32, f64p, f64p, ctypes.c_int,
                                                ctypes.c_double, f64p]
        L.orc_householder_q.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p, f64p]
        L.orc_basis.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p, ctypes.c_int,
                                ctypes.c_uint64, f64p, f64p]
        L.orc_subspace_angle.restype = ctypes.c_double
        L.orc_subspace_angle.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p, f64p]
        L.orc_start_matrix.argtypes = [ctypes.c_uint64, ctypes.c_size_t, f64p]
        L.orc_widened_range.argtypes = [ctypes.c_double, ctypes.c_double, f32p, f32p]
        L.orc_quantize.restype = ctypes.c_uint32
        L.orc_quantize.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_double]
        L.orc_dequantize.restype = ctypes.c_double
        L.orc_dequantize.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_uint32]
        L.orc_anchor_count.restype = ctypes.c_uint32
        L.orc_anchor_count.argtypes = [ctypes.c_uint32, ctypes.c_double]
        L.orc_select_anchors.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                         ctypes.c_uint64, u32p]
        L.orc_quantize_rows.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p, intp, f32p, f32p, u32p]
        L.orc_dequantize_rows.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, f32p,
                                          f32p, u8p, u32p, f64p]
        L.orc_solve_anchored.argtypes = [ctypes.c_uint32, u32p, u32p, f64p, ctypes.c_uint32, f64p,
                                         ctypes.c_uint32, u32p, f64p, f64p, ctypes.c_int]
        L.orc_encode.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p * 3, u32p, ctypes.c_uint32,
                                 ctypes.c_uint32, intp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(OrcEncoded), f64p,
                                 f64p, ctypes.POINTER(OrcTiming), ctypes.c_int]
        L.orc_decode.argtypes = [ctypes.POINTER(OrcEncoded), f64p * 3, ctypes.POINTER(OrcTiming),
                                 ctypes.c_int]
        L.orc_encode_variant.argtypes = [ctypes.c_int] + L.orc_encode.argtypes
        L.orc_solve_mean_constrained.argtypes = [ctypes.c_uint32, u32p, u32p, f64p,
                                                 ctypes.c_uint32, f64p, f64p, f64p, ctypes.c_int]
        L.orc_encode_blocks.argtypes = [
            ctypes.c_uint32, ctypes.c_uint32, f64p * 3, u32p, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_uint32, intp, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_double, ctypes.POINTER(OrcEncoded), f64p, ctypes.c_int]
        L.orc_decode_dictionaries.argtypes = [ctypes.POINTER(OrcEncoded), ctypes.c_int, f64p]
        L.orc_serialize.restype = ctypes.c_size_t
        L.orc_serialize.argtypes = [ctypes.POINTER(OrcEncoded), u8p, ctypes.POINTER(OrcSections)]
        L.orc_rate_exact.argtypes = [ctypes.POINTER(OrcSections), ctypes.c_uint32, ctypes.c_uint32,
                                     f64p]
        L.orc_frame_rms.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p * 3, f64p * 3, f64p]
        _lib = L
    return _lib


def P(a, t):
    return a.ctypes.data_as(t)


# ---- thin numpy front-ends ------------------------------------------------

def connectivity(faces: np.ndarray, n: int):
    faces = np.ascontiguousarray(faces, dtype=np.uint32)
    rp = np.zeros(n + 1, dtype=np.uint32)
    col = np.zeros(max(1, 6 * len(faces)), dtype=np.uint32)
    nnz = lib().orc_build_connectivity(P(faces, u32p), len(faces), n, P(rp, u32p), P(col, u32p))
    if nnz < 0:
        raise ValueError(f"build_connectivity error code {-nnz}")
    return rp, col[:nnz].copy()


def laplacian(faces: np.ndarray, n: int, kind: int = 0):
    rp, col = connectivity(faces, n)
    nnz = n + len(col)
    lrow = np.zeros(n + 1, dtype=np.uint32)
    lcol = np.zeros(nnz, dtype=np.uint32)
    lval = np.zeros(nnz, dtype=np.float64)
    lib().orc_build_laplacian(n, P(rp, u32p), P(col, u32p), kind, P(lrow, u32p), P(lcol, u32p),
                              P(lval, f64p))
    return lrow, lcol, lval


def dense_laplacian(faces, n, kind=0):
    lrow, lcol, lval = laplacian(faces, n, kind)
    L = np.zeros((n, n))
    for i in range(n):
        for p in range(lrow[i], lrow[i + 1]):
            L[i, lcol[p]] = lval[p]
    return L


def delta(faces, X: np.ndarray):
    n, F = X.shape
    lrow, lcol, lval = laplacian(faces, n)
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty_like(X)
    lib().orc_delta(n, F, P(lrow, u32p), P(lcol, u32p), P(lval, f64p), P(X, f64p), P(out, f64p))
    return out


def autocorrelation(X: np.ndarray):
    n, F = X.shape
    X = np.ascontiguousarray(X, dtype=np.float64)
    R = np.empty((F, F), dtype=np.float64)  # symmetric: layout irrelevant
    lib().orc_autocorrelation(n, F, P(X, f64p), P(R, f64p))
    return R


def _colmajor(A):
    return np.asfortranarray(A, dtype=np.float64)


def full_eigenbasis(R: np.ndarray):
    m = R.shape[0]
    Rf = _colmajor(R)
    U = np.empty((m, m), dtype=np.float64, order="F")
    ev = np.empty(m)
    rc = lib().orc_full_eigenbasis(m, P(Rf, f64p), P(U, f64p), P(ev, f64p))
    if rc:
        raise ArithmeticError(f"full_eigenbasis code {rc}")
    return U, ev


def basis(R: np.ndarray, k: int, rounds: int, seed: int):
    F = R.shape[0]
    Rf = _colmajor(R)
    U = np.empty((F, F), dtype=np.float64, order="F")
    ev = np.empty(F)
    rc = lib().orc_basis(F, k, P(Rf, f64p), rounds, seed, P(U, f64p), P(ev, f64p))
    if rc:
        raise ArithmeticError(f"basis code {rc}")
    return U, ev


def orthogonal_iterations(R, U_init, t_max, stop_tol=-1.0):
    m = R.shape[0]
    Rf = _colmajor(R)
    Ui = _colmajor(U_init)
    U = np.empty((m, m), dtype=np.float64, order="F")
    rc = lib().orc_orthogonal_iterations(m, P(Rf, f64p), P(Ui, f64p), t_max, stop_tol, P(U, f64p))
    if rc:
        raise ArithmeticError(f"orthogonal_iterations code {rc}")
    return U


def householder_q(Z):
    m, p = Z.shape
    Zf = _colmajor(Z)
    Q = np.empty((m, p), dtype=np.float64, order="F")
    lib().orc_householder_q(m, p, P(Zf, f64p), P(Q, f64p))
    return Q


def subspace_angle(U, V):
    m, p = U.shape
    Uf, Vf = _colmajor(U), _colmajor(V)
    return lib().orc_subspace_angle(m, p, P(Uf, f64p), P(Vf, f64p))


def canonicalize_signs(U):
    Uf = _colmajor(U).copy(order="F")
    lib().orc_canonicalize_signs(Uf.shape[0], Uf.shape[1], P(Uf, f64p))
    return Uf


def widened_range(lo, hi):
    a, b = ctypes.c_float(), ctypes.c_float()
    lib().orc_widened_range(lo, hi, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def quantize(mn, mx, bits, x):
    return lib().orc_quantize(mn, mx, bits, x)


def dequantize(mn, mx, bits, level):
    return lib().orc_dequantize(mn, mx, bits, level)


def anchor_count(n, fraction=0.01):
    return lib().orc_anchor_count(n, fraction)


def select_anchors(n, n_c, strategy=0, seed=0):
    out = np.zeros(max(n_c, 1), dtype=np.uint32)
    rc = lib().orc_select_anchors(n, n_c, strategy, seed, P(out, u32p))
    if rc:
        raise ValueError(f"select_anchors code {rc}")
    return out[:n_c]


def quantize_rows(C: np.ndarray, k_l: int, row_bits):
    rows, n = C.shape
    C = np.ascontiguousarray(C, dtype=np.float64)
    rb = np.ascontiguousarray(row_bits, dtype=np.int32)
    rmin = np.zeros(max(k_l, 1), np.float32)
    rmax = np.zeros(max(k_l, 1), np.float32)
    q = np.zeros((max(k_l, 1), n), np.uint32)
    lib().orc_quantize_rows(k_l, n, P(C, f64p), P(rb, intp), P(rmin, f32p), P(rmax, f32p), P(q, u32p))
    return rmin[:k_l], rmax[:k_l], q[:k_l]


def dequantize_rows(rmin, rmax, rbits, q, m, n):
    k_l = len(rmin)
    out = np.zeros((m, n))
    rmin = np.ascontiguousarray(rmin, np.float32)
    rmax = np.ascontiguousarray(rmax, np.float32)
    rbits = np.ascontiguousarray(rbits, np.uint8)
    q = np.ascontiguousarray(q, np.uint32) if k_l else np.zeros(1, np.uint32)
    rc = lib().orc_dequantize_rows(k_l, m, n, P(rmin, f32p), P(rmax, f32p), P(rbits, u8p),
                                   P(q, u32p), P(out, f64p))
    if rc:
        raise ValueError(f"dequantize_rows code {rc}")
    return out


def solve_anchored(faces, n, delta: np.ndarray, idx, anchors, nthreads=1):
    lrow, lcol, lval = laplacian(faces, n)
    W = delta.shape[1]
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    anchors = np.ascontiguousarray(anchors, dtype=np.float64)
    X = np.empty((n, W))
    rc = lib().orc_solve_anchored(n, P(lrow, u32p), P(lcol, u32p), P(lval, f64p), W,
                                  P(delta, f64p), len(idx), P(idx, u32p), P(anchors, f64p),
                                  P(X, f64p), nthreads)
    if rc:
        raise ArithmeticError(f"solve_anchored code {rc}")
    return X


def solve_mean_constrained(faces, n, delta: np.ndarray, means, nthreads=1):
    """solve_mean_constrained (src/solver.cpp:105-133) via orc_solve_mean_constrained."""
    lrow, lcol, lval = laplacian(faces, n)
    delta = np.ascontiguousarray(delta, np.float64)
    W = delta.shape[1]
    means = np.ascontiguousarray(means, np.float64)
    X = np.zeros((n, W))
    rc = lib().orc_solve_mean_constrained(n, P(lrow, u32p), P(lcol, u32p), P(lval, f64p), W,
                                          P(delta, f64p), P(means, f64p), P(X, f64p), nthreads)
    if rc:
        raise ArithmeticError(f"solve_mean_constrained code {rc}")
    return X


class Encoded:
    """Owner of the numpy buffers behind an OrcEncoded view."""

    def __init__(self, n, F, k_l, n_c, faces, anchor_bits=16, dict_bits=16, variant=4, n_b=1,
                 diff_bits=8):
        self.faces = np.ascontiguousarray(faces, dtype=np.uint32)
        pad = (n_b - F % n_b) % n_b
        kf = (F + pad) // n_b
        self.n_b, self.pad, self.kf = n_b, pad, kf
        # [col][row] = col-major; blocks: (n_b, kf, kf), first block then differences
        self.dict_q = [np.zeros((F, F) if n_b == 1 else (n_b, kf, kf), np.uint32)
                       for _ in range(3)]
        self.diff_min = [np.zeros(max(n_b - 1, 1), np.float32) for _ in range(3)]
        self.diff_max = [np.zeros(max(n_b - 1, 1), np.float32) for _ in range(3)]
        rows = max(k_l, 1) * n_b   # blocks: block b at row b * k_l
        self.row_min = [np.zeros(rows, np.float32) for _ in range(3)]
        self.row_max = [np.zeros(rows, np.float32) for _ in range(3)]
        self.row_bits = [np.zeros(rows, np.uint8) for _ in range(3)]
        self.coeff_q = [np.zeros((rows, n), np.uint32) for _ in range(3)]
        self.anchor_idx = np.zeros(max(n_c, 1), np.uint32)
        self.anchor_q = [np.zeros((max(n_c, 1), F), np.uint32) for _ in range(3)]
        self.means = [np.zeros(F, np.float32) for _ in range(3)]
        s = OrcEncoded()
        s.variant = variant
        s.n, s.F, s.k_l, s.n_c, s.n_faces = n, F, k_l, n_c, len(self.faces)
        s.anchor_bits, s.dict_bits, s.diff_bits = anchor_bits, dict_bits, diff_bits
        s.n_b, s.pad = n_b, pad
        s.faces = P(self.faces, u32p)
        for a in range(3):
            s.dict_q[a] = P(self.dict_q[a], u32p)
            s.row_min[a] = P(self.row_min[a], f32p)
            s.row_max[a] = P(self.row_max[a], f32p)
            s.row_bits[a] = P(self.row_bits[a], u8p)
            s.coeff_q[a] = P(self.coeff_q[a], u32p)
            s.anchor_q[a] = P(self.anchor_q[a], u32p)
            s.means[a] = P(self.means[a], f32p)
            s.diff_min[a] = P(self.diff_min[a], f32p)
            s.diff_max[a] = P(self.diff_max[a], f32p)
        s.anchor_idx = P(self.anchor_idx, u32p)
        self.s = s

    @property
    def anchor_min(self):
        return list(self.s.anchor_min)

    @property
    def anchor_max(self):
        return list(self.s.anchor_max)


VARIANTS = {"pca": 0, "pca_q": 1, "v2v": 2, "pca_qs": 3, "pca_qp": 4}


def encode(seq, k_l, bits, rounds=0, seed=0, anchor_fraction=0.01, anchor_bits=16, dict_bits=16,
           nthreads=1, timing=None, variant=4):
    """codec.cpp:351-473 for the n_b = 1 variants 0-4 (default pca_qp)."""
    n, F = seq.axes[0].shape
    variant = VARIANTS.get(variant, variant)
    axes = [np.ascontiguousarray(a, dtype=np.float64) for a in seq.axes]
    n_c = anchor_count(n, anchor_fraction) if variant in (3, 4) else 0
    enc = Encoded(n, F, k_l, n_c, seq.faces, anchor_bits, dict_bits, variant)
    rb = np.full(max(k_l, 1), bits, dtype=np.int32) if np.isscalar(bits) else \
        np.ascontiguousarray(bits, np.int32)
    U = np.zeros((3, F, F))  # per axis, [col][row] => U[a].T is the matrix
    ev = np.zeros((3, F))
    tm = OrcTiming()
    rc = lib().orc_encode_variant(variant, n, F, (f64p * 3)(*[P(a, f64p) for a in axes]),
                                  P(enc.faces, u32p),
                          len(enc.faces), k_l, P(rb, intp), anchor_fraction, anchor_bits, dict_bits,
                          rounds, seed, ctypes.byref(enc.s), P(U, f64p), P(ev, f64p),
                          ctypes.byref(tm), nthreads)
    if rc:
        raise ValueError(f"orc_encode error code {rc}")
    enc.U = [U[a].T.copy() for a in range(3)]  # (F, F) matrices, column j = basis vector j
    enc.evals = ev
    if timing is not None:
        timing.update({k: getattr(tm, k) for k, _ in OrcTiming._fields_})
    return enc


def encode_blocks(seq, n_b, k_l, bits, t_max=4, stop_tol=-1.0, anchor_fraction=0.01,
                  anchor_bits=16, dict_bits=16, diff_bits=8, nthreads=1):
    """codec.cpp:351-473 for the blocks variant (n_b blocks, block_dictionaries
    codec.cpp:149-172, encode_dictionaries codec.cpp:290-328).  enc.U: (3, n_b,
    kf, kf) unquantised dictionaries, enc.U[a][b] the matrix."""
    n, F = seq.axes[0].shape
    axes = [np.ascontiguousarray(a, dtype=np.float64) for a in seq.axes]
    n_c = anchor_count(n, anchor_fraction)
    enc = Encoded(n, F, k_l, n_c, seq.faces, anchor_bits, dict_bits, 5, n_b, diff_bits)
    rb = np.full(max(k_l, 1), bits, dtype=np.int32) if np.isscalar(bits) else \
        np.ascontiguousarray(bits, np.int32)
    kf = enc.kf
    U = np.zeros((3, n_b, kf, kf))  # [a][b][col][row]
    rc = lib().orc_encode_blocks(n, F, (f64p * 3)(*[P(a, f64p) for a in axes]),
                                 P(enc.faces, u32p), len(enc.faces), n_b, k_l, P(rb, intp),
                                 anchor_fraction, anchor_bits, dict_bits, diff_bits, t_max,
                                 stop_tol, ctypes.byref(enc.s), P(U, f64p), nthreads)
    if rc:
        raise ValueError(f"orc_encode_blocks error code {rc}")
    enc.U = np.ascontiguousarray(np.swapaxes(U, 2, 3))
    return enc


def decode_dictionaries(enc: Encoded, a: int):
    """decode_dictionaries (codec.cpp:330-349): (n_b, kf, kf) matrices."""
    nb, kf = enc.n_b, enc.kf
    out = np.zeros((nb, kf, kf))
    rc = lib().orc_decode_dictionaries(ctypes.byref(enc.s), a, P(out, f64p))
    if rc:
        raise ValueError(f"decode_dictionaries code {rc}")
    return np.ascontiguousarray(np.swapaxes(out, 1, 2))


def decode(enc: Encoded, nthreads=1, timing=None):
    n, F = enc.s.n, enc.s.F
    out = [np.empty((n, F)) for _ in range(3)]
    tm = OrcTiming()
    rc = lib().orc_decode(ctypes.byref(enc.s), (f64p * 3)(*[P(a, f64p) for a in out]),
                          ctypes.byref(tm), nthreads)
    if rc:
        raise ValueError(f"orc_decode error code {rc}")
    if timing is not None:
        timing.update({k: getattr(tm, k) for k, _ in OrcTiming._fields_})
    return out


def serialize(enc: Encoded):
    s = OrcSections()
    size = lib().orc_serialize(ctypes.byref(enc.s), None, ctypes.byref(s))
    buf = np.zeros(size, np.uint8)
    lib().orc_serialize(ctypes.byref(enc.s), P(buf, u8p), ctypes.byref(s))
    return buf.tobytes(), {k: getattr(s, k) for k, _ in OrcSections._fields_}


def rate_exact(enc: Encoded):
    s = OrcSections()
    lib().orc_serialize(ctypes.byref(enc.s), None, ctypes.byref(s))
    out = np.zeros(5)
    lib().orc_rate_exact(ctypes.byref(s), enc.s.n, enc.s.F, P(out, f64p))
    return dict(zip(("q", "q_a", "q_d", "aux", "q_s"), out.tolist()))


def frame_rms(a, b):
    n, F = a[0].shape
    a = [np.ascontiguousarray(x, np.float64) for x in a]
    b = [np.ascontiguousarray(x, np.float64) for x in b]
    out = np.zeros(F)
    lib().orc_frame_rms(n, F, (f64p * 3)(*[P(x, f64p) for x in a]),
                        (f64p * 3)(*[P(x, f64p) for x in b]), P(out, f64p))
    return out
