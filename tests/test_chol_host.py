"""Host side of the direct solver (csrc/chol_symbolic.cpp), no GPU: the
symbolic analysis (nested dissection, etree, Gilbert-Ng-Peyton column
counts cross-checked against row-subtree counting, supernodes, extend-add
maps, scatter list) and the CPU numerics over the same structures solve
M x = b for M = L^T L + S^T S (reference src/solver.cpp:62-90) to the
accuracy of scipy's sparse LU."""
import ctypes
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

os.environ["DMCG_CHECK_SYMBOLIC"] = "1"  # abort on a column-count mismatch

import pyoracle as O  # noqa: E402
from paper_2111_10105_b200 import _lib as L  # noqa: E402
from paper_2111_10105_b200 import synth  # noqa: E402

u32p = ctypes.POINTER(ctypes.c_uint32)
f64p = ctypes.POINTER(ctypes.c_double)


def _normal_matrix(faces, n, anchors):
    lrow, lcol, lval = O.laplacian(faces, n)
    Lm = sp.csr_matrix((lval, lcol, lrow), shape=(n, n))
    S = sp.csr_matrix((np.ones(len(anchors)), (np.arange(len(anchors)), anchors)),
                      shape=(len(anchors), n))
    return (Lm.T @ Lm + S.T @ S).tocsc()


def _debug_chol(faces, n, anchors, b):
    lib = L.lib()
    fn = lib.dmcg_debug_chol
    fn.argtypes = [ctypes.c_uint32, u32p, ctypes.c_uint32, ctypes.c_uint32, u32p, ctypes.c_uint32,
                   f64p, f64p, f64p]
    fn.restype = ctypes.c_int
    faces = np.ascontiguousarray(faces, dtype=np.uint32)
    anchors = np.ascontiguousarray(anchors, dtype=np.uint32)
    W = b.shape[1]
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    st = np.zeros(8)
    rc = fn(n, faces.ctypes.data_as(u32p), len(faces), len(anchors), anchors.ctypes.data_as(u32p),
            W, b.ctypes.data_as(f64p), x.ctypes.data_as(f64p), st.ctypes.data_as(f64p))
    assert rc == 0
    return x, st


@pytest.mark.parametrize("mesh", ["ico3", "torus48", "torus96", "grid"])
def test_direct_solve_matches_sparse_lu(mesh):
    if mesh == "ico3":
        s = synth.sphere(3, 4)
    elif mesh == "torus48":
        s = synth.torus(48, 40, 4)
    elif mesh == "torus96":
        s = synth.torus(96, 96, 4)
    else:
        s = synth.grid(60, 70, 4)
    n = s.n
    anchors = O.select_anchors(n, O.anchor_count(n))
    rng = np.random.default_rng(7)
    b = rng.standard_normal((n, 5))
    x, st = _debug_chol(s.faces, n, anchors, b)
    nsup, nlev, nnz_l = st[0], st[1], st[2]
    assert 0 < nsup <= n and nlev >= 1 and nnz_l >= n
    M = _normal_matrix(s.faces, n, anchors)
    xr = spla.spsolve(M, b)
    assert np.abs(x - xr).max() <= 1e-9 * np.abs(xr).max()
    # residual check independent of scipy's solution
    r = M @ x - b
    assert np.abs(r).max() <= 1e-10 * np.abs(b).max() * 64


def test_analysis_is_deterministic():
    s = synth.torus(96, 96, 4)
    anchors = O.select_anchors(s.n, O.anchor_count(s.n))
    b = np.ones((s.n, 1))
    x1, st1 = _debug_chol(s.faces, s.n, anchors, b)
    x2, st2 = _debug_chol(s.faces, s.n, anchors, b)
    assert np.array_equal(x1, x2) and np.array_equal(st1[:7], st2[:7])


def test_preordered_analysis_matches(monkeypatch):
    """The drop-in computes the nested-dissection ordering beside the normal-matrix
    build (chol_order_graph, then chol_analyze with it): same plan, same solution bits
    as the analysis that orders by itself."""
    s = synth.grid(90, 80, 4)
    anchors = O.select_anchors(s.n, O.anchor_count(s.n))
    b = np.random.default_rng(3).standard_normal((s.n, 3))
    x1, st1 = _debug_chol(s.faces, s.n, anchors, b)
    monkeypatch.setenv("DMCG_DEBUG_PREORDER", "1")
    x2, st2 = _debug_chol(s.faces, s.n, anchors, b)
    assert np.array_equal(x1, x2) and np.array_equal(st1[:7], st2[:7])


def test_ordering_fill_on_a_grid():
    """Nested dissection by BFS level sets: on a k x k grid the factor of M = L^T L + S^T S
    stays near the O(n log n) fill of a dissection ordering (a banded ordering of this
    22 500-vertex grid would hold ~ 2 * 150 * n = 6.8 M entries)."""
    s = synth.grid(150, 150, 2)
    anchors = O.select_anchors(s.n, O.anchor_count(s.n))
    _, st = _debug_chol(s.faces, s.n, anchors, np.ones((s.n, 1)))
    nnz_l = st[2]
    assert nnz_l < 3.5e6, nnz_l
