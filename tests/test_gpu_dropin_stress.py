"""Drop-in encode / decode through the pipelined paths (page-locked arrays: input
axes and coefficient symbols streamed per axis, decode in frame windows, the
decode plan prepared by the previous encode) on a mix of shapes, back to back on
ONE context: every stream and every decoded frame equals the pageable-array
path bit for bit, whatever ran before on the context (host.cpp dmcg_encode /
dmcg_decode, pipeline.cu enqueue_encode / enqueue_decode_direct)."""
import numpy as np
import pytest

from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import synth

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t.numpy()


CASES = [
    # (maker, k, rounds, f32)
    (lambda: synth.grid(24, 20, 48, f32=True, seed=1), 12, 4, True),
    (lambda: synth.sphere(3, 130, 3, 0, seed=2), 20, 5, False),      # F not a multiple of 64
    (lambda: synth.grid(33, 31, 512, f32=True, seed=3), 64, 3, True),  # three decode windows
    (lambda: synth.torus(24, 20, 70, seed=4), 70, 0, False),          # full eigenbasis, k = F
    (lambda: synth.grid(24, 20, 48, f32=True, seed=5), 1, 2, True),   # k = 1
    (lambda: synth.sphere(2, 256, 3, 0, seed=6, f32=True), 16, 4, True),
]


def test_pinned_and_pageable_paths_agree_back_to_back(codec):
    for make, k, rounds, f32 in CASES + CASES[:2]:
        s = make()
        npdt = np.float32 if f32 else np.float64
        cfg = C.EncoderConfig(k_l=k, row_bits=[12] * k, oi_rounds=rounds)
        # pageable everything
        g0 = codec.encode(s, cfg)
        x0 = codec.decode(g0, dtype=npdt)
        # page-locked input, stream and output
        hs = synth.Sequence(s.faces, [_pinned(np.asarray(x, dtype=npdt)) for x in s.axes])
        buf = C.CompressedAnimation.allocate(g0.n, g0.F, g0.k_l, g0.n_c, s.faces, pinned=True,
                                             variant=g0.variant)
        g1 = codec.encode(hs, cfg, out=buf)
        out = [_pinned(np.zeros((s.n, s.F), dtype=npdt)) for _ in range(3)]
        x1 = codec.decode(g1, out=out, dtype=npdt)
        assert np.array_equal(g1.anchor_idx, g0.anchor_idx), s.name
        for a in range(3):
            assert np.array_equal(g1.coeff_q[a], g0.coeff_q[a]), (s.name, a)
            assert np.array_equal(g1.dict_q[a], g0.dict_q[a]), (s.name, a)
            assert np.array_equal(g1.row_min[a], g0.row_min[a]), (s.name, a)
            assert np.array_equal(g1.row_max[a], g0.row_max[a]), (s.name, a)
            assert np.array_equal(g1.anchor_q[a], g0.anchor_q[a]), (s.name, a)
            assert np.array_equal(np.asarray(x1[a]), np.asarray(x0[a])), (s.name, a)
        # a second decode of the same stream (no prepared plan any more)
        x2 = codec.decode(g1, dtype=npdt)
        for a in range(3):
            assert np.array_equal(np.asarray(x2[a]), np.asarray(x0[a])), (s.name, a)


@pytest.mark.parametrize("variant,n_b", [(0, 1), (1, 1), (2, 1), (3, 1), (5, 4)])
def test_variants_with_page_locked_arrays(codec, variant, n_b):
    """pca, pca_q, v2v, pca_qs and blocks through the drop-in calls with
    page-locked input, stream and output arrays: the same arrays and frames as
    with pageable ones (these variants take the batched launches behind the
    streamed input; v2v has no solve, the mean variants no anchors, blocks its
    own encode path)."""
    s = synth.grid(26, 22, 64, f32=True, seed=8)
    kw = dict(k_l=8, row_bits=[12] * 8, oi_rounds=4, variant=variant)
    if n_b > 1:
        kw.update(n_b=n_b, oi_rounds=0)
    cfg = C.EncoderConfig(**kw)
    g0 = codec.encode(s, cfg)
    x0 = codec.decode(g0, dtype=np.float32)
    hs = synth.Sequence(s.faces, [_pinned(np.asarray(x, dtype=np.float32)) for x in s.axes])
    buf = C.CompressedAnimation.allocate(g0.n, g0.F, g0.k_l, g0.n_c, s.faces, n_b=g0.n_b,
                                         pinned=True, variant=g0.variant)
    g1 = codec.encode(hs, cfg, out=buf)
    out = [_pinned(np.zeros((s.n, s.F), dtype=np.float32)) for _ in range(3)]
    x1 = codec.decode(g1, out=out, dtype=np.float32)
    for a in range(3):
        assert np.array_equal(g1.coeff_q[a], g0.coeff_q[a]), a
        assert np.array_equal(g1.dict_q[a], g0.dict_q[a]), a
        assert np.array_equal(np.asarray(x1[a]), np.asarray(x0[a])), a
