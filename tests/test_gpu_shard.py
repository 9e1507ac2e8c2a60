"""Multi-GPU vertex-row sharding on one B200.

gpurun gives one GPU, and ranks whose kernels wait on each other must not
share it, so the N-rank encode is checked two ways:
  * "virtual ranks": S shard plans on the same GPU driven phase by phase
    (dmcg_shard_encode_phase), with the three collectives the NCCL path
    performs (sum of the Gram partials, max of the range keys, all-gather of
    the symbols) done by the test between phases.  The assembled stream must
    meet the oracle parity contract (test_gpu_parity.check_parity tolerances)
    and be identical on every shard.
  * a real one-rank communicator through dmcg_shard_encode_device (the NCCL
    code path with N = 1), which must reproduce the single-GPU plan bit for
    bit.
Decode splits frames across ranks: frame windows must reproduce the full
decode bit for bit.
"""
import numpy as np
import pytest
import torch

import pyoracle as O
from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import shard, synth

from test_gpu_parity import _agreeing_columns, _cfg, _oracle_stream_of

pytestmark = pytest.mark.gpu


class _DevArray:
    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def _view(plan, which, typestr):
    ptr, cnt = plan.buffer(which)
    return torch.as_tensor(_DevArray(ptr, cnt, typestr), device="cuda")


def _virtual_ranks_encode(codec, s, ec, S, dtype=np.float64):
    plans = [shard.ShardPlan(codec, s.n, s.F, s.faces, ec, S, q, None, dtype=dtype)
             for q in range(S)]
    loc = [[torch.from_numpy(a).cuda() for a in p.local_rows(s.axes)] for p in plans]
    ptrs = [[t.data_ptr() for t in lt] for lt in loc]
    for q, p in enumerate(plans):
        p.encode_phase(0, ptrs[q])
    torch.cuda.synchronize()
    gram = [_view(p, shard.SHARD_GRAM, "<f8") for p in plans]
    tot = gram[0].clone()
    for g in gram[1:]:
        tot += g
    for g in gram:
        g.copy_(tot)
    torch.cuda.synchronize()
    for q, p in enumerate(plans):
        p.encode_phase(1, ptrs[q])
    torch.cuda.synchronize()
    keys = [_view(p, shard.SHARD_KEYS, "<i8") for p in plans]
    kmax = np.max(np.stack([k.cpu().numpy().view(np.uint64) for k in keys]), axis=0)
    for k in keys:
        k.copy_(torch.from_numpy(kmax.view(np.int64)))
    torch.cuda.synchronize()
    for q, p in enumerate(plans):
        p.encode_phase(2, ptrs[q])
    torch.cuda.synchronize()
    syms = [_view(p, shard.SHARD_SYMBOLS, "<i2") for p in plans]
    for q, p in enumerate(plans):
        b, c = p.info["stage_begin"], p.info["stage_count"]
        for r in range(S):
            if r != q:
                syms[r][b:b + c].copy_(syms[q][b:b + c])
    torch.cuda.synchronize()
    for q, p in enumerate(plans):
        p.encode_phase(3, ptrs[q])
    return plans


def _assert_same_stream(g, h):
    for a in range(3):
        for f in ("dict_q", "row_min", "row_max", "row_bits", "coeff_q", "anchor_q"):
            assert np.array_equal(getattr(g, f)[a], getattr(h, f)[a]), (f, a)
        assert g.anchor_min[a] == h.anchor_min[a] and g.anchor_max[a] == h.anchor_max[a]


def _check_against_oracle(g, s, spec):
    o = O.encode(s, spec.k, spec.bits, rounds=spec.rounds, seed=0, nthreads=8, variant=g.variant)
    assert g.n_c == o.s.n_c
    if g.n_c:
        assert np.array_equal(g.anchor_idx, o.anchor_idx)
    for a in range(3):
        if g.n_c:
            assert np.array_equal(g.anchor_q[a], o.anchor_q[a])   # P2: bit-exact
            assert g.anchor_min[a] == o.s.anchor_min[a] and g.anchor_max[a] == o.s.anchor_max[a]
        for j in _agreeing_columns(o.evals[a], spec.k):       # P3 / P4
            dq = np.abs(g.dict_q[a][j].astype(np.int64) - o.dict_q[a][j].astype(np.int64))
            assert dq.max() <= 1 and np.count_nonzero(dq) <= 2, (a, j)
            assert g.row_min[a][j] == o.row_min[a][j] and g.row_max[a][j] == o.row_max[a][j]
            d = g.coeff_q[a][j].astype(np.int64) - o.coeff_q[a][j].astype(np.int64)
            assert np.abs(d).max() <= 1 and np.count_nonzero(d) <= max(1, 1e-4 * s.n), (a, j)
    assert C.rate_exact(g) == pytest.approx(O.rate_exact(o), rel=0, abs=0)   # P6
    return o


@pytest.mark.parametrize("name,S,variant", [("c0", 3, 4), ("c1", 4, 4), ("c0", 2, 2)])
def test_virtual_ranks_encode_matches_oracle(codec, name, S, variant):
    """pca_qp (4) and v2v (2, the trajectories projected row-block by row-block)."""
    spec = synth.CONFIGS[name]
    s = spec.make()
    plans = _virtual_ranks_encode(codec, s, _cfg(spec, variant=variant), S)
    streams = [p.download() for p in plans]
    for h in streams[1:]:
        _assert_same_stream(streams[0], h)      # every rank holds the same stream
    g = streams[0]
    _check_against_oracle(g, s, spec)
    # P5: the stream decodes like the oracle's decode of the same stream
    xg = codec.decode(g, rtol=1e-10)
    xo = O.decode(_oracle_stream_of(g, s), nthreads=8)
    bbox = float(np.linalg.norm([ax.max() - ax.min() for ax in s.axes]))
    for a in range(3):
        assert np.abs(xg[a] - xo[a]).max() <= 1e-8 * bbox


def test_one_rank_nccl_path_is_bit_identical_to_plan(codec):
    spec = synth.CONFIGS["c1"]
    s = spec.make()
    ec = _cfg(spec)
    comm = shard.Comm(0, 1, 0)
    sp = shard.ShardPlan(codec, s.n, s.F, s.faces, ec, 1, 0, comm)
    assert sp.info["n_halo"] == 0 and sp.info["n_own"] == s.n
    d_in = [torch.from_numpy(a).cuda() for a in s.axes]
    sp.encode_device([t.data_ptr() for t in d_in])
    p = C.Plan(codec, s.n, s.F, s.faces, ec)
    p.encode_device([t.data_ptr() for t in d_in])
    _assert_same_stream(sp.download(), p.download())
    assert sp.serialize()[0] == p.serialize()[0]
    sp.close()
    comm.close()


def test_shard_refuses_mean_variants(codec):
    spec = synth.CONFIGS["c0"]
    s = spec.make()
    with pytest.raises(C.DmcError) as e:
        shard.ShardPlan(codec, s.n, s.F, s.faces, _cfg(spec, variant=1), 2, 0, None)
    assert e.value.code == 11


def test_one_rank_nccl_path_implicit_oi(codec):
    """The sharded implicit OI (X^T (X Q) partials allreduced every round) with
    one rank equals the single-GPU implicit plan bit for bit."""
    spec = synth.CONFIGS["c1"]
    s = spec.make()
    ec = _cfg(spec, implicit=True)
    comm = shard.Comm(0, 1, 0)
    sp = shard.ShardPlan(codec, s.n, s.F, s.faces, ec, 1, 0, comm)
    d_in = [torch.from_numpy(a).cuda() for a in s.axes]
    sp.encode_device([t.data_ptr() for t in d_in])
    p = C.Plan(codec, s.n, s.F, s.faces, ec)
    p.encode_device([t.data_ptr() for t in d_in])
    _assert_same_stream(sp.download(), p.download())
    assert p.stats()["ms_gram"] < 0.05      # R is never formed
    sp.close()
    comm.close()


def test_frame_windows_reproduce_full_decode(codec):
    spec = synth.CONFIGS["c1"]
    s = spec.make()
    p = C.Plan(codec, s.n, s.F, s.faces, _cfg(spec))
    d_in = [torch.from_numpy(a).cuda() for a in s.axes]
    p.encode_device([t.data_ptr() for t in d_in])
    full = [torch.empty_like(t) for t in d_in]
    p.decode_device([t.data_ptr() for t in full])
    win = [torch.full_like(t, float("nan")) for t in d_in]
    for f0, f1 in [(0, 67), (67, 134), (134, 200)]:     # 3 ranks' windows
        p.decode_device([t.data_ptr() for t in win], frames=(f0, f1))
    for a in range(3):
        assert torch.equal(full[a], win[a])
    # a window writes only its own columns; bad windows are refused
    part = [torch.zeros_like(t) for t in d_in]
    p.decode_device([t.data_ptr() for t in part], frames=(10, 20))
    assert torch.equal(part[0][:, 10:20], full[0][:, 10:20])
    assert not part[0][:, :10].any() and not part[0][:, 20:].any()
    with pytest.raises(C.DmcError) as e:
        p.decode_device([t.data_ptr() for t in part], frames=(150, 250))
    assert e.value.code == 5
    # the drop-in decode honours the window too (host output)
    g = p.download()
    xh = codec.decode(g, frames=(50, 90))
    assert np.array_equal(xh[1][:, 50:90], full[1][:, 50:90].cpu().numpy())


def test_virtual_ranks_f32_grid(codec):
    """A small c3-style grid (f32 storage): the rank count does not change the
    stream beyond the Gram summation order; decode windows per rank."""
    s = synth.grid(48, 48, 64, seed=5)
    ec = C.EncoderConfig(k_l=24, row_bits=[12] * 24, oi_rounds=8)
    plans = _virtual_ranks_encode(codec, s, ec, 4, dtype=np.float32)
    g = plans[0].download()
    ref = codec.encode(s, ec)
    o = O.encode(s, 24, 12, rounds=8, seed=0, nthreads=8)
    for a in range(3):
        assert np.array_equal(g.anchor_q[a], ref.anchor_q[a])
        for j in _agreeing_columns(o.evals[a], 24):
            d = g.coeff_q[a][j].astype(np.int64) - ref.coeff_q[a][j].astype(np.int64)
            assert np.abs(d).max() <= 1 and np.count_nonzero(d) <= max(1, 1e-2 * s.n), (a, j)
    out = [torch.zeros((s.n, s.F), dtype=torch.float32, device="cuda") for _ in range(3)]
    for p in plans:
        p.decode_device([t.data_ptr() for t in out], frames=p.frames())
    x = [t.cpu().numpy() for t in out]
    xr = codec.decode(g, dtype=np.float32)
    for a in range(3):
        assert np.array_equal(x[a], xr[a])
