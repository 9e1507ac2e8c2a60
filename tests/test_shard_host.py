"""Vertex-row shard layout on CPU: libdmcg's host-only
dmcg_shard_layout, and the sharded encode's arithmetic decomposition run
over real gloo collectives (world_size 2) with numpy standing in for the
per-rank kernels: the sum-allreduced Gram partials equal the full Gram, the
max-allreduced (-min, max) keys equal the global ranges, and each rank's
delta rows computed from its local rows (owned + halo) equal the full delta
rows bit for bit (same CSR order)."""
import os
import socket
import sys

import numpy as np
import pytest

from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import shard, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _adjacency(n, faces):
    nb = [set() for _ in range(n)]
    for a, b, c in faces:
        nb[a] |= {b, c}
        nb[b] |= {a, c}
        nb[c] |= {a, b}
    return [sorted(x) for x in nb]


def _delta_rows(rows, axis, nb, index_of):
    """delta_i = deg_i x_i - sum_j x_j, accumulated in ascending global column
    order with the diagonal in place (laplacian.cpp:45 / encode.cu k_delta)."""
    out = np.zeros((len(rows), axis.shape[1]))
    for r, i in enumerate(rows):
        acc = np.zeros(axis.shape[1])
        for j in sorted(nb[i] + [i]):
            v = float(len(nb[i])) if j == i else -1.0
            acc = acc + v * axis[index_of(j)]
        out[r] = acc
    return out


@pytest.mark.parametrize("name,N", [("c0", 3), ("c1", 4), ("c1", 7)])
def test_layout_partitions_rows_anchors_and_symbols(name, N):
    spec = synth.CONFIGS[name]
    s = spec.make()
    cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
    nb = _adjacency(s.n, s.faces)
    anchors = C.select_anchors(s.n, C.anchor_count(s.n))
    rows, slots, stage = [], [], 0
    for q in range(N):
        info, halo = shard.shard_layout(s.n, s.F, s.faces, cfg, N, q)
        b, e = info["row_begin"], info["row_end"]
        assert b == q * s.n // N and e == (q + 1) * s.n // N and info["n_own"] == e - b
        want = sorted({j for i in range(b, e) for j in nb[i] if not b <= j < e})
        assert halo.tolist() == want and info["n_loc"] == e - b + len(want)
        ab, ae = info["anchor_begin"], info["anchor_end"]
        assert all(b <= a < e for a in anchors[ab:ae])
        assert info["stage_begin"] == stage
        assert info["stage_count"] == 3 * spec.k * (e - b) + 3 * (ae - ab) * s.F
        stage += info["stage_count"]
        rows.append((b, e))
        slots.append((ab, ae))
    assert rows[0][0] == 0 and rows[-1][1] == s.n and all(
        rows[q][1] == rows[q + 1][0] for q in range(N - 1))
    assert slots[0][0] == 0 and slots[-1][1] == len(anchors)
    assert stage == info["gather_count"] == 3 * spec.k * s.n + 3 * len(anchors) * s.F


def test_layout_rejects_bad_arguments():
    s = synth.CONFIGS["c0"].make()
    cfg = C.EncoderConfig(k_l=8)
    with pytest.raises(ValueError):
        shard.shard_layout(s.n, s.F, s.faces, cfg, 2, 2)
    with pytest.raises(ValueError):
        shard.shard_layout(s.n, s.F, s.faces, cfg, s.n + 1, 0)


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2111_10105_b200 import codec as C
    from paper_2111_10105_b200 import shard, synth
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        s = synth.sphere(2, 16, 3, 0, seed=11)       # 162 vertices, F = 16
        cfg = C.EncoderConfig(k_l=6, row_bits=[12] * 6, oi_rounds=4)
        info, halo = shard.shard_layout(s.n, s.F, s.faces, cfg, world, rank)
        loc = shard.local_rows(info, halo, s.axes)
        b, e = info["row_begin"], info["row_end"]
        nb = _adjacency(s.n, s.faces)
        pos = {g: i for i, g in enumerate(list(range(b, e)) + halo.tolist())}
        ok_delta = all(np.array_equal(
            _delta_rows(range(b, e), loc[a], nb, lambda j: pos[j]),
            _delta_rows(range(b, e), s.axes[a], nb, lambda j: j)) for a in range(3))
        # Gram partial of the owned rows -> allreduce(sum)
        part = torch.from_numpy(np.stack([loc[a][:e - b].T @ loc[a][:e - b] for a in range(3)]))
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        full = np.stack([s.axes[a].T @ s.axes[a] for a in range(3)])
        gram_err = float(np.abs(part.numpy() - full).max() / np.abs(full).max())
        # range keys (-min, max) of the owned anchor trajectories -> allreduce(max)
        anchors = C.select_anchors(s.n, C.anchor_count(s.n))
        own = [a for a in anchors if b <= a < e]
        loc_rows = [a - b for a in own]
        keys = torch.tensor([[-(loc[a][loc_rows].min()) if own else -np.inf,
                              loc[a][loc_rows].max() if own else -np.inf] for a in range(3)])
        dist.all_reduce(keys, op=dist.ReduceOp.MAX)
        want = np.array([[-s.axes[a][anchors].min(), s.axes[a][anchors].max()] for a in range(3)])
        q.put((rank, ok_delta, gram_err, bool(np.array_equal(keys.numpy(), want))))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_decomposition():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    for _, ok_delta, gram_err, ok_keys in res:
        assert ok_delta and ok_keys and gram_err < 1e-13
