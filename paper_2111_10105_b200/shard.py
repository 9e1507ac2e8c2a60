"""Multi-GPU layouts of the bench / drop-in path.

Two layouts, one process per GPU:

* Independent sequences (c1 bench, c4): the reference codes one animation
  per call and sequences are independent, so N GPUs run N independent
  encode+decode streams with no data-path collective (weak scaling).  The
  only collectives are the timing reductions (barrier + max of the per-rank
  device time).
* Vertex-row shards of ONE large sequence (c3): ``ShardPlan`` over the C ABI
  ``dmcg_plan_create_shard`` / ``dmcg_shard_encode_device`` (libdmcg,
  csrc/shard.cpp): rank q owns a contiguous block of vertex rows; the Gram
  partials are allreduced (sum), the quantiser range keys allreduced (max)
  and the symbols all-gathered over NCCL inside the library, on the plan
  stream; the decode splits frames across ranks (no exchange).
  ``local_rows`` builds a rank's local input (owned rows + halo rows).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np


def dist_env():
    """(rank, world, local_rank) from the torchrun environment (1 process when unset)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def sequence_for_rank(cfgname: str, rank: int):
    """The sequence rank `rank` codes: rank 0 gets the config's own sequence,
    other ranks the same generator family (same mesh, frames, k, bits) with
    a distinct seed, so every rank does the same amount of distinct work."""
    from . import synth
    spec = synth.CONFIGS[cfgname]
    if rank == 0:
        return spec, spec.make(0)
    if cfgname == "c1":
        return spec, synth.torus(96, 96, 200, seed=1 + 1000 * rank)
    if cfgname == "c4":
        return spec, spec.make(rank)
    if cfgname == "c0":
        return spec, synth.sphere(4, 64, 4, 0, seed=1000 * rank)
    return spec, spec.make(0)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device time of the timed region) over all ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank_step: float, world: int, steps: int, max_ms: float) -> float:
    """Aggregate throughput: units every rank processed over the slowest rank's time."""
    return units_per_rank_step * world * steps / (max_ms / 1e3)


# ---- vertex-row shards of one sequence (libdmcg shard ABI) -----------------

def shard_layout(n, F, faces, cfg, nranks, rank):
    """Host-only layout of rank `rank` (dmcg_shard_layout): (info dict, halo ids)."""
    from . import _lib as L
    faces = np.ascontiguousarray(faces, dtype=np.uint32)
    info = L.DmcgShardInfo()
    c = cfg.to_c()
    rc = L.lib().dmcg_shard_layout(n, F, faces.ctypes.data_as(L.u32p), len(faces), ctypes.byref(c),
                                   nranks, rank, ctypes.byref(info), None)
    if rc:
        raise ValueError(f"dmcg_shard_layout failed ({rc})")
    halo = np.zeros(max(info.n_halo, 1), np.uint32)
    L.lib().dmcg_shard_layout(n, F, faces.ctypes.data_as(L.u32p), len(faces), ctypes.byref(c),
                              nranks, rank, ctypes.byref(info), halo.ctypes.data_as(L.u32p))
    return {f: getattr(info, f) for f, _ in L.DmcgShardInfo._fields_}, halo[:info.n_halo]


def local_rows(info, halo, axes):
    """A rank's local input rows (owned rows, then halo rows) of host axes."""
    b, e = info["row_begin"], info["row_end"]
    return [np.ascontiguousarray(np.concatenate([a[b:e], a[halo]], axis=0)) for a in axes]


class Comm:
    """NCCL communicator owned by libdmcg (dmcg_comm_create).  The 128-byte
    unique id is created on rank 0 and shared over torch.distributed."""

    def __init__(self, device, nranks, rank, dist=None):
        from . import _lib as L
        uid = np.zeros(128, np.uint8)
        if nranks > 1:
            if rank == 0 and L.lib().dmcg_comm_unique_id(uid.ctypes.data_as(L.u8p)):
                raise RuntimeError("dmcg_comm_unique_id failed (NCCL missing?)")
            import torch
            t = torch.from_numpy(uid.astype(np.int64))
            if dist.get_backend() == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0)
            uid = t.cpu().numpy().astype(np.uint8)
        self._c = ctypes.c_void_p()
        rc = L.lib().dmcg_comm_create(device, uid.ctypes.data_as(L.u8p), nranks, rank,
                                      ctypes.byref(self._c))
        if rc:
            raise RuntimeError(f"dmcg_comm_create failed ({rc})")
        self.nranks, self.rank = nranks, rank

    @property
    def handle(self):
        return self._c

    def close(self):
        from . import _lib as L
        if self._c:
            L.lib().dmcg_comm_destroy(self._c)
            self._c = ctypes.c_void_p()


def _shard_plan_class():
    from . import _lib as L
    from .codec import Plan, _check

    class ShardPlan(Plan):
        """A rank's plan over a vertex-row shard of one sequence.  Encode takes
        the rank's local rows (n_loc x F per axis, device pointers); after it,
        the plan holds the whole encoded stream (download / serialize /
        decode_device work as for a single-GPU plan)."""

        def __init__(self, codec, n, F, faces, cfg, nranks, rank, comm=None,
                     dtype=np.float64):
            self.codec = codec
            self.n, self.F, self.k_l = n, F, cfg.k_l
            self.dtype = L.DMCG_F32 if dtype == np.float32 else L.DMCG_F64
            self.faces = np.ascontiguousarray(faces, dtype=np.uint32)
            self._cfg = cfg.to_c()
            self._p = ctypes.c_void_p()
            _check(codec.handle, L.lib().dmcg_plan_create_shard(
                codec.handle, n, F, self.dtype, self.faces.ctypes.data_as(L.u32p),
                len(self.faces), ctypes.byref(self._cfg), nranks, rank,
                comm.handle if comm is not None else None, ctypes.byref(self._p)))
            self.n_c = L.lib().dmcg_anchor_count(n, cfg.anchor_fraction) \
                if cfg.variant in (L.DMCG_PCA_QS, L.DMCG_PCA_QP) else 0
            self.cfg = cfg
            codec._plans.add(self)
            info = L.DmcgShardInfo()
            L.lib().dmcg_shard_info_get(self._p, ctypes.byref(info), None)
            halo = np.zeros(max(info.n_halo, 1), np.uint32)
            L.lib().dmcg_shard_info_get(self._p, ctypes.byref(info), halo.ctypes.data_as(L.u32p))
            self.info = {f: getattr(info, f) for f, _ in L.DmcgShardInfo._fields_}
            self.halo = halo[:info.n_halo]

        def local_rows(self, axes):
            return local_rows(self.info, self.halo, axes)

        def encode_device(self, d_loc_axes):
            ptrs = (ctypes.c_void_p * 3)(*[int(p) for p in d_loc_axes])
            _check(self.codec.handle, L.lib().dmcg_shard_encode_device(self._p, ptrs))

        def encode_phase(self, phase, d_loc_axes):
            ptrs = (ctypes.c_void_p * 3)(*[int(p) for p in d_loc_axes])
            _check(self.codec.handle, L.lib().dmcg_shard_encode_phase(self._p, phase, ptrs))

        def buffer(self, which):
            """(device pointer, element count) of DMCG_SHARD_GRAM (f64) / KEYS (u64) /
            SYMBOLS (u16)."""
            ptr, cnt = ctypes.c_void_p(), ctypes.c_size_t()
            _check(self.codec.handle, L.lib().dmcg_shard_buffer(self._p, which, ctypes.byref(ptr),
                                                               ctypes.byref(cnt)))
            return ptr.value, cnt.value

        def frames(self):
            """This rank's decode window: frames [q F / N, (q+1) F / N)."""
            q, N = self.info["rank"], self.info["nranks"]
            return (q * self.F // N, (q + 1) * self.F // N)

    return ShardPlan


def ShardPlan(*args, **kw):  # noqa: N802 (class factory: codec imports this module lazily)
    return _shard_plan_class()(*args, **kw)


SHARD_GRAM, SHARD_KEYS, SHARD_SYMBOLS = 0, 1, 2
