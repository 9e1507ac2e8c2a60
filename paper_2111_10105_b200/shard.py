"""Multi-GPU layout of the bench / drop-in path.

The reference codes one animation sequence per call; sequences are
independent, so N GPUs run N independent encode+decode streams — one process
per GPU, each coding its own sequence, with no data-path collective (weak
scaling).  The only collectives are the timing reductions (barrier + max of
the per-rank device time), which bench.py runs over NCCL on the GPU box and
the tests run over gloo on CPU.
"""
from __future__ import annotations

import os


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
