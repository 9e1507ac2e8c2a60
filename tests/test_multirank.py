"""N > 1 path on CPU (gloo, world_size 2): every rank codes its own sequence
with no data-path collective; the timing reductions are max-over-ranks; the
reference arm runs on rank 0 only under torchrun."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    from paper_2111_10105_b200 import shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = shard.dist_env()
        mx = shard.max_over_ranks(10.0 + 7.0 * rank, dist, "cpu")
        spec, s = shard.sequence_for_rank("c0", r)
        digest = float(np.sum(s.axes[0][:50, :8]))
        q.put((r, w, lr, mx, s.n, s.F, s.faces.sum(), digest))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_max_reduction():
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    (r0, w0, l0, m0, n0, f0, fc0, d0), (r1, w1, l1, m1, n1, f1, fc1, d1) = res
    assert (r0, r1) == (0, 1) and w0 == w1 == 2 and (l0, l1) == (0, 1)
    assert m0 == m1 == 17.0                      # max over ranks, seen identically by both
    assert (n0, f0, fc0) == (n1, f1, fc1)        # same mesh and frame count per rank
    assert d0 != d1                              # distinct sequences: no duplicated work


def test_whole_job_rate_is_units_over_slowest_rank():
    from paper_2111_10105_b200 import shard
    assert shard.whole_job_rate(1000, 4, 5, 2000.0) == pytest.approx(1000 * 4 * 5 / 2.0)
    assert shard.max_over_ranks(3.5) == 3.5


def test_reference_arm_under_torchrun_prints_on_rank0_only():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl",
           "reference", "--config", "c0", "--gpus", "2", "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["cpu_baseline"]["kind"] == "port"


def test_gpus_flag_relaunches_itself_under_torchrun():
    """`python bench.py --gpus 2` with no torchrun environment re-executes itself
    under torch.distributed.run with 2 ranks (loopback rendezvous) instead of
    silently running one process; rank 0 alone prints the line."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--config", "c0", "--gpus", "2",
           "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2


def test_gpus_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c0",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stdout
