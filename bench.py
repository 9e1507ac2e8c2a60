"""bench.py — encode+decode vertex-frames/s of the pca_qp hot path on B200.

Contract: one JSON line on rank 0.
  * workload (N = 1): BASELINE.json configs[3] — the largest single-GPU
    config (512 x 512 grid, 262 144 vertices, F = 512, k = 256, 20 OI rounds,
    12-bit, fp32 storage) unless --config says otherwise; a "step" = one full
    encode + decode of ONE sequence.  configs[3] names the covariance
    "applied implicitly as X(X^T Q)"; the explicit R = X^T X (same iteration,
    2 F^2 n flops once instead of 4 F n k per round) is the headline and the
    implicit form is reported beside it (key "implicit_covariance").
  * value: device-resident (inputs already in HBM, mesh plan built once
    outside the timed region), CUDA events on the plan stream, L2 flushed
    (256 MiB write) between steps outside the events; max over ranks.
  * e2e: the same metric through the drop-in C ABI (dmcg_encode +
    dmcg_decode) from pinned host buffers: H2D of the inputs, mesh build,
    D2H of the encoded symbols, H2D for decode, normal matrix + symbolic
    analysis, D2H of the vertices — all inside the timed region.
  * cpu_baseline: the oracle port (kind "port"; the reference itself needs
    Eigen3, absent) on a bounded sample of the same workload — the config's
    generator at a smaller vertex count with the same F / k / rounds / bits —
    single-thread (the reference is single-threaded) and on all host cores,
    with per-stage times.
  * N > 1 (torchrun, or --gpus N which re-launches itself under
    torch.distributed.run): default --mode rows — ONE c3 sequence sharded by
    vertex rows across the N ranks (libdmcg shard ABI: NCCL allreduce of the
    Gram partials and range keys, all-gather of the symbols; decode split by
    frame windows) -> scaling "strong".  --mode sequences: every rank codes
    its own independent sequences, no data-path collective -> "weak".
  * small configs (<= 4 M vertex-frames: c0, c1, c4) keep K independent
    sequences in flight per GPU (--inflight, default 8 there) — one sequence
    of those is a latency chain that leaves most SMs idle.
  * --impl reference: the CPU oracle port on all host cores, rank 0 only,
    each step the bounded sample above.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2111_10105_b200.shard import (dist_env, max_over_ranks, sequence_for_rank,  # noqa: E402
                                         whole_job_rate)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
FP64_DMMA_TFLOPS = 37.1  # profiles/r01_peaks.md (tools/peak_fp64.cu)
# dram__bytes_read.sum + dram__bytes_write.sum per launch, per config and
# kernel, from the committed ncu captures (tools/kernel_roofline.py --traffic-json)
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "roofline_traffic.json")

# Bounded CPU samples (cpu_baseline and --impl reference): the config's own
# generator at a smaller size, same F / k / OI rounds / bits / dtype.
CPU_SAMPLES = {
    "c3": {1: ("grid", 64, 64), 0: ("grid", 256, 256)},   # 0 = all host cores
}


def traffic_of(cfgname, kernel_prefix):
    try:
        data = json.load(open(TRAFFIC_PATH))[cfgname]
    except Exception:
        return None
    if kernel_prefix in data:  # base name over all template instantiations
        return int(data[kernel_prefix])
    for name, b in data.items():
        if name.replace("void ", "").startswith(kernel_prefix):
            return int(b)
    return None

WORKLOADS = {
    "c0": "c0: icosphere L4 (2562 v), F=64, k=32, 10 OI rounds, 12-bit, fp64",
    "c1": "c1: torus 96x96 (9216 v), F=200, k=64, 15 OI rounds, 12-bit, fp64",
    "c2": "c2: icosphere L6 (40962 v), F=256, k=128, 20 OI rounds, 10-bit, fp64",
    "c2f32": "c2f32: icosphere L6 (40962 v), F=256, k=128, 20 OI rounds, 10-bit, fp32 storage",
    "c3": "c3: grid 512x512 (262144 v), F=512, k=256, 20 OI rounds, 12-bit, fp32 storage",
    "c4": "c4: icosphere L5 (10242 v) sequences, F=128, k=64, 10 OI rounds, 12-bit, fp64",
}


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.path = f"/tmp/dmcg_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def load_peak():
    try:
        return float(json.load(open(PEAKS_PATH))["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def cpu_sample(cfgname, threads):
    """(sequence, description) of the bounded CPU sample of a config: c3 uses
    its generator at 64 x 64 (one thread) / 256 x 256 (all cores) vertices with
    the same F, k, OI rounds, bits and dtype; the small configs run whole."""
    from paper_2111_10105_b200 import synth
    spec = synth.CONFIGS[cfgname]
    samp = CPU_SAMPLES.get(cfgname)
    if samp is None:
        return spec, spec.make(0), f"the full {cfgname} sequence"
    kind, nx, ny = samp[1 if threads == 1 else 0]
    s = synth.grid(nx, ny, 512, seed=3)
    return spec, s, (f"{cfgname} generator at {nx}x{ny} = {s.n} vertices (full config 512x512), "
                     f"same F={s.F}, k={spec.k}, {spec.rounds} OI rounds, {spec.bits}-bit, "
                     "fp32 storage")


def time_oracle(cfgname, threads, steps=1):
    """Oracle port (oracle/dmc_oracle.c) encode + decode of the bounded
    sample: vertex-frames/s and per-stage seconds (median over `steps`)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    spec, s, desc = cpu_sample(cfgname, threads)
    walls, stages = [], []
    for _ in range(steps):
        te, td = {}, {}
        t0 = time.perf_counter()
        enc = O.encode(s, spec.k, spec.bits, rounds=spec.rounds, nthreads=threads, timing=te)
        O.decode(enc, nthreads=threads, timing=td)
        walls.append(time.perf_counter() - t0)
        stages.append({"connectivity": te["t_connectivity"] + td["t_connectivity"],
                       "gram": te["t_gram"], "eigen_oi": te["t_eigen"], "delta": te["t_delta"],
                       "projection": te["t_project"], "quantize": te["t_quantize"],
                       "anchors": te["t_anchors"], "dict_decode": td["t_dict_decode"],
                       "reconstruct": td["t_reconstruct"], "anchored_solve": td["t_solve"]})
    wall = float(np.median(walls))
    st = {k: round(float(np.median([d[k] for d in stages])), 4) for k in stages[0]}
    return {"value": s.n * s.F / wall, "unit": "vertex-frames/s", "threads": threads,
            "seconds": wall, "vertex_frames": s.n * s.F, "sample": desc, "stage_s": st,
            "walls": walls}


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle port of the reference path (the
    reference itself needs Eigen3, absent) on all host cores, rank 0 only;
    each step one encode + decode of the bounded sample."""
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    r = time_oracle(args.config, threads, steps=args.warmup + args.steps)
    walls = r["walls"][args.warmup:]
    tot = sum(walls)
    value = r["vertex_frames"] * len(walls) / tot
    line = {
        "impl": "reference", "metric": "encode+decode vertex-frames/sec", "value": value,
        "unit": "vertex-frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(walls), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, DESIGN.md §2)",
        "config": {"workload": WORKLOADS[args.config], "solver": "sparse LDL^T + 1 refinement"},
        "cpu_baseline": {"value": value, "unit": "vertex-frames/s", "cores": threads, "kind": "port",
                         "sample": r["sample"] + " per step (oracle/dmc_oracle.c; the reference "
                                                 "needs Eigen3, absent)",
                         "stage_s": r["stage_s"]},
        "e2e": {"value": value, "unit": "vertex-frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args):
    """Two rows on the box's host cores: single-thread (like the reference) and
    all cores; each its own bounded sample, per-stage seconds."""
    threads = os.cpu_count() or 1
    rows = [time_oracle(args.config, 1), time_oracle(args.config, threads)]
    for r in rows:
        r.pop("walls")
    allc = rows[1]
    return {"value": allc["value"], "unit": "vertex-frames/s", "cores": threads, "kind": "port",
            "sample": allc["sample"] + f"; {allc['seconds']:.2f} s on {threads} threads",
            "rows": rows}


class _DevArray:
    """__cuda_array_interface__ view of a libdmcg device buffer (for torch)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def run_rows(args, rank, world, local, dist):
    """One sequence, vertex rows sharded over the ranks."""
    import torch
    from paper_2111_10105_b200 import codec as C
    from paper_2111_10105_b200 import shard, synth

    spec = synth.CONFIGS[args.config]
    s = spec.make(0)
    cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds,
                          oi_implicit=args.implicit)
    f32 = spec.dtype == "f32"
    npdt = np.float32 if f32 else np.float64
    tdt = torch.float32 if f32 else torch.float64
    codec = C.Codec(local)
    comm = shard.Comm(local, world, rank, dist)
    plan = shard.ShardPlan(codec, s.n, s.F, s.faces, cfg, world, rank, comm, dtype=npdt)
    info = plan.info
    loc_host = plan.local_rows([np.asarray(a, dtype=npdt) for a in s.axes])
    d_loc = [torch.from_numpy(a).cuda() for a in loc_host]
    d_out = [torch.zeros((s.n, s.F), dtype=tdt, device="cuda") for _ in range(3)]
    f0, f1 = plan.frames()
    stream = torch.cuda.ExternalStream(plan.stream())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        plan.encode_device([t.data_ptr() for t in d_loc])
        plan.decode_device([t.data_ptr() for t in d_out], rtol=args.rtol, frames=(f0, f1))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms, stages, launches = [], [], 0
    with Clocks(local) as clk:
        for it in range(args.steps):
            flush.fill_(it & 0xFF)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            st = plan.stats()
            stages.append({k: v for k, v in st.items() if k.startswith("ms_")})
            launches += st["kernel_launches_encode"] + st["kernel_launches_decode"]
    total_ms = max_over_ranks(float(sum(step_ms)), dist, "cuda")
    value = s.n * s.F * args.steps / (total_ms / 1e3)

    # e2e: pinned host local rows -> H2D, sharded encode, D2H of this rank's
    # symbols (its share of the compressed stream), frame-window decode, D2H of
    # the window's frames.
    pin_in = [torch.from_numpy(a).pin_memory() for a in loc_host]
    sym_ptr, _ = plan.buffer(shard.SHARD_SYMBOLS)
    sb, sc = info["stage_begin"], info["stage_count"]
    syms = torch.as_tensor(_DevArray(sym_ptr, info["gather_count"], "<i2"), device="cuda")
    pin_sym = torch.empty(sc, dtype=torch.int16).pin_memory()
    pin_out = [torch.empty((s.n, f1 - f0), dtype=tdt).pin_memory() for _ in range(3)]
    e2e_ms = []
    for it in range(max(2, args.steps) + 1):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for a in range(3):
                d_loc[a].copy_(pin_in[a], non_blocking=True)
        plan.encode_device([t.data_ptr() for t in d_loc])
        with torch.cuda.stream(stream):
            pin_sym.copy_(syms[sb:sb + sc], non_blocking=True)
        plan.decode_device([t.data_ptr() for t in d_out], rtol=args.rtol, frames=(f0, f1))
        with torch.cuda.stream(stream):
            for a in range(3):
                pin_out[a].copy_(d_out[a][:, f0:f1], non_blocking=True)
        stream.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if it > 0:
            e2e_ms.append(dt)
    e2e_total = max_over_ranks(float(sum(e2e_ms)), dist, "cuda")
    e2e_value = s.n * s.F * len(e2e_ms) / (e2e_total / 1e3)
    es = np.dtype(npdt).itemsize
    h2d = sum(a.nbytes for a in loc_host)
    d2h = sc * 2 + 3 * s.n * (f1 - f0) * es
    out = [t.cpu().numpy() for t in d_out]
    bbox = float(np.linalg.norm([a.max() - a.min() for a in s.axes]))
    err = max(float(np.abs(out[a][:, f0:f1].astype(np.float64) - s.axes[a][:, f0:f1]).max())
              for a in range(3))
    st = plan.stats()
    if rank == 0:
        med = {k: float(np.median([d[k] for d in stages])) for k in stages[0]}
        oi_flops = float(st["flops_oi"])
        oi_ms = med.get("ms_oi", 0.0)
        achieved = oi_flops / (oi_ms / 1e3) / 1e12 if oi_ms > 0 else 0.0
        line = {
            "metric": "encode+decode vertex-frames/sec", "value": value, "unit": "vertex-frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if not f32 else "f64 (f32 storage)",
            "data": "synthetic (seeded generator, DESIGN.md §2)",
            "config": {"workload": WORKLOADS[args.config], "per_gpu": "1/N of one sequence per step",
                       "covariance": "implicit X^T (X Q), partials allreduced per round"
                       if args.implicit else "explicit R = X^T X (allreduced once)",
                       "parallelism": f"vertex rows x{world} (encode: NCCL allreduce of Gram "
                                      "partials + range keys, all-gather of symbols; decode: "
                                      "frame windows, replicated factor)",
                       "rows_per_rank": info["n_own"], "halo_rows": info["n_halo"],
                       "frames_decoded_per_rank": f1 - f0,
                       "l2": "256 MiB flush between timed steps", "cg_rtol": args.rtol},
            # `roofline` = the kernel with the largest share of the step (CUDA
            # events); the others beside it
            "roofline": {"kernel": "k_oi_cluster", "bound": "tensor", "achieved": achieved,
                         "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_DMMA_TFLOPS,
                         "traffic": traffic_of(args.config, "k_oi_cluster"),
                         "algorithmic_flops": oi_flops, "ms": oi_ms,
                         "share_of_step": oi_ms / (total_ms / args.steps)},
            "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": "vertex-frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_total / len(e2e_ms),
                    "note": "per rank: pinned local rows in, own symbols + own frame window out; "
                            "plan (mesh, halo, symbolic analysis) built once outside"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "quality": {"max_err_over_bbox_rank0_window": err / bbox},
            "stage_ms_rank0": med,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    comm.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def time_plan(plan, d_in, d_out, args, stream, flush, dist, local):
    """W untimed warm-up steps, then K steps each bracketed by CUDA events on
    the plan stream (the L2 flush and the host sync sit outside the events).
    Returns (per-step ms, per-step plan stats, launches, Clocks)."""
    import torch
    for _ in range(args.warmup):
        plan.encode_device([t.data_ptr() for t in d_in])
        plan.decode_device([t.data_ptr() for t in d_out], rtol=args.rtol)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms, stats, launches = [], [], 0
    with Clocks(local) as clk:
        for it in range(args.steps):
            flush.fill_(it & 0xFF)               # L2 flush, outside the timed events
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.encode_device([t.data_ptr() for t in d_in])
            plan.decode_device([t.data_ptr() for t in d_out], rtol=args.rtol)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            st = plan.stats()
            stats.append(st)
            launches += st["kernel_launches_encode"] + st["kernel_launches_decode"]
    torch.cuda.synchronize()
    return step_ms, stats, launches, clk


def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without a torchrun environment: re-exec this
    script under torch.distributed.run with N ranks on this node (loopback
    rendezvous) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-implicit", action="store_true",
                    help="skip the extra implicit-covariance measurement (c3)")
    ap.add_argument("--implicit", action="store_true",
                    help="headline with the implicit OI: Z = X^T (X Q) per round, R never formed")
    ap.add_argument("--inflight", type=int, default=None,
                    help="independent sequences in flight per GPU (one context / CUDA stream / "
                         "host thread each); default 8 for sequences of <= 4 M vertex-frames "
                         "(c0, c1, c4), else 1")
    ap.add_argument("--n-b", type=int, default=1,
                    help="blocks variant with this many frame blocks (SURVEY 8f f2); "
                         "k_l = min(config k, k_f); default 1 = the pca_qp hot path")
    ap.add_argument("--mode", choices=["rows", "sequences"], default=None,
                    help="N > 1: rows = one sequence sharded by vertex rows (default), "
                         "sequences = independent sequences per rank")
    ap.add_argument("--rows", action="store_true", help="same as --mode rows")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.rows:
        args.mode = "rows"
    if args.mode is None:
        args.mode = "rows" if world > 1 and args.n_b == 1 else "sequences"

    import torch
    from paper_2111_10105_b200 import codec as C

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator / NVLS lines
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.mode == "rows":
        return run_rows(args, rank, world, local, dist)

    spec, s = sequence_for_rank(args.config, rank)
    cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds,
                          oi_implicit=args.implicit)
    if args.n_b > 1:  # blocks variant: n_b dictionaries of k_f frames
        kf = (s.F + (args.n_b - s.F % args.n_b) % args.n_b) // args.n_b
        kl = min(spec.k, kf)
        cfg = C.EncoderConfig(variant=C.L.DMCG_BLOCKS, n_b=args.n_b, k_l=kl,
                              row_bits=[spec.bits] * kl)
    f32 = spec.dtype == "f32"
    npdt = np.float32 if f32 else np.float64
    codec = C.Codec(local)

    # ---- device-resident value --------------------------------------------
    plan = C.Plan(codec, s.n, s.F, s.faces, cfg, dtype=npdt)
    d_in = [torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).cuda() for x in s.axes]
    d_out = [torch.empty_like(t) for t in d_in]
    stream = torch.cuda.ExternalStream(plan.stream())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    step_ms, stats, launches, clk = time_plan(plan, d_in, d_out, args, stream, flush, dist, local)
    fac_ms = [st["ms_factor"] for st in stats]
    sol_ms = [st["ms_solve"] for st in stats]
    oi_ms = [st["ms_oi"] for st in stats]
    total_ms = max_over_ranks(float(sum(step_ms)), dist, "cuda")
    if dist:
        dist.barrier()

    # ---- the implicit covariance of configs[3] (extra key) ------------------
    implicit = None
    if args.config == "c3" and not args.implicit and not args.no_implicit and args.n_b == 1:
        icfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds,
                               oi_implicit=True)
        iplan = C.Plan(codec, s.n, s.F, s.faces, icfg, dtype=npdt)
        istream = torch.cuda.ExternalStream(iplan.stream())
        i_ms, i_stats, i_launch, i_clk = time_plan(iplan, d_in, d_out, args, istream, flush, dist,
                                                   local)
        i_total = max_over_ranks(float(sum(i_ms)), dist, "cuda")
        implicit = {"value": whole_job_rate(s.n * s.F, world, args.steps, i_total),
                    "ms_per_step": i_total / args.steps,
                    "covariance": "implicit: every OI round P = X Q, Z = X^T P (R never formed)",
                    "gpu_launches": i_launch, "clocks": i_clk.summary(),
                    "stage_ms": {k: float(np.median([d[k] for d in i_stats]))
                                 for k in i_stats[0] if k.startswith("ms_")}}
        iplan.close()
    vf_step = s.n * s.F
    value = whole_job_rate(vf_step, world, args.steps, total_ms)
    single_ms = total_ms / args.steps   # one sequence at a time (latency of one encode+decode)

    # ---- K sequences in flight per GPU (throughput mode) -------------------
    # One sequence leaves most of the 148 SMs idle (the OI, Jacobi and the
    # factor's top levels are latency chains on a few SMs), so the serving
    # configuration keeps K independent sequences in flight: K contexts, each
    # with its own CUDA stream, plan and host thread.  A step = all K
    # encode+decode pairs; device-timed from one start event every plan
    # stream waits on to the last plan stream's end event.
    K = max(1, args.inflight if args.inflight is not None else (8 if vf_step <= 4_000_000 else 1))
    inflight = None
    if K > 1:
        import threading
        seqs = [s] + [sequence_for_rank(args.config, world * j + rank)[1] for j in range(1, K)]
        codecs = [codec] + [C.Codec(local) for _ in range(1, K)]
        plans = [plan] + [C.Plan(codecs[j], seqs[j].n, seqs[j].F, seqs[j].faces, cfg, dtype=npdt)
                          for j in range(1, K)]
        ins = [d_in] + [[torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).cuda()
                         for x in seqs[j].axes] for j in range(1, K)]
        outs = [d_out] + [[torch.empty_like(t) for t in ins[j]] for j in range(1, K)]
        pstreams = [torch.cuda.ExternalStream(p.stream()) for p in plans]

        def one(j, ends=None):
            plans[j].encode_device([t.data_ptr() for t in ins[j]])
            plans[j].decode_device([t.data_ptr() for t in outs[j]], rtol=args.rtol)
            if ends is not None:
                ends[j].record(pstreams[j])

        def concurrent(ends=None):
            th = [threading.Thread(target=one, args=(j, ends)) for j in range(K)]
            for t in th:
                t.start()
            for t in th:
                t.join()

        for _ in range(args.warmup):
            concurrent()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        k_ms, k_launch = [], 0
        with Clocks(local) as kclk:
            for it in range(args.steps):
                flush.fill_(it & 0xFF)
                torch.cuda.synchronize()
                start = torch.cuda.Event(enable_timing=True)
                start.record()
                for ps in pstreams:
                    ps.wait_event(start)
                ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
                concurrent(ends)
                torch.cuda.synchronize()
                k_ms.append(max(start.elapsed_time(e) for e in ends))
                for p in plans:
                    st_j = p.stats()
                    k_launch += st_j["kernel_launches_encode"] + st_j["kernel_launches_decode"]
        k_total = max_over_ranks(float(sum(k_ms)), dist, "cuda")
        if dist:
            dist.barrier()
        inflight = {"K": K, "ms_per_step": k_total / args.steps, "clocks": kclk.summary(),
                    "launches": k_launch,
                    "value": whole_job_rate(vf_step * K, world, args.steps, k_total)}
        value = inflight["value"]
        total_ms = k_total
        launches = k_launch
        clk = kclk

    # roofline of the dominant kernel, k_oi_cluster (the fused orthogonal
    # iterations, one cluster of k/8 CTAs per axis): algorithmic flops per launch
    # over its launch time, CUDA events around the launch on
    # the plan stream (stats.ms_oi), median over the timed steps.  The
    # decode's direct solve (K7) is reported beside it.
    st = plan.stats()
    oi_flops = float(st["flops_oi"])
    oi_sec = float(np.median(oi_ms)) / 1e3 if oi_ms else 0.0
    peak = FP64_DMMA_TFLOPS
    achieved = oi_flops / oi_sec / 1e12 if oi_sec > 0 else 0.0
    k7_flops = float(st["flops_factor"] + st["flops_solve"])
    k7_sec = float(np.median(fac_ms) + np.median(sol_ms)) / 1e3
    k7_achieved = k7_flops / k7_sec / 1e12 if k7_sec > 0 else 0.0
    # the solve GEMMs (k_fwd / k_bwd, one launch per tree level and solve):
    # one untimed pass with CUDA events around every launch (plan stream)
    plan.set_kernel_timing(True)
    plan.encode_device([t.data_ptr() for t in d_in])
    plan.decode_device([t.data_ptr() for t in d_out], rtol=args.rtol)
    torch.cuda.synchronize()
    kst = plan.stats()
    plan.set_kernel_timing(False)
    solve_launches = int(st["levels"]) * 2  # per direction: levels x (solve + refinement)

    def solve_roofline(name, ms, flops):
        ach = flops / (ms / 1e3) / 1e12 if ms > 0 else 0.0
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": peak,
                "peak_kind": "measured FP64 DMMA, whole GPU (profiles/r01_peaks.md)",
                "unit": "TFLOP/s", "frac": ach / peak,
                "traffic": traffic_of(args.config, name),
                "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, mean per "
                                  f"launch, {args.config} (profiles/roofline_traffic.json)",
                "launches_per_step": solve_launches, "algorithmic_flops": flops / solve_launches,
                "algorithmic_flops_per_step": flops, "ms": ms,
                "share_of_step": ms / single_ms,
                "share_basis": "summed launch times of one encode+decode timed alone (CUDA events "
                               "around every launch on the plan stream)",
                "model": "per solve 2 W sum_s m_s w_s (P_s r_s forward / P_s^T [y; x] backward), "
                         "W = 3F; DESIGN.md §5"}
    roof_fwd = solve_roofline("k_fwd", float(kst["ms_solve_fwd"]), float(kst["flops_solve_fwd"]))
    roof_bwd = solve_roofline("k_bwd", float(kst["ms_solve_bwd"]), float(kst["flops_solve_bwd"]))
    roof_main = roof_fwd if roof_fwd["ms"] >= roof_bwd["ms"] else roof_bwd

    # ---- e2e through the drop-in C ABI from pinned host memory -------------
    pinned = [torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).pin_memory() for x in s.axes]
    host_seq = type(s)(s.faces, [p.numpy() for p in pinned])
    pinned_out = [torch.empty(x.shape, dtype=torch.float32 if f32 else torch.float64).pin_memory()
                  .numpy() for x in s.axes]
    # K in flight: K host threads, each through its own drop-in context with
    # its own pinned buffers; a step ends when the last of the K returns.
    hosts = [(codec, host_seq, pinned_out)]
    for j in range(1, K):
        pj = [torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).pin_memory() for x in seqs[j].axes]
        oj = [torch.empty(x.shape, dtype=torch.float32 if f32 else torch.float64).pin_memory()
              .numpy() for x in seqs[j].axes]
        hosts.append((codecs[j], type(s)(seqs[j].faces, [q.numpy() for q in pj]), oj))
    e2e_res = [None] * K
    # the encoded stream lands in page-locked host arrays allocated once per
    # worker (after its untimed warm-up pair), like the input and output
    enc_buf = [None] * K

    def e2e_one(j):
        cj, sj, oj = hosts[j]
        ej = cj.encode(sj, cfg, out=enc_buf[j])
        if enc_buf[j] is None:
            enc_buf[j] = C.CompressedAnimation.allocate(
                ej.n, ej.F, ej.k_l, ej.n_c, ej.faces, n_b=ej.n_b, pinned=True,
                anchor_bits=ej.anchor_bits, dict_bits=ej.dict_bits, diff_bits=ej.diff_bits,
                variant=ej.variant)
        e2e_res[j] = (ej, cj.decode(ej, rtol=args.rtol, dtype=npdt, out=oj))

    e2e_ms = []
    n_e2e = max(2, args.steps)
    if K == 1:
        for it in range(n_e2e + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_one(0)
            dt = (time.perf_counter() - t0) * 1e3
            if it > 0:
                e2e_ms.append(dt)
    else:
        # Steady state of K workers: after one synchronised warm-up pair each,
        # every worker runs n_e2e encode+decode pairs back to back with no
        # barrier between steps, so one worker's H2D / encode overlaps another's
        # decode / D2H (a step-synchronised loop would run all K encodes, then
        # all K decodes, leaving the copy engines and SMs idle in turns).
        # Per-step time = wall time of the whole run / n_e2e.
        def worker(j):
            for _ in range(n_e2e):
                e2e_one(j)

        for fn in (e2e_one, worker):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            th = [threading.Thread(target=fn, args=(j,)) for j in range(K)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            dt = (time.perf_counter() - t0) * 1e3
        e2e_ms = [dt / n_e2e] * n_e2e
    enc, out = e2e_res[0]
    e2e_total = max_over_ranks(float(sum(e2e_ms)), dist, "cuda")
    e2e_value = whole_job_rate(vf_step * K, world, len(e2e_ms), e2e_total)
    es = np.dtype(npdt).itemsize
    enc_bytes = sum(x.nbytes for x in enc.dict_q + enc.row_min + enc.row_max + enc.row_bits +
                    enc.coeff_q + enc.anchor_q) + enc.anchor_idx.nbytes
    h2d = K * (3 * s.n * s.F * es + s.faces.nbytes + enc_bytes + s.faces.nbytes)
    d2h = K * (enc_bytes + 3 * s.n * s.F * es)
    bbox = float(np.linalg.norm([a.max() - a.min() for a in s.axes]))
    rms = float(np.sqrt(np.mean([np.mean((out[a].astype(np.float64) - s.axes[a]) ** 2)
                                 for a in range(3)])) * np.sqrt(3))

    if rank == 0:
        cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(args)
        line = {
            "metric": "encode+decode vertex-frames/sec", "value": value, "unit": "vertex-frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if not f32 else "f64 (f32 storage)",
            "data": "synthetic (seeded generator, DESIGN.md §2)",
            "config": {"workload": WORKLOADS[args.config] + (
                           f"; blocks variant n_b={args.n_b}, k_l={cfg.k_l}, t_max=4"
                           if args.n_b > 1 else ""),
                       "per_gpu": (f"{K} independent sequences in flight per step (one context / "
                                   "CUDA stream / host thread each)") if K > 1
                       else "one sequence per step",
                       "inflight": K,
                       "ms_one_sequence_alone": single_ms,
                       "covariance": "implicit X^T (X Q) per round" if args.implicit
                       else "explicit R = X^T X",
                       "parallelism": f"sequences x{world}, no collective",
                       "l2": "256 MiB flush between timed steps",
                       "plan": "mesh plan (CSR, anchors, normal matrix) built once outside value; "
                               "inside e2e", "cg_rtol": args.rtol},
            # `roofline` = the kernel with the largest share of the step (CUDA
            # events); the others beside it
            "roofline": roof_main,
            "roofline_other_solve": roof_bwd if roof_main is roof_fwd else roof_fwd,
            "roofline_oi": {"kernel": "k_oi_cluster", "bound": "tensor", "achieved": achieved,
                         "peak": peak, "peak_kind": "measured FP64 DMMA, whole GPU (profiles/r01_peaks.md)",
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic_of(args.config, "k_oi_cluster"),
                         "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per "
                                           f"launch, {args.config} (profiles/roofline_traffic.json)",
                         "launches_per_step": 1, "ctas": 3 * ((spec.k + 7) // 8),
                         "cluster": (spec.k + 7) // 8,
                         "algorithmic_flops": oi_flops, "ms": oi_sec * 1e3,
                         "share_of_step": oi_sec * 1e3 / single_ms,
                         "share_basis": "of one sequence's encode+decode timed alone",
                         "model": "3 axes x ((rounds+1) x (2F^2k + 4Fk^2 - 4k^3/3) + 2Fk^2)",
                         "note": "one cluster per axis, 8 or 16 columns of Z / Q per CTA; every "
                                 "OI round is a wavefront of dependent block-Householder steps "
                                 "(latency-bound), so the ceiling is the cluster's SMs, not the "
                                 "device peak; see DESIGN.md §5"},
            "roofline_k7": {"kernel": "K7 direct solve (k_panel/k_trailing/k_inv_*/k_fwd*/k_bwd*)",
                            "bound": "tensor", "achieved": k7_achieved, "peak": peak, "unit": "TFLOP/s",
                            "frac": k7_achieved / peak, "algorithmic_flops": k7_flops,
                            "ms_factor": float(np.median(fac_ms)), "ms_solve": float(np.median(sol_ms)),
                            "supernodes": st["supernodes"], "nnz_factor": st["nnz_factor"]},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "vertex-frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_total / len(e2e_ms),
                    "schedule": (f"{K} drop-in workers (host thread + context each) in steady "
                                 f"state, {n_e2e} encode+decode pairs each, no barrier between "
                                 "steps; ms_per_step = wall / pairs per worker")
                    if K > 1 else "one drop-in encode+decode per step"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "quality": {"rmse_over_bbox": rms / bbox},
            "stage_ms": {k: float(np.median([d[k] for d in stats])) for k in stats[0]
                         if k.startswith("ms_")},
            "implicit_covariance": implicit,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
