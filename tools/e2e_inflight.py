"""Drop-in e2e with K sequences in flight (one host thread + context each),
per-thread encode / decode wall times; DMCG_TIMING=1 adds the host phases.
python tools/e2e_inflight.py c1 4"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec, synth  # noqa: E402
from paper_2111_10105_b200.shard import sequence_for_rank  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hosts = []
for j in range(K):
    spec, s = sequence_for_rank(name, j)
    cfg = codec.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
    pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in s.axes]
    out = [torch.empty(x.shape, dtype=torch.float64).pin_memory().numpy() for x in s.axes]
    hosts.append((codec.Codec(0), synth.Sequence(s.faces, pin), out, cfg))
times = [None] * K


def one(j):
    cd, hs, out, cfg = hosts[j]
    t0 = time.perf_counter()
    enc = cd.encode(hs, cfg)
    t1 = time.perf_counter()
    cd.decode(enc, out=out)
    t2 = time.perf_counter()
    times[j] = (1e3 * (t1 - t0), 1e3 * (t2 - t1))


for it in range(4):
    t0 = time.perf_counter()
    th = [threading.Thread(target=one, args=(j,)) for j in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = 1e3 * (time.perf_counter() - t0)
    print(f"step {it}: {dt:.2f} ms; per thread enc/dec ms: " +
          " ".join(f"{a:.1f}/{b:.1f}" for a, b in times), flush=True)
