"""C4 throughput: 64 independent icosphere-L5 sequences (F=128, k=64) on one GPU,
coded by K concurrent device-resident plans (one context / CUDA stream / host
thread each): python tools/c4_throughput.py [K ...]"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec as C, synth  # noqa: E402

spec = synth.CONFIGS["c4"]
NSEQ = 64
seqs = [spec.make(i) for i in range(NSEQ)]
cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
dev_in = [[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in s.axes] for s in seqs]
dev_out = [[torch.empty_like(t) for t in d] for d in dev_in]
vf = sum(s.n * s.F for s in seqs)


def run(K):
    codecs = [C.Codec(0) for _ in range(K)]
    plans = [C.Plan(codecs[j], seqs[0].n, seqs[0].F, seqs[0].faces, cfg) for j in range(K)]
    for j in range(K):  # warm-up: graphs captured per pointer set, so code every sequence once
        for i in range(j, NSEQ, K):
            plans[j].encode_device([t.data_ptr() for t in dev_in[i]])
            plans[j].decode_device([t.data_ptr() for t in dev_out[i]], reuse_factor=REUSE)
    torch.cuda.synchronize()

    def worker(j):
        for i in range(j, NSEQ, K):
            plans[j].encode_device([t.data_ptr() for t in dev_in[i]])
            plans[j].decode_device([t.data_ptr() for t in dev_out[i]], reuse_factor=REUSE)

    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(j,)) for j in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"K={K} reuse_factor={REUSE}: {NSEQ} sequences in {dt * 1e3:.1f} ms -> {vf / dt / 1e6:.1f} M vertex-frames/s")
    for p in plans:
        p.close()
    for c in codecs:
        c.close()


REUSE = False
for K in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    REUSE = False
    run(K)
    REUSE = True
    run(K)
