"""K independent sequences in flight on one GPU (one context / plan / stream /
host thread each): device-timed throughput of K concurrent encode+decode.
python tools/inflight_probe.py c1 1 2 4"""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec as C  # noqa: E402
from paper_2111_10105_b200.shard import sequence_for_rank  # noqa: E402

name = sys.argv[1]
Ks = [int(a) for a in sys.argv[2:]] or [1, 2, 4]
for K in Ks:
    seqs = [sequence_for_rank(name, j) for j in range(K)]
    spec = seqs[0][0]
    cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
    codecs = [C.Codec(0) for _ in range(K)]
    plans = [C.Plan(codecs[j], s.n, s.F, s.faces, cfg) for j, (_, s) in enumerate(seqs)]
    din = [[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in s.axes] for _, s in seqs]
    dout = [[torch.empty_like(t) for t in d] for d in din]
    streams = [torch.cuda.ExternalStream(p.stream()) for p in plans]

    def step(j):
        plans[j].encode_device([t.data_ptr() for t in din[j]])
        plans[j].decode_device([t.data_ptr() for t in dout[j]])

    for _ in range(3):
        th = [threading.Thread(target=step, args=(j,)) for j in range(K)]
        [t.start() for t in th]
        [t.join() for t in th]
    torch.cuda.synchronize()
    times = []
    for it in range(5):
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        for st in streams:
            st.wait_event(start)
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]

        def work(j):
            step(j)
            ends[j].record(streams[j])
        th = [threading.Thread(target=work, args=(j,)) for j in range(K)]
        [t.start() for t in th]
        [t.join() for t in th]
        torch.cuda.synchronize()
        times.append(max(start.elapsed_time(e) for e in ends))
    ms = float(np.median(times))
    vf = sum(s.n * s.F for _, s in seqs)
    print(f"{name} K={K}: {ms:.2f} ms per step of {K} sequences -> {vf / ms / 1e3:.1f} M vertex-frames/s",
          flush=True)
    for p in plans:
        p.close()
    for c in codecs:
        c.close()
