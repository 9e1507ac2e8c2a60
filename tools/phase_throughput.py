"""Which phase bounds the in-flight throughput?  K plans on K contexts run
only encodes, only decodes, or both, concurrently (one host thread each);
device time from one start event to the last plan stream's end event.
python tools/phase_throughput.py c1 4"""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec as C  # noqa: E402
from paper_2111_10105_b200.shard import sequence_for_rank  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = 5
seqs = [sequence_for_rank(name, j) for j in range(K)]
spec = seqs[0][0]
cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
codecs = [C.Codec(0) for _ in range(K)]
plans = [C.Plan(codecs[j], s.n, s.F, s.faces, cfg) for j, (_, s) in enumerate(seqs)]
din = [[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in s.axes] for _, s in seqs]
dout = [[torch.empty_like(t) for t in d] for d in din]
streams = [torch.cuda.ExternalStream(p.stream()) for p in plans]


def run(mode):
    def one(j):
        for _ in range(reps):
            if mode in ("enc", "both"):
                plans[j].encode_device([t.data_ptr() for t in din[j]])
            if mode in ("dec", "both"):
                plans[j].decode_device([t.data_ptr() for t in dout[j]])
    for j in range(K):
        one(j)  # warm (graphs captured)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    th = [threading.Thread(target=one, args=(j,)) for j in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / (reps * K)
    st = plans[0].stats()
    return ms, st


for mode in ("enc", "dec", "both"):
    ms, st = run(mode)
    print(f"K={K} {mode}: {ms:.3f} ms per sequence (wall / (reps*K)); single-plan stats "
          f"enc {st['ms_encode']:.3f} dec {st['ms_decode']:.3f} launches "
          f"{st['kernel_launches_encode']}+{st['kernel_launches_decode']}", flush=True)
