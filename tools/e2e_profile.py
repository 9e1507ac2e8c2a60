"""Drop-in e2e loop for host-phase timing: DMCG_TIMING=1 python tools/e2e_profile.py c1"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
spec = synth.CONFIGS[name]
s = spec.make()
cd = codec.Codec(0)
cfg = codec.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
npdt = np.float32 if spec.dtype == "f32" else np.float64
pin = [torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).pin_memory().numpy() for x in s.axes]
hs = synth.Sequence(s.faces, pin)
out = [torch.empty(x.shape, dtype=torch.float32 if npdt == np.float32 else torch.float64)
       .pin_memory().numpy() for x in s.axes]
enc_buf = None  # the stream in page-locked arrays after the first (warm-up) call, as in bench.py
for it in range(3):
    t0 = time.perf_counter()
    enc = cd.encode(hs, cfg, out=enc_buf)
    if enc_buf is None:
        enc_buf = codec.CompressedAnimation.allocate(enc.n, enc.F, enc.k_l, enc.n_c, enc.faces,
                                                     n_b=enc.n_b, pinned=True, variant=enc.variant)
    t1 = time.perf_counter()
    cd.decode(enc, out=out, dtype=npdt)
    t2 = time.perf_counter()
    print(f"e2e encode {1e3 * (t1 - t0):.2f} ms decode {1e3 * (t2 - t1):.2f} ms", flush=True)
