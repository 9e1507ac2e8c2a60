"""Short decode-only driver for ncu launch lists: python tools/decode_profile.py c1 [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = synth.CONFIGS[name]
s = spec.make()
cd = codec.Codec(0)
cfg = codec.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
npdt = np.float32 if spec.dtype == "f32" else np.float64
plan = codec.Plan(cd, s.n, s.F, s.faces, cfg, dtype=npdt)
d_in = [torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).cuda() for x in s.axes]
d_out = [torch.empty_like(t) for t in d_in]
for _ in range(reps):
    plan.encode_device([t.data_ptr() for t in d_in])
    plan.decode_device([t.data_ptr() for t in d_out])
    st = plan.stats()
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()})
