"""GPU vs host DMC1 serialisation time: python tools/serialize_bench.py c1 [c2 ...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec as C, synth  # noqa: E402

cd = C.Codec(0)
for name in sys.argv[1:] or ["c1"]:
    spec = synth.CONFIGS[name]
    s = spec.make()
    cfg = C.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
    plan = C.Plan(cd, s.n, s.F, s.faces, cfg, dtype=np.float32 if spec.dtype == "f32" else np.float64)
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in s.axes]
    plan.encode_device([t.data_ptr() for t in d])
    plan.serialize()
    t0 = time.perf_counter()
    for _ in range(3):
        gb, _ = plan.serialize()
    t1 = time.perf_counter()
    enc = plan.download()
    t2 = time.perf_counter()
    for _ in range(3):
        hb, _ = C.serialize(enc)
    t3 = time.perf_counter()
    assert gb == hb
    print(f"{name}: stream {len(gb) / 1e6:.2f} MB; dmcg_plan_serialize {1e3 * (t1 - t0) / 3:.2f} ms "
          f"(device symbols -> host bytes); download + host dmcg_serialize "
          f"{1e3 * (t2 - t1) + 1e3 * (t3 - t2) / 3:.2f} ms")
