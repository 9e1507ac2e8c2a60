import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec, synth
spec = synth.CONFIGS["c3"]; s = spec.make(); cd = codec.Codec(0)
cfg = codec.EncoderConfig(k_l=spec.k, row_bits=[spec.bits] * spec.k, oi_rounds=spec.rounds)
pin = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).pin_memory().numpy() for x in s.axes]
hs = synth.Sequence(s.faces, pin)
out = [torch.empty(x.shape, dtype=torch.float32).pin_memory().numpy() for x in s.axes]
enc_buf = None
for it in range(4):
    t0 = time.perf_counter(); enc = cd.encode(hs, cfg, out=enc_buf)
    if enc_buf is None:
        enc_buf = codec.CompressedAnimation.allocate(enc.n, enc.F, enc.k_l, enc.n_c, enc.faces, n_b=enc.n_b, pinned=True, variant=enc.variant)
    t1 = time.perf_counter(); st = cd.stats()
    cd.decode(enc, out=out, dtype=np.float32); t2 = time.perf_counter(); st2 = cd.stats()
    print(f"e2e encode {1e3*(t1-t0):.1f} decode {1e3*(t2-t1):.1f} | dev encode {st['ms_encode']:.1f} (delta {st['ms_delta']:.1f} gram {st['ms_gram']:.1f} basis {st['ms_basis']:.1f} proj {st['ms_project']:.1f}) | dev decode {st2['ms_decode']:.1f} recon {st2['ms_reconstruct']:.1f} factor {st2['ms_factor']:.1f} solve {st2['ms_solve']:.1f}", flush=True)
