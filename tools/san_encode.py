"""compute-sanitizer driver: python tools/san_encode.py c0 -> one encode + decode."""
import sys

sys.path.insert(0, ".")
from paper_2111_10105_b200 import codec, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0"
cfg = synth.CONFIGS[name]
s = cfg.make()
cd = codec.Codec(0)
g = cd.encode(s, codec.EncoderConfig(k_l=cfg.k, row_bits=[cfg.bits] * cfg.k, oi_rounds=cfg.rounds))
cd.decode(g)
print("ok")
