"""Ad-hoc GPU-vs-oracle diagnostic (not a test): python tools/gpu_check.py c0 [c1 ...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import pyoracle as O  # noqa: E402
from paper_2111_10105_b200 import codec, synth  # noqa: E402


def main(names):
    cd = codec.Codec(0)
    for name in names:
        cfg = synth.CONFIGS[name]
        s = cfg.make()
        n, F = s.n, s.F
        ec = codec.EncoderConfig(k_l=cfg.k, row_bits=[cfg.bits] * cfg.k, oi_rounds=cfg.rounds)
        t = time.time()
        g = cd.encode(s, ec)
        t_enc = time.time() - t
        st = cd.stats()
        t = time.time()
        o = O.encode(s, cfg.k, cfg.bits, rounds=cfg.rounds, seed=0, nthreads=8)
        t_oenc = time.time() - t
        print(f"== {name} n={n} F={F} k={cfg.k}: gpu encode {t_enc*1e3:.1f} ms (dev {st['ms_encode']:.2f} ms:"
              f" delta {st['ms_delta']:.2f} gram {st['ms_gram']:.2f} basis {st['ms_basis']:.2f}"
              f" proj {st['ms_project']:.2f}), oracle {t_oenc*1e3:.0f} ms")
        for a in range(3):
            dq = (g.dict_q[a].astype(np.int64) - o.dict_q[a].astype(np.int64))
            # agreeing columns: per column j compare levels
            col_ok = [(dq[j] == 0).all() for j in range(F)]
            rows_eq = [(g.coeff_q[a][r] == o.coeff_q[a][r]).mean() for r in range(cfg.k)]
            mm_eq = [(g.row_min[a][r] == o.row_min[a][r] and g.row_max[a][r] == o.row_max[a][r])
                     for r in range(cfg.k)]
            ev = o.evals[a]
            print(f" axis {a}: dict cols equal {sum(col_ok[:cfg.k])}/{cfg.k} (all {sum(col_ok)}/{F});"
                  f" anchors eq {np.array_equal(g.anchor_q[a], o.anchor_q[a])}"
                  f" rng eq {g.anchor_min[a] == o.anchor_min[a] and g.anchor_max[a] == o.anchor_max[a]}")
            print("   symbol-row match frac:", " ".join(f"{x:.3f}" for x in rows_eq[:24]))
            print("   minmax eq:", "".join("1" if x else "0" for x in mm_eq),
                  " ev/ev0:", " ".join(f"{x:.1e}" for x in (ev[:cfg.k] / ev[0])[:16]))
        gb, gs = codec.serialize(g)
        ob, os_ = O.serialize(o)
        print(" bytes equal:", gb == ob, len(gb), len(ob), "rate", codec.rate_exact(g)["q_s"], O.rate_exact(o)["q_s"])
        # decode parity: same stream through both decoders
        t = time.time()
        xg = cd.decode(g, rtol=1e-10)
        t_dec = time.time() - t
        st = cd.stats()
        t = time.time()
        xo = O.decode(o, nthreads=8)
        t_odec = time.time() - t
        bbox = float(np.linalg.norm([a.max() - a.min() for a in s.axes]))
        # decode the GPU stream with the oracle to isolate decoder parity
        og = O.Encoded(n, F, cfg.k, g.n_c, s.faces)
        for a in range(3):
            og.dict_q[a][:] = g.dict_q[a]
            og.row_min[a][:] = g.row_min[a][:cfg.k]
            og.row_max[a][:] = g.row_max[a][:cfg.k]
            og.row_bits[a][:] = g.row_bits[a][:cfg.k]
            og.coeff_q[a][:] = g.coeff_q[a][:cfg.k]
            og.anchor_q[a][:] = g.anchor_q[a]
            og.s.anchor_min[a] = g.anchor_min[a]
            og.s.anchor_max[a] = g.anchor_max[a]
        og.anchor_idx[:] = g.anchor_idx
        xog = O.decode(og, nthreads=8)
        dmax = max(np.abs(xg[a] - xog[a]).max() for a in range(3))
        rms_g = O.frame_rms(s.axes, xg).mean()
        rms_o = O.frame_rms(s.axes, xo).mean()
        print(f" decode: gpu {t_dec*1e3:.1f} ms (dev {st['ms_decode']:.2f}: recon {st['ms_reconstruct']:.2f}"
              f" factor {st['ms_factor']:.2f} solve {st['ms_solve']:.2f} | sup {st['supernodes']}"
              f" lev {st['levels']} nnzL {st['nnz_factor']:.3g} analyze {st['analyze_seconds']:.3f}s);"
              f" oracle {t_odec*1e3:.0f} ms")
        if "--cg" in sys.argv:
            xc = cd.decode(g, rtol=1e-10, solver="cg")
            stc = cd.stats()
            print(f"   cg: {stc['ms_cg']:.1f} ms, iters {stc['cg_iterations_max']};"
                  f" max|x_cg - x_direct|/bbox = {max(np.abs(xc[a]-xg[a]).max() for a in range(3))/bbox:.2e}")
        print(f"   same-stream max|x_gpu-x_cpu|/bbox = {dmax/bbox:.2e}; rmse gpu {rms_g:.4e} cpu {rms_o:.4e}"
              f" ratio-1 {rms_g/rms_o-1:.2e}")


if __name__ == "__main__":
    main([a for a in sys.argv[1:] if not a.startswith("--")] or ["c0"])
