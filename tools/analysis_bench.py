"""Host-only timing of the decoder's mesh analysis (build_mesh, normal matrix,
chol_analyze) on a grid mesh: DMCG_TIMING=1 python tools/analysis_bench.py [nx] [reps]"""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2111_10105_b200 import _lib, synth  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
flags = sys.argv[3:]  # "cuda": with a live CUDA context; "thread": every rep on a fresh thread
if "cuda" in flags:
    import torch
    torch.zeros(1, device="cuda")
s = synth.grid(nx, nx, 2)
lib = _lib.lib()
u32p = ctypes.POINTER(ctypes.c_uint32)
f64p = ctypes.POINTER(ctypes.c_double)
fn = lib.dmcg_debug_chol
fn.argtypes = [ctypes.c_uint32, u32p, ctypes.c_uint32, ctypes.c_uint32, u32p, ctypes.c_uint32,
               f64p, f64p, f64p]
fn.restype = ctypes.c_int
faces = np.ascontiguousarray(s.faces, dtype=np.uint32)
n_c = lib.dmcg_anchor_count(s.n, ctypes.c_double(0.01))
anchors = np.zeros(n_c, dtype=np.uint32)
lib.dmcg_select_anchors(s.n, n_c, 0, ctypes.c_uint64(0), anchors.ctypes.data_as(u32p))
st = np.zeros(8)
if "tune" in flags:
    h = ctypes.c_void_p()
    lib.dmcg_create(ctypes.byref(h), 0)
for _ in range(reps):
    t0 = time.perf_counter()
    rcs = []

    def call():
        rcs.append(fn(s.n, faces.ctypes.data_as(u32p), len(faces), n_c,
                      anchors.ctypes.data_as(u32p), 0, None, None, st.ctypes.data_as(f64p)))

    if "thread" in flags:
        import threading
        th = threading.Thread(target=call)
        th.start()
        th.join()
    else:
        call()
    t1 = time.perf_counter()
    assert rcs[0] == 0
    print(f"analysis total {1e3 * (t1 - t0):.1f} ms: nsup {int(st[0])} levels {int(st[1])} "
          f"nnz(L) {int(st[2])} flops {st[3]:.3e} solve flops/rhs {st[4]:.3e} max front {int(st[5])}",
          flush=True)
