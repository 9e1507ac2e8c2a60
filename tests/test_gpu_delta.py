"""K1 delta coordinates (reference src/laplacian.cpp:39-46, called at
src/codec.cpp:419) read back from the device after an encode and compared
BIT FOR BIT with the oracle's orc_delta: the vectorised kernel (k_delta_vec,
16-byte loads, neighbour indices broadcast by shuffles) on f64 and f32 inputs
up to config 3's full size, the scalar kernel (DMCG_DELTA_SCALAR, and the
automatic fallback when rows are not 16-byte aligned), and the non-finite
check riding on the kernel (validate_sequence, codec.cpp:366)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import pyoracle as O
from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _device_delta(codec, s, k, rounds, f32):
    import torch
    npdt = np.float32 if f32 else np.float64
    cfg = C.EncoderConfig(k_l=k, row_bits=[12] * k, oi_rounds=rounds)
    plan = C.Plan(codec, s.n, s.F, s.faces, cfg, dtype=npdt)
    d_in = [torch.from_numpy(np.ascontiguousarray(x, dtype=npdt)).cuda() for x in s.axes]
    plan.encode_device([t.data_ptr() for t in d_in])
    out = [plan.delta(a) for a in range(3)]
    plan.close()
    return out


@pytest.mark.parametrize("name,f32", [("c0", False), ("c1", False), ("c2", True), ("c3", True),
                                      ("odd", False)])
def test_delta_bit_exact(codec, name, f32):
    if name == "odd":   # F = 7: rows are not 16-byte aligned -> scalar kernel
        s = synth.sphere(2, 7, 3, 0, seed=5)
        k, rounds = 4, 3
    else:
        spec = synth.CONFIGS[name]
        s = spec.make()
        k, rounds = spec.k, 2
    got = _device_delta(codec, s, k, rounds, f32)
    for a in range(3):
        x = s.axes[a].astype(np.float32).astype(np.float64) if f32 else s.axes[a]
        ref = O.delta(s.faces, x)
        assert np.array_equal(got[a], ref), (name, a, float(np.abs(got[a] - ref).max()))


def test_delta_scalar_kernel_bit_exact():
    """DMCG_DELTA_SCALAR=1 selects the scalar k_delta (read once per process)."""
    code = ("import sys; sys.path[:0] = ['tests', '.', 'oracle'];"
            "import numpy as np, pyoracle as O, test_gpu_delta as T;"
            "from paper_2111_10105_b200 import codec as C, synth;"
            "s = synth.CONFIGS['c1'].make(); cd = C.Codec(0);"
            "g = T._device_delta(cd, s, 64, 2, False);"
            "assert all(np.array_equal(g[a], O.delta(s.faces, s.axes[a])) for a in range(3));"
            "print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, DMCG_DELTA_SCALAR="1"))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("f32", [False, True])
def test_delta_flags_non_finite(codec, f32):
    s = synth.sphere(2, 16, 3, 0, seed=6)
    bad = [ax.copy() for ax in s.axes]
    bad[2][7, 9] = np.inf
    with pytest.raises(C.DmcError) as e:
        _device_delta(codec, synth.Sequence(s.faces, bad), 4, 2, f32)
    assert e.value.code == 4 and "axis z" in str(e.value)
