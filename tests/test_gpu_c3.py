"""Config 3 (BASELINE configs[3]: 512 x 512 jittered grid, 262 144 vertices,
F = 512, k = 256, 20 OI rounds, 12-bit, fp32 storage) against the CPU oracle —
the full P1-P6 contract of test_gpu_parity.check_parity, once with the
explicit covariance R = X^T X and once with the covariance applied implicitly
as X^T (X Q) (the form configs[3] names), plus the principal angle of the
20-round basis to the full eigenbasis.

The oracle runs on all host cores (about 50 s encode + 25 s per decode on the
16-core GPU box); its encode and end-to-end decode are computed once per
module and shared by the tests.  Reference path restated: src/codec.cpp:351-552.
"""
import numpy as np
import pytest

import pyoracle as O
from paper_2111_10105_b200 import codec as C
from paper_2111_10105_b200 import synth

from test_gpu_parity import (NTHREADS, _cfg, _log_counts, check_parity,
                             oi_vs_eigenbasis_angles)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SPEC = synth.CONFIGS["c3"]


@pytest.fixture(scope="module")
def c3():
    s = SPEC.make()
    o = O.encode(s, SPEC.k, SPEC.bits, rounds=SPEC.rounds, seed=0, nthreads=NTHREADS)
    xo = O.decode(o, nthreads=NTHREADS)
    return s, o, xo


def test_c3_parity_explicit_covariance(codec, c3):
    s, o, xo = c3
    check_parity(codec, s, SPEC, f32_out=True, oracle=o, oracle_x=xo, tag="c3-explicit")


def test_c3_parity_implicit_covariance(codec, c3):
    """oi_implicit = 1: every round is P = X Q, Z = X^T P (R never formed) —
    the same iteration as the oracle's R Q, so the same contract holds."""
    s, o, xo = c3
    check_parity(codec, s, SPEC, f32_out=True, implicit=True, oracle=o, oracle_x=xo,
                 tag="c3-implicit")


def test_c3_oi_basis_within_spec_angle_of_full_eigenbasis(codec, c3):
    import torch
    s, _, _ = c3
    plan = C.Plan(codec, s.n, s.F, s.faces, _cfg(SPEC), dtype=np.float32)
    d = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda() for x in s.axes]
    plan.encode_device([t.data_ptr() for t in d])
    angles = oi_vs_eigenbasis_angles(plan, s, SPEC.k)
    _log_counts({"case": "c3", "oi_vs_eigenbasis": angles})
    for r, ang in angles:
        assert r >= 1 and ang < 1e-3, angles


def test_c3_full_size_properties(codec, c3):
    """Size-independent properties: bvpv = the analytic BASELINE.md §2 value,
    serialize -> parse -> serialize identity, decode error < 1e-2 bbox."""
    s, _, _ = c3
    g = codec.encode(s, _cfg(SPEC))
    data, _ = C.serialize(g)
    assert abs(C.rate_exact(g)["q_s"] - 18.948) < 2e-3
    assert C.serialize(C.parse(data))[0] == data
    x = codec.decode(g, dtype=np.float32)
    bbox = float(np.linalg.norm([ax.max() - ax.min() for ax in s.axes]))
    err = max(np.abs(x[a] - s.axes[a]).max() for a in range(3))
    assert err < 1e-2 * bbox
