"""Seeded synthetic inputs for the five BASELINE.json configs.

The paper's datasets are third-party and absent from this image; BASELINE.json
names synthetic stand-ins (shape, size and deformation) and this module builds
them through ``libdmcg_synth.so`` (csrc/synth/synth.cpp).  Under-specified
choices (std vs variance, bone layout, bump sizes, OI rounds / bits for
configs 3 and 4) are recorded in DESIGN.md §2 and fixed here.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def _synth_lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libdmcg_synth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() first")
        lib = ctypes.CDLL(path)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        vpp = ctypes.c_void_p * 3
        lib.dmcg_synth_icosphere_size.argtypes = [ctypes.c_int, u32p, u32p]
        lib.dmcg_synth_sphere.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_uint64, ctypes.c_int, u32p, vpp]
        lib.dmcg_synth_torus.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_uint32, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_uint64, ctypes.c_int, u32p, vpp]
        lib.dmcg_synth_grid.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_int, ctypes.c_uint64, ctypes.c_int, u32p, vpp]
        _lib = lib
    return _lib


@dataclass
class Sequence:
    """A mesh sequence in the reference layout (mesh.hpp:36-57): ``axes[a]``
    is (n, F) C-contiguous, i.e. the k x n column-major Eigen matrix."""
    faces: np.ndarray          # (m, 3) uint32
    axes: list                 # 3 x (n, F) float64 or float32
    name: str = ""

    @property
    def n(self) -> int:
        return self.axes[0].shape[0]

    @property
    def F(self) -> int:
        return self.axes[0].shape[1]


def _alloc(n, F, f32):
    dt = np.float32 if f32 else np.float64
    axes = [np.empty((n, F), dtype=dt) for _ in range(3)]
    ptrs = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in axes])
    return axes, ptrs


def sphere(level: int, F: int, lmax: int = 4, bones: int = 0, seed: int = 0, f32=False) -> Sequence:
    lib = _synth_lib()
    n = ctypes.c_uint32()
    m = ctypes.c_uint32()
    lib.dmcg_synth_icosphere_size(level, ctypes.byref(n), ctypes.byref(m))
    faces = np.empty((m.value, 3), dtype=np.uint32)
    axes, ptrs = _alloc(n.value, F, f32)
    rc = lib.dmcg_synth_sphere(level, F, lmax, bones, seed, int(f32),
                               faces.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ptrs)
    assert rc == 0
    return Sequence(faces, axes, f"ico{level}_F{F}_l{lmax}_b{bones}_s{seed}")


def torus(nu: int, nv: int, F: int, waves: int = 8, jitter: float = 1e-4, seed: int = 1,
          R=1.0, r=0.3, f32=False) -> Sequence:
    lib = _synth_lib()
    faces = np.empty((2 * nu * nv, 3), dtype=np.uint32)
    axes, ptrs = _alloc(nu * nv, F, f32)
    rc = lib.dmcg_synth_torus(nu, nv, R, r, F, waves, jitter, seed, int(f32),
                              faces.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ptrs)
    assert rc == 0
    return Sequence(faces, axes, f"torus{nu}x{nv}_F{F}_s{seed}")


def grid(nx: int, ny: int, F: int, bumps: int = 32, seed: int = 3, f32=True) -> Sequence:
    lib = _synth_lib()
    faces = np.empty((2 * (nx - 1) * (ny - 1), 3), dtype=np.uint32)
    axes, ptrs = _alloc(nx * ny, F, f32)
    rc = lib.dmcg_synth_grid(nx, ny, F, bumps, seed, int(f32),
                             faces.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ptrs)
    assert rc == 0
    return Sequence(faces, axes, f"grid{nx}x{ny}_F{F}_s{seed}")


@dataclass
class Config:
    """One BASELINE.json config: generator + codec settings (k = k_l, N OI
    rounds, row bits).  Codec defaults otherwise follow EncoderConfig
    (reference include/dmc/codec.hpp:30-49): 1% Stride anchors, 16-bit
    anchors and dictionary."""
    name: str
    k: int
    rounds: int
    bits: int
    dtype: str
    make: object = field(repr=False)
    batch: int = 1


CONFIGS = {
    # config 0: icosphere L4, F=64, k=32, 10 OI rounds, 12 bits, f64
    "c0": Config("c0", 32, 10, 12, "f64", lambda i=0: sphere(4, 64, 4, 0, seed=0)),
    # config 1: torus 96x96, F=200, k=64, 15 rounds, 12 bits, f64
    "c1": Config("c1", 64, 15, 12, "f64", lambda i=0: torus(96, 96, 200, seed=1)),
    # config 2: icosphere L6, F=256, l<=8 + 4-bone bend, k=128, 20 rounds, 10 bits
    "c2": Config("c2", 128, 20, 10, "f64", lambda i=0: sphere(6, 256, 8, 4, seed=2)),
    "c2f32": Config("c2f32", 128, 20, 10, "f32", lambda i=0: sphere(6, 256, 8, 4, seed=2, f32=True)),
    # config 3: 512x512 grid, F=512, k=256; rounds/bits unspecified -> 20 / 12
    "c3": Config("c3", 256, 20, 12, "f32", lambda i=0: grid(512, 512, 512, seed=3)),
    # config 4: 64 x icosphere L5, F=128, k=64; rounds/dtype unspecified -> 10 / f64
    "c4": Config("c4", 64, 10, 12, "f64", lambda i=0: sphere(5, 128, 4, 0, seed=1000 + i), batch=64),
}
