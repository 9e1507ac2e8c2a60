"""Python mirror of the reference codec interface (include/dmc/codec.hpp,
include/dmc/stream.hpp, include/dmc/metrics.hpp) over the libdmcg C ABI.

The reference is a C++ library; its drop-in on the B200 path is the C ABI in
include/dmcg.h (plus the C++ header include/dmc/codec.hpp).  This module is
the Python host side that the tests, smoke() and bench.py call: the same
names (``EncoderConfig``, ``encode``, ``decode``, ``serialize``, ``parse``,
``rate_exact``, ``select_anchors``, ``anchor_count``), the same argument
meaning and the same error taxonomy (``DmcError.code`` = dmc::Error::code()).
Every numeric operation runs in libdmcg.so on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence as Seq

import numpy as np

from . import _lib as L

ERROR_KINDS = {3: "ParseError", 4: "ValidationError", 5: "ConfigError", 6: "CorruptStream",
               7: "VersionMismatch", 8: "IoError", 9: "NumericalError", 10: "CudaError",
               11: "Unsupported"}


class DmcError(RuntimeError):
    """Mirror of dmc::Error (include/dmc/errors.hpp:24-34): .code, .kind."""

    def __init__(self, code: int, what: str):
        super().__init__(what)
        self.code = code
        self.kind = what.split(":", 1)[0] if ":" in what else ERROR_KINDS.get(code, "Error")


@dataclass
class EncoderConfig:
    """dmc::EncoderConfig (include/dmc/codec.hpp:30-49) + B200 basis controls."""
    variant: int = L.DMCG_PCA_QP
    k_l: int = 20
    row_bits: Seq[int] = ()        # empty = all 16 (codec.cpp:106-113)
    n_b: int = 1
    t_max: int = 4
    anchor_fraction: float = 0.01
    anchor_bits: int = 16
    dict_bits: int = 16
    diff_bits: int = 8
    anchor_strategy: int = 0       # 0 Stride, 1 SeededRandom
    seed: int = 0
    laplacian: int = 0             # Combinatorial
    raw_payload: bool = False
    oi_rounds: int = 0             # 0 = full eigenbasis (reference n_b = 1 path)
    oi_seed: int = 0
    oi_implicit: bool = False      # Z = X^T (X Q) per round instead of R Q (R never formed)
    oi_tolerance: Optional[float] = None  # blocks: principal-angle stop (spectral.cpp:90-97)

    def to_c(self):
        c = L.DmcgConfig()
        L.lib().dmcg_config_default(ctypes.byref(c))
        # the row-bit array lives as long as the struct that points at it (no
        # shared state on self: concurrent encodes may share one config)
        rb = np.ascontiguousarray(list(self.row_bits), dtype=np.int32)
        c._row_bits_keep = rb
        c.variant, c.k_l, c.n_b, c.t_max = self.variant, self.k_l, self.n_b, self.t_max
        c.row_bits = rb.ctypes.data_as(L.intp) if len(rb) else None
        c.n_row_bits = len(rb)
        c.anchor_fraction = self.anchor_fraction
        c.anchor_bits, c.dict_bits, c.diff_bits = self.anchor_bits, self.dict_bits, self.diff_bits
        c.anchor_strategy, c.seed, c.laplacian = self.anchor_strategy, self.seed, self.laplacian
        c.raw_payload = int(self.raw_payload)
        c.oi_rounds, c.oi_seed = self.oi_rounds, self.oi_seed
        c.oi_implicit = int(self.oi_implicit)
        c.oi_tolerance = -1.0 if self.oi_tolerance is None else float(self.oi_tolerance)
        return c


@dataclass
class CompressedAnimation:
    """dmc::CompressedAnimation (stream.hpp:130-155) for the variants pca,
    pca_q, v2v, pca_qs, pca_qp and blocks.

    dict_q[a] is (F, F) with dict_q[a][j, i] = level of U(i, j) (column-major
    pack order); coeff_q[a] is (k_l, n); anchor_q[a] is (n_c, F) (anchored
    variants); means[a] is (F,) float32 (pca / pca_q).  Blocks (n_b > 1, k_f =
    (F + pad) / n_b): dict_q[a] is (n_b, k_f, k_f) -- dict_first then the
    n_b - 1 dict_diffs, each [j, i] = level (i, j); diff_min / diff_max[a] the
    (n_b - 1,) difference ranges; row_*[a] (n_b * k_l,) and coeff_q[a]
    (n_b * k_l, n), block b at rows b * k_l."""
    n: int
    F: int
    k_l: int
    n_c: int
    faces: np.ndarray
    anchor_bits: int = 16
    dict_bits: int = 16
    diff_bits: int = 8
    variant: int = L.DMCG_PCA_QP
    dict_q: list = field(default_factory=list)
    row_min: list = field(default_factory=list)
    row_max: list = field(default_factory=list)
    row_bits: list = field(default_factory=list)
    coeff_q: list = field(default_factory=list)
    anchor_idx: Optional[np.ndarray] = None
    anchor_min: list = field(default_factory=lambda: [0.0] * 3)
    anchor_max: list = field(default_factory=lambda: [0.0] * 3)
    anchor_q: list = field(default_factory=list)
    means: list = field(default_factory=list)
    n_b: int = 1
    pad: int = 0
    diff_min: list = field(default_factory=list)
    diff_max: list = field(default_factory=list)

    @property
    def k_f(self) -> int:
        return (self.F + self.pad) // self.n_b

    @classmethod
    def allocate(cls, n, F, k_l, n_c, faces, n_b=1, pinned=False, **kw):
        """Zeroed arrays for an encode of this shape; pinned=True places the
        payload arrays in page-locked host memory (DMA-speed download/upload,
        for callers that reuse the object across encodes)."""
        c = cls(n, F, k_l, n_c, np.ascontiguousarray(faces, dtype=np.uint32), **kw)
        if pinned:
            import torch

            def zeros(shape, dt):
                t = torch.zeros(shape, dtype=getattr(torch, np.dtype(dt).name), pin_memory=True)
                return t.numpy()
        else:
            zeros = np.zeros
        c.n_b = max(int(n_b), 1)
        c.pad = (c.n_b - F % c.n_b) % c.n_b if c.n_b > 1 else 0
        kf = c.k_f
        rows = max(k_l, 1) * c.n_b
        c.dict_q = [zeros((F, F) if c.n_b == 1 else (c.n_b, kf, kf), np.uint16)
                    for _ in range(3)]
        c.diff_min = [np.zeros(max(c.n_b - 1, 1), np.float32) for _ in range(3)]
        c.diff_max = [np.zeros(max(c.n_b - 1, 1), np.float32) for _ in range(3)]
        c.row_min = [np.zeros(rows, np.float32) for _ in range(3)]
        c.row_max = [np.zeros(rows, np.float32) for _ in range(3)]
        c.row_bits = [np.zeros(rows, np.uint8) for _ in range(3)]
        c.coeff_q = [zeros((rows, n), np.uint16) for _ in range(3)]
        c.anchor_idx = np.zeros(max(n_c, 1), np.uint32)
        c.anchor_q = [zeros((max(n_c, 1), F), np.uint16) for _ in range(3)]
        c.means = [np.zeros(F, np.float32) for _ in range(3)]
        return c

    def to_c(self) -> L.DmcgEncoded:
        e = L.DmcgEncoded()
        e.n, e.F, e.k_l, e.n_c = self.n, self.F, self.k_l, self.n_c
        self.faces = np.ascontiguousarray(self.faces, dtype=np.uint32)
        e.n_faces = len(self.faces)
        e.variant, e.flags = self.variant, 0
        e.anchor_bits, e.dict_bits, e.diff_bits = self.anchor_bits, self.dict_bits, self.diff_bits
        e.faces = self.faces.ctypes.data_as(L.u32p)
        e.n_b, e.pad = self.n_b, self.pad
        for a in range(3):
            if self.n_b > 1:
                e.diff_min[a] = self.diff_min[a].ctypes.data_as(L.f32p)
                e.diff_max[a] = self.diff_max[a].ctypes.data_as(L.f32p)
            e.dict_q[a] = self.dict_q[a].ctypes.data_as(L.u16p)
            e.row_min[a] = self.row_min[a].ctypes.data_as(L.f32p)
            e.row_max[a] = self.row_max[a].ctypes.data_as(L.f32p)
            e.row_bits[a] = self.row_bits[a].ctypes.data_as(L.u8p)
            e.coeff_q[a] = self.coeff_q[a].ctypes.data_as(L.u16p)
            e.anchor_q[a] = self.anchor_q[a].ctypes.data_as(L.u16p)
            e.anchor_min[a] = self.anchor_min[a]
            e.anchor_max[a] = self.anchor_max[a]
            if len(self.means) == 3:
                e.means[a] = self.means[a].ctypes.data_as(L.f32p)
        e.anchor_idx = self.anchor_idx.ctypes.data_as(L.u32p)
        return e

    def refresh_from_c(self, e: L.DmcgEncoded):
        self.anchor_min = [float(e.anchor_min[a]) for a in range(3)]
        self.anchor_max = [float(e.anchor_max[a]) for a in range(3)]


def _decode_opts(rtol, max_iter, solver, refine, reuse_factor=False, frames=None):
    if solver not in ("direct", "cg"):
        raise ValueError(f"solver must be 'direct' or 'cg', not {solver!r}")
    f0, fc = (0, 0) if frames is None else (int(frames[0]), int(frames[1]) - int(frames[0]))
    return L.DmcgDecodeOptions(rtol, max_iter, 0 if solver == "direct" else 1, refine,
                               1 if reuse_factor else 0, f0, fc)


def _check(ctx, rc):
    if rc != L.DMCG_OK:
        msg = L.lib().dmcg_last_error(ctx).decode() if ctx else ERROR_KINDS.get(rc, "Error")
        raise DmcError(rc, msg)


class Codec:
    """Owns one dmcg_ctx (device, stream, device memory pool)."""

    def __init__(self, device: int = 0):
        import weakref
        self._plans = weakref.WeakSet()  # plans must die before the context
        self._ctx = ctypes.c_void_p()
        rc = L.lib().dmcg_create(ctypes.byref(self._ctx), device)
        if rc != L.DMCG_OK:
            raise DmcError(rc, f"CudaError: dmcg_create(device={device}) failed (code {rc})")

    def close(self):
        for p in list(self._plans):
            p.close()
        if self._ctx:
            L.lib().dmcg_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._ctx

    def encode(self, seq, cfg: EncoderConfig, out: Optional[CompressedAnimation] = None
               ) -> CompressedAnimation:
        """dmc::encode (include/dmc/codec.hpp:90; src/codec.cpp:351-473).  `out`:
        a CompressedAnimation of this shape to fill (e.g. allocate(..., pinned=True),
        reused across calls); a new one is allocated otherwise."""
        axes = [np.ascontiguousarray(a) for a in seq.axes]
        dt = L.DMCG_F32 if axes[0].dtype == np.float32 else L.DMCG_F64
        axes = [a.astype(np.float32 if dt else np.float64, copy=False) for a in axes]
        n, F = axes[0].shape
        faces = np.ascontiguousarray(seq.faces, dtype=np.uint32)
        s = L.DmcgSeq()
        s.n, s.F, s.dtype = n, F, dt
        for a in range(3):
            s.axes[a] = axes[a].ctypes.data
        s.faces = faces.ctypes.data_as(L.u32p)
        s.n_faces = len(faces)
        cc = cfg.to_c()
        sizes = L.DmcgSizes()
        L.lib().dmcg_encoded_sizes(n, F, ctypes.byref(cc), ctypes.byref(sizes))
        if out is None:
            out = CompressedAnimation.allocate(n, F, cfg.k_l, sizes.anchor_idx, faces, n_b=cfg.n_b,
                                               anchor_bits=cfg.anchor_bits, dict_bits=cfg.dict_bits,
                                               diff_bits=cfg.diff_bits, variant=cfg.variant)
        else:
            assert (out.n, out.F, out.k_l, out.n_c, out.n_b) == (n, F, cfg.k_l, sizes.anchor_idx,
                                                                 max(cfg.n_b, 1))
            out.faces = faces
            out.anchor_bits, out.dict_bits = cfg.anchor_bits, cfg.dict_bits
            out.diff_bits, out.variant = cfg.diff_bits, cfg.variant
        e = out.to_c()
        _check(self._ctx, L.lib().dmcg_encode(self._ctx, ctypes.byref(s), ctypes.byref(cc),
                                              ctypes.byref(e)))
        out.refresh_from_c(e)
        return out

    def decode(self, c: CompressedAnimation, rtol: float = 1e-10, max_iter: int = 20000,
               dtype=np.float64, solver: str = "direct", refine: int = 1, out=None, frames=None):
        """dmc::decode (include/dmc/codec.hpp:91; src/codec.cpp:475-552).
        Returns the three (n, F) axis arrays.  solver "direct" (supernodal
        Cholesky + refine passes, the reference scheme) or "cg".  frames=(f0, f1)
        decodes only those frames (other columns of `out` are left untouched)."""
        opt = _decode_opts(rtol, max_iter, solver, refine, frames=frames)
        if out is None:
            out = [np.empty((c.n, c.F), dtype=dtype) for _ in range(3)]
        else:  # caller-provided (e.g. pinned) host buffers
            assert all(o.shape == (c.n, c.F) and o.dtype == dtype and o.flags.c_contiguous
                       for o in out)
        ptrs = (ctypes.c_void_p * 3)(*[o.ctypes.data for o in out])
        e = c.to_c()
        _check(self._ctx, L.lib().dmcg_decode(self._ctx, ctypes.byref(e), ctypes.byref(opt), ptrs,
                                              L.DMCG_F32 if dtype == np.float32 else L.DMCG_F64))
        return out

    def stats(self) -> dict:
        st = L.DmcgStats()
        L.lib().dmcg_ctx_stats(self._ctx, ctypes.byref(st))
        return {k: getattr(st, k) for k, _ in L.DmcgStats._fields_}


class Plan:
    """Device-resident plan (dmcg_plan_*): one connectivity + config bound
    to HBM buffers; encode / decode take device pointers (e.g. torch
    tensors' data_ptr())."""

    def __init__(self, codec: Codec, n, F, faces, cfg: EncoderConfig, dtype=np.float64):
        self.codec = codec
        self.n, self.F, self.k_l = n, F, cfg.k_l
        self.dtype = L.DMCG_F32 if dtype == np.float32 else L.DMCG_F64
        self.faces = np.ascontiguousarray(faces, dtype=np.uint32)
        self._cfg = cfg.to_c()
        self._p = ctypes.c_void_p()
        _check(codec.handle, L.lib().dmcg_plan_create(codec.handle, n, F, self.dtype,
                                                      self.faces.ctypes.data_as(L.u32p),
                                                      len(self.faces), ctypes.byref(self._cfg),
                                                      ctypes.byref(self._p)))
        self.n_c = _n_anchors(n, cfg)
        self.cfg = cfg
        codec._plans.add(self)

    def close(self):
        if self._p:
            L.lib().dmcg_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def encode_device(self, d_axes):
        ptrs = (ctypes.c_void_p * 3)(*[int(p) for p in d_axes])
        _check(self.codec.handle, L.lib().dmcg_plan_encode_device(self._p, ptrs))

    def decode_device(self, d_out, rtol=1e-10, max_iter=20000, solver="direct", refine=1,
                      reuse_factor=False, frames=None):
        """reuse_factor: keep the plan's numeric factor of M across decodes (many
        sequences on one mesh); off by default (the reference factors every call).
        frames=(f0, f1): decode only frames f0..f1-1 (direct solver; writes only
        those columns of d_out) -- the multi-GPU decoder's frame split."""
        opt = _decode_opts(rtol, max_iter, solver, refine, reuse_factor, frames)
        ptrs = (ctypes.c_void_p * 3)(*[int(p) for p in d_out])
        _check(self.codec.handle, L.lib().dmcg_plan_decode_device(self._p, ctypes.byref(opt), ptrs))

    def download(self) -> CompressedAnimation:
        out = CompressedAnimation.allocate(self.n, self.F, self.k_l, self.n_c, self.faces,
                                           n_b=self.cfg.n_b, anchor_bits=self.cfg.anchor_bits,
                                           dict_bits=self.cfg.dict_bits,
                                           diff_bits=self.cfg.diff_bits, variant=self.cfg.variant)
        e = out.to_c()
        _check(self.codec.handle, L.lib().dmcg_plan_download(self._p, ctypes.byref(e)))
        out.refresh_from_c(e)
        return out

    def upload(self, c: CompressedAnimation):
        e = c.to_c()
        _check(self.codec.handle, L.lib().dmcg_plan_upload(self._p, ctypes.byref(e)))

    def set_kernel_timing(self, on: bool):
        """CUDA events around every solve GEMM launch (stats ms_solve_fwd / _bwd)."""
        _check(self.codec.handle, L.lib().dmcg_plan_set_kernel_timing(self._p, 1 if on else 0))

    def delta(self, axis: int):
        """K1's delta coordinates (n x F, f64) of the last device encode."""
        d = np.zeros((self.n, self.F))
        _check(self.codec.handle, L.lib().dmcg_plan_delta(self._p, axis, d.ctypes.data_as(L.f64p)))
        return d

    def basis(self, axis: int):
        """(U, evals); blocks: U is (n_b, k_f, k_f), U[b] block b's dictionary."""
        nb = max(self.cfg.n_b, 1)
        if nb > 1:
            Fp = self.F + (nb - self.F % nb) % nb
            kf = Fp // nb
            U = np.zeros((nb, kf, kf))
            ev = np.zeros(Fp)
        else:
            U = np.zeros((self.F, self.F))  # column-major buffer -> U[j, i] = U(i, j)
            ev = np.zeros(self.F)
        _check(self.codec.handle, L.lib().dmcg_plan_basis(self._p, axis, U.ctypes.data_as(L.f64p),
                                                          ev.ctypes.data_as(L.f64p)))
        return np.ascontiguousarray(np.swapaxes(U, -1, -2)), ev

    def stats(self) -> dict:
        st = L.DmcgStats()
        L.lib().dmcg_plan_stats(self._p, ctypes.byref(st))
        return {k: getattr(st, k) for k, _ in L.DmcgStats._fields_}

    def stream(self) -> int:
        return L.lib().dmcg_plan_stream(self._p) or 0

    def distortion(self, d_orig, d_recon, vertex_errors=False):
        """distortion_report (src/metrics.cpp:67-129) on the GPU for two device
        sequences of this plan's shape: (frame_rms[F], nmsve[F], vertex_mean_error[n] or None)."""
        rms = np.zeros(self.F)
        nm = np.zeros(self.F)
        vme = np.zeros(self.n) if vertex_errors else None
        a = (ctypes.c_void_p * 3)(*[int(p) for p in d_orig])
        b = (ctypes.c_void_p * 3)(*[int(p) for p in d_recon])
        _check(self.codec.handle, L.lib().dmcg_plan_distortion(
            self._p, a, b, rms.ctypes.data_as(L.f64p), nm.ctypes.data_as(L.f64p),
            vme.ctypes.data_as(L.f64p) if vme is not None else None))
        return rms, nm, vme

    def serialize(self):
        """DMC1 bytes of the device-resident symbols, payload bit-packed on the
        GPU (dmcg_plan_serialize): (bytes, SectionSizes dict), identical to
        serialize(self.download())."""
        s = L.DmcgSections()
        size = L.lib().dmcg_plan_serialize(self._p, None, 0, ctypes.byref(s))
        if size == 0:
            _check(self.codec.handle, L.DMCG_E_CUDA)
        buf = np.zeros(size, np.uint8)
        got = L.lib().dmcg_plan_serialize(self._p, buf.ctypes.data_as(L.u8p), size, ctypes.byref(s))
        if got != size:
            _check(self.codec.handle, L.DMCG_E_CUDA)
        return buf.tobytes(), {f: getattr(s, f) for f, _ in L.DmcgSections._fields_}


# ---- stream / metrics / helpers (host C++ in libdmcg.so) --------------------

def serialize(c: CompressedAnimation):
    """serialize (src/stream.cpp:172-292): returns (bytes, SectionSizes dict)."""
    e = c.to_c()
    s = L.DmcgSections()
    size = L.lib().dmcg_serialize(ctypes.byref(e), None, 0, ctypes.byref(s))
    buf = np.zeros(size, np.uint8)
    got = L.lib().dmcg_serialize(ctypes.byref(e), buf.ctypes.data_as(L.u8p), size, ctypes.byref(s))
    assert got == size
    return buf.tobytes(), {k: getattr(s, k) for k, _ in L.DmcgSections._fields_}


def parse(data: bytes) -> CompressedAnimation:
    """parse (src/stream.cpp:294-469); raises DmcError like the reference."""
    buf = np.frombuffer(data, dtype=np.uint8).copy()
    hdr = L.DmcgEncoded()
    rc = L.lib().dmcg_parse_header(buf.ctypes.data_as(L.u8p), len(buf), ctypes.byref(hdr))
    if rc:
        raise DmcError(rc, L.lib().dmcg_parse_error().decode())
    c = CompressedAnimation.allocate(hdr.n, hdr.F, hdr.k_l, hdr.n_c,
                                     np.zeros((hdr.n_faces, 3), np.uint32), n_b=hdr.n_b,
                                     anchor_bits=hdr.anchor_bits, dict_bits=hdr.dict_bits,
                                     diff_bits=hdr.diff_bits, variant=hdr.variant)
    e = c.to_c()
    rc = L.lib().dmcg_parse(buf.ctypes.data_as(L.u8p), len(buf), ctypes.byref(e), None)
    if rc:
        raise DmcError(rc, L.lib().dmcg_parse_error().decode())
    c.refresh_from_c(e)
    return c


def rate_exact(c: CompressedAnimation) -> dict:
    """rate_exact (src/metrics.cpp:46-65)."""
    e = c.to_c()
    s = L.DmcgSections()
    L.lib().dmcg_serialize(ctypes.byref(e), None, 0, ctypes.byref(s))
    out = np.zeros(5)
    L.lib().dmcg_rate_exact(ctypes.byref(s), c.n, c.F, out.ctypes.data_as(L.f64p))
    return dict(zip(("q", "q_a", "q_d", "aux", "q_s"), out.tolist()))


def _n_anchors(n, cfg) -> int:
    """n_c of an encode (codec.cpp:374): anchored variants only."""
    return anchor_count(n, cfg.anchor_fraction) \
        if cfg.variant in (L.DMCG_PCA_QS, L.DMCG_PCA_QP, L.DMCG_BLOCKS) else 0


def anchor_count(n: int, fraction: float = 0.01) -> int:
    return int(L.lib().dmcg_anchor_count(n, fraction))


def select_anchors(n: int, n_c: int, strategy: int = 0, seed: int = 0) -> np.ndarray:
    out = np.zeros(max(n_c, 1), np.uint32)
    rc = L.lib().dmcg_select_anchors(n, n_c, strategy, seed, out.ctypes.data_as(L.u32p))
    if rc:
        raise DmcError(rc, f"InvalidCount: anchor count {n_c} outside 1..{n}")
    return out[:n_c]


_default = None


def _codec():
    global _default
    if _default is None:
        _default = Codec(0)
    return _default


def encode(seq, cfg: EncoderConfig) -> CompressedAnimation:
    return _codec().encode(seq, cfg)


def decode(c: CompressedAnimation, **kw):
    return _codec().decode(c, **kw)
