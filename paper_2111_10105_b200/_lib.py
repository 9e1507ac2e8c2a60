"""ctypes declarations of libdmcg.so (include/dmcg.h).

The library is built in-tree by ``__graft_entry__.build()`` (make -C
paper_2111_10105_b200/csrc).  There is no fallback: importing the product
API without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdmcg.so")

u8p = ctypes.POINTER(ctypes.c_uint8)
u16p = ctypes.POINTER(ctypes.c_uint16)
u32p = ctypes.POINTER(ctypes.c_uint32)
f32p = ctypes.POINTER(ctypes.c_float)
f64p = ctypes.POINTER(ctypes.c_double)
intp = ctypes.POINTER(ctypes.c_int)
vp = ctypes.c_void_p

DMCG_OK = 0
DMCG_E_CUDA = 10
DMCG_F64, DMCG_F32 = 0, 1
DMCG_PCA, DMCG_PCA_Q, DMCG_V2V, DMCG_PCA_QS, DMCG_PCA_QP, DMCG_BLOCKS = 0, 1, 2, 3, 4, 5

# symbols declared in include/dmcg.h (tests check every one is exported)
EXPORTS = [
    "dmcg_abi_version", "dmcg_create", "dmcg_destroy", "dmcg_last_error", "dmcg_config_default",
    "dmcg_decode_options_default", "dmcg_encoded_sizes", "dmcg_encode", "dmcg_decode",
    "dmcg_serialize", "dmcg_parse_header", "dmcg_parse", "dmcg_parse_error", "dmcg_rate_exact",
    "dmcg_anchor_count", "dmcg_select_anchors", "dmcg_plan_create", "dmcg_plan_destroy",
    "dmcg_plan_encode_device", "dmcg_plan_decode_device", "dmcg_plan_download", "dmcg_plan_upload",
    "dmcg_plan_basis", "dmcg_plan_stats", "dmcg_ctx_stats", "dmcg_plan_stream", "dmcg_debug_chol",
    "dmcg_plan_serialize", "dmcg_plan_distortion", "dmcg_comm_unique_id", "dmcg_comm_create",
    "dmcg_comm_destroy", "dmcg_shard_layout", "dmcg_plan_create_shard", "dmcg_shard_info_get",
    "dmcg_shard_encode_device", "dmcg_shard_encode_phase", "dmcg_shard_buffer",
    "dmcg_build_connectivity", "dmcg_host_error", "dmcg_ozaki_gemm", "dmcg_plan_delta",
    "dmcg_plan_set_kernel_timing",
]


class DmcgConfig(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("k_l", ctypes.c_uint32), ("row_bits", intp),
                ("n_row_bits", ctypes.c_uint32), ("n_b", ctypes.c_uint16), ("t_max", ctypes.c_int),
                ("anchor_fraction", ctypes.c_double), ("anchor_bits", ctypes.c_int),
                ("dict_bits", ctypes.c_int), ("diff_bits", ctypes.c_int),
                ("anchor_strategy", ctypes.c_int), ("seed", ctypes.c_uint64),
                ("laplacian", ctypes.c_int), ("raw_payload", ctypes.c_int),
                ("oi_rounds", ctypes.c_int), ("oi_seed", ctypes.c_uint64),
                ("oi_implicit", ctypes.c_int), ("oi_tolerance", ctypes.c_double)]


class DmcgDecodeOptions(ctypes.Structure):
    _fields_ = [("cg_rtol", ctypes.c_double), ("cg_max_iter", ctypes.c_int),
                ("solver", ctypes.c_int), ("refine", ctypes.c_int), ("reuse_factor", ctypes.c_int),
                ("frame_begin", ctypes.c_uint32), ("frame_count", ctypes.c_uint32)]


class DmcgShardInfo(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("row_begin", ctypes.c_uint32), ("row_end", ctypes.c_uint32),
                ("n_own", ctypes.c_uint32), ("n_halo", ctypes.c_uint32), ("n_loc", ctypes.c_uint32),
                ("anchor_begin", ctypes.c_uint32), ("anchor_end", ctypes.c_uint32),
                ("stage_begin", ctypes.c_uint64), ("stage_count", ctypes.c_uint64),
                ("gather_count", ctypes.c_uint64)]


class DmcgSeq(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("F", ctypes.c_uint32), ("dtype", ctypes.c_int),
                ("axes", vp * 3), ("faces", u32p), ("n_faces", ctypes.c_uint32)]


class DmcgEncoded(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("F", ctypes.c_uint32), ("k_l", ctypes.c_uint32),
                ("n_c", ctypes.c_uint32), ("n_faces", ctypes.c_uint32),
                ("variant", ctypes.c_uint8), ("flags", ctypes.c_uint8),
                ("anchor_bits", ctypes.c_uint8), ("dict_bits", ctypes.c_uint8),
                ("diff_bits", ctypes.c_uint8), ("faces", u32p), ("dict_q", u16p * 3),
                ("row_min", f32p * 3), ("row_max", f32p * 3), ("row_bits", u8p * 3),
                ("coeff_q", u16p * 3), ("anchor_idx", u32p), ("anchor_min", ctypes.c_float * 3),
                ("anchor_max", ctypes.c_float * 3), ("anchor_q", u16p * 3), ("means", f32p * 3),
                ("n_b", ctypes.c_uint16), ("pad", ctypes.c_uint16),
                ("diff_min", f32p * 3), ("diff_max", f32p * 3)]


class DmcgSizes(ctypes.Structure):
    _fields_ = [(k, ctypes.c_size_t) for k in ("dict_q", "rows", "coeff_q", "anchor_idx", "anchor_q",
                                              "means", "dict_ranges")] + \
        [("n_b", ctypes.c_uint16), ("pad", ctypes.c_uint16)]


class DmcgSections(ctypes.Structure):
    _fields_ = [(k, ctypes.c_size_t) for k in (
        "header", "connectivity", "dict_payload", "dict_ranges", "coeff_headers", "coeff_payload",
        "means", "anchor_indices", "anchor_ranges", "anchor_payload")]


class DmcgStats(ctypes.Structure):
    _fields_ = [("cg_iterations_max", ctypes.c_int), ("cg_rel_residual_max", ctypes.c_double),
                ("ms_encode", ctypes.c_float), ("ms_decode", ctypes.c_float),
                ("ms_delta", ctypes.c_float), ("ms_gram", ctypes.c_float),
                ("ms_basis", ctypes.c_float), ("ms_project", ctypes.c_float),
                ("ms_reconstruct", ctypes.c_float), ("ms_cg", ctypes.c_float),
                ("kernel_launches_encode", ctypes.c_int), ("kernel_launches_decode", ctypes.c_int),
                ("nnz_normal", ctypes.c_longlong), ("nnz_laplacian", ctypes.c_longlong),
                ("ms_factor", ctypes.c_float), ("ms_solve", ctypes.c_float), ("solver", ctypes.c_int),
                ("supernodes", ctypes.c_int), ("levels", ctypes.c_int),
                ("nnz_factor", ctypes.c_longlong), ("flops_factor", ctypes.c_double),
                ("flops_solve", ctypes.c_double), ("analyze_seconds", ctypes.c_double),
                ("ms_oi", ctypes.c_float), ("flops_oi", ctypes.c_double),
                ("ms_solve_fwd", ctypes.c_float), ("ms_solve_bwd", ctypes.c_float),
                ("flops_solve_fwd", ctypes.c_double), ("flops_solve_bwd", ctypes.c_double)]


_lib = None


def lib():
    """Loads libdmcg.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                           "(make -C paper_2111_10105_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    L.dmcg_abi_version.restype = ctypes.c_int
    L.dmcg_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
    L.dmcg_destroy.argtypes = [vp]
    L.dmcg_destroy.restype = None
    L.dmcg_last_error.argtypes = [vp]
    L.dmcg_last_error.restype = ctypes.c_char_p
    L.dmcg_config_default.argtypes = [ctypes.POINTER(DmcgConfig)]
    L.dmcg_config_default.restype = None
    L.dmcg_decode_options_default.argtypes = [ctypes.POINTER(DmcgDecodeOptions)]
    L.dmcg_decode_options_default.restype = None
    L.dmcg_encoded_sizes.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(DmcgConfig),
                                     ctypes.POINTER(DmcgSizes)]
    L.dmcg_encode.argtypes = [vp, ctypes.POINTER(DmcgSeq), ctypes.POINTER(DmcgConfig),
                              ctypes.POINTER(DmcgEncoded)]
    L.dmcg_decode.argtypes = [vp, ctypes.POINTER(DmcgEncoded), ctypes.POINTER(DmcgDecodeOptions),
                              vp * 3, ctypes.c_int]
    L.dmcg_serialize.restype = ctypes.c_size_t
    L.dmcg_serialize.argtypes = [ctypes.POINTER(DmcgEncoded), u8p, ctypes.c_size_t,
                                 ctypes.POINTER(DmcgSections)]
    L.dmcg_parse_header.argtypes = [u8p, ctypes.c_size_t, ctypes.POINTER(DmcgEncoded)]
    L.dmcg_parse.argtypes = [u8p, ctypes.c_size_t, ctypes.POINTER(DmcgEncoded),
                             ctypes.POINTER(DmcgSections)]
    L.dmcg_parse_error.restype = ctypes.c_char_p
    L.dmcg_rate_exact.argtypes = [ctypes.POINTER(DmcgSections), ctypes.c_uint32, ctypes.c_uint32,
                                  f64p]
    L.dmcg_rate_exact.restype = None
    L.dmcg_build_connectivity.argtypes = [u32p, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p,
                                          ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    L.dmcg_host_error.restype = ctypes.c_char_p
    L.dmcg_ozaki_gemm.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_long, ctypes.c_long,
                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_long,
                                  ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_void_p]
    L.dmcg_anchor_count.restype = ctypes.c_uint32
    L.dmcg_anchor_count.argtypes = [ctypes.c_uint32, ctypes.c_double]
    L.dmcg_select_anchors.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                      ctypes.c_uint64, u32p]
    L.dmcg_plan_create.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, u32p,
                                   ctypes.c_uint32, ctypes.POINTER(DmcgConfig), ctypes.POINTER(vp)]
    L.dmcg_plan_destroy.argtypes = [vp]
    L.dmcg_plan_destroy.restype = None
    L.dmcg_plan_encode_device.argtypes = [vp, vp * 3]
    L.dmcg_plan_decode_device.argtypes = [vp, ctypes.POINTER(DmcgDecodeOptions), vp * 3]
    L.dmcg_plan_download.argtypes = [vp, ctypes.POINTER(DmcgEncoded)]
    L.dmcg_plan_upload.argtypes = [vp, ctypes.POINTER(DmcgEncoded)]
    L.dmcg_plan_basis.argtypes = [vp, ctypes.c_int, f64p, f64p]
    L.dmcg_plan_delta.argtypes = [vp, ctypes.c_int, f64p]
    L.dmcg_plan_set_kernel_timing.argtypes = [vp, ctypes.c_int]
    L.dmcg_plan_stats.argtypes = [vp, ctypes.POINTER(DmcgStats)]
    L.dmcg_ctx_stats.argtypes = [vp, ctypes.POINTER(DmcgStats)]
    L.dmcg_plan_stream.argtypes = [vp]
    L.dmcg_plan_stream.restype = vp
    L.dmcg_plan_serialize.restype = ctypes.c_size_t
    L.dmcg_plan_serialize.argtypes = [vp, u8p, ctypes.c_size_t, ctypes.POINTER(DmcgSections)]
    L.dmcg_plan_distortion.argtypes = [vp, vp * 3, vp * 3, f64p, f64p, f64p]
    # multi-GPU vertex-row shards
    L.dmcg_comm_unique_id.argtypes = [u8p]
    L.dmcg_comm_create.argtypes = [ctypes.c_int, u8p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.dmcg_comm_destroy.argtypes = [vp]
    L.dmcg_comm_destroy.restype = None
    L.dmcg_shard_layout.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u32p, ctypes.c_uint32,
                                    ctypes.POINTER(DmcgConfig), ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(DmcgShardInfo), u32p]
    L.dmcg_plan_create_shard.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, u32p,
                                         ctypes.c_uint32, ctypes.POINTER(DmcgConfig), ctypes.c_int,
                                         ctypes.c_int, vp, ctypes.POINTER(vp)]
    L.dmcg_shard_info_get.argtypes = [vp, ctypes.POINTER(DmcgShardInfo), u32p]
    L.dmcg_shard_encode_device.argtypes = [vp, vp * 3]
    L.dmcg_shard_encode_phase.argtypes = [vp, ctypes.c_int, vp * 3]
    L.dmcg_shard_buffer.argtypes = [vp, ctypes.c_int, ctypes.POINTER(vp),
                                    ctypes.POINTER(ctypes.c_size_t)]
    _lib = L
    return L
