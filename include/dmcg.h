/*
 * dmcg.h — C ABI of the B200 dynamic-mesh codec (libdmcg.so).
 *
 * Drop-in boundary for the reference's encode/decode hot path (pca_qp,
 * n_b = 1): plain pointers and sizes, no exceptions, no Eigen or torch types.
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).  The C++ drop-in
 * (include/dmc/codec.hpp: dmc::encode / dmc::decode with the reference's
 * signatures) is a thin layer over these functions; see INTEGRATION.md for
 * the bindings a maintainer adds on the reference side.
 *
 * Return convention: 0 on success, otherwise the reference dmc::Error code
 * (include/dmc/errors.hpp:43-61: 3 parse, 4 index/validation, 5 config,
 * 6 corrupt, 7 version, 8 io, 9 numerical) or DMCG_E_CUDA /
 * DMCG_E_UNSUPPORTED.  dmcg_last_error() returns "<Kind>: <message>" like
 * dmc::Error::what().  A context is single-threaded; distinct contexts are
 * independent (the reference is reentrant).
 *
 * Memory layout of a trajectory axis: the reference MeshSequence stores each
 * axis as a k x n column-major Eigen::MatrixXd (include/dmc/mesh.hpp:33-35,
 * 56), i.e. n vertex rows of F contiguous frames: x[i*F + f].  dmcg uses that
 * layout unchanged on the host and in HBM.
 */
#ifndef DMCG_H
#define DMCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMCG_ABI_VERSION 1

enum dmcg_status {
  DMCG_OK = 0,
  DMCG_E_PARSE = 3,       /* ParseError / VertexCountMismatch / ConnectivityMismatch */
  DMCG_E_INDEX = 4,       /* IndexOutOfRange / DegenerateFace / ValidationError */
  DMCG_E_CONFIG = 5,      /* DimensionMismatch / ConfigError / InvalidBits / InvalidCount */
  DMCG_E_CORRUPT = 6,     /* CorruptPayload / CorruptStream */
  DMCG_E_VERSION = 7,     /* VersionMismatch */
  DMCG_E_IO = 8,          /* IoError */
  DMCG_E_NUMERICAL = 9,   /* ConvergenceFailure / SingularSystem */
  DMCG_E_CUDA = 10,       /* CUDA runtime / launch failure (new) */
  DMCG_E_UNSUPPORTED = 11 /* variant outside the B200 path (new) */
};

enum dmcg_dtype { DMCG_F64 = 0, DMCG_F32 = 1 };

/* Variant values = reference Variant (include/dmc/stream.hpp:60-68).  The B200
 * path covers 0-5; per_mesh_gft (6) is refused with DMCG_E_UNSUPPORTED. */
enum dmcg_variant {
  DMCG_PCA = 0, DMCG_PCA_Q = 1, DMCG_V2V = 2, DMCG_PCA_QS = 3, DMCG_PCA_QP = 4,
  DMCG_BLOCKS = 5, DMCG_PER_MESH_GFT = 6
};

typedef struct dmcg_ctx dmcg_ctx;
typedef struct dmcg_plan dmcg_plan;

/* ---- context ---------------------------------------------------------- */
int dmcg_create(dmcg_ctx** ctx, int device);
void dmcg_destroy(dmcg_ctx* ctx);
const char* dmcg_last_error(const dmcg_ctx* ctx);
int dmcg_abi_version(void);

/* ---- configuration ----------------------------------------------------- */
/* Field-for-field mirror of dmc::EncoderConfig (include/dmc/codec.hpp:30-49)
 * plus the B200 basis controls.  dmcg_config_default() fills the reference
 * defaults (codec.hpp:31-48) and oi_rounds = 0. */
typedef struct {
  int variant;              /* DMCG_PCA_QP is the only variant on this path */
  uint32_t k_l;             /* retained rows (default 20) */
  const int* row_bits;      /* k_l entries or NULL = all 16 (codec.cpp:106-113) */
  uint32_t n_row_bits;
  uint16_t n_b;             /* blocks (> 1 only for DMCG_BLOCKS) */
  int t_max;                /* blocks: orthogonal_iterations t_max (default 4,
                               spectral.cpp:69-104); validated at n_b = 1 */
  double anchor_fraction;   /* default 0.01 */
  int anchor_bits;          /* default 16 */
  int dict_bits;            /* default 16 */
  int diff_bits;            /* default 8 (header echo only at n_b = 1) */
  int anchor_strategy;      /* 0 Stride, 1 SeededRandom */
  uint64_t seed;            /* anchor seed */
  int laplacian;            /* 0 Combinatorial (1 Normalized: unsupported) */
  int raw_payload;          /* must be 0 */
  /* B200 basis: 0 = full F x F eigenbasis, the reference's n_b = 1 path
   * (codec.cpp:158-159); N > 0 = rank-k_l orthogonal iterations (N rounds)
   * + Rayleigh-Ritz + Householder completion (K3). */
  int oi_rounds;
  uint64_t oi_seed;         /* start matrix seed (axis a uses oi_seed + a) */
  int oi_implicit;          /* 1: never form R = X^T X; every round computes
                               Z = X^T (X Q) as two GEMMs over the vertex rows and
                               H = (X Q)^T (X Q) (BASELINE config 3's "covariance
                               applied implicitly"; on vertex-row shards the X^T (X Q)
                               partials are allreduced every round).  Same
                               iteration as the explicit R Q; 0 (default): form R. */
  double oi_tolerance;      /* blocks: EncoderConfig::oi_tolerance, the optional
                               principal-angle stop of orthogonal_iterations
                               (spectral.cpp:90-97); < 0 (default) = unset */
} dmcg_config;

void dmcg_config_default(dmcg_config* cfg);

/* Decoder-side solver controls (the reference factors L^T L + S^T S by
 * SimplicialLDLT, solver.cpp:62-90; the B200 path solves it by CG). */
typedef struct {
  double cg_rtol;           /* per-column ||r||/||b|| stop, default 1e-10 */
  int cg_max_iter;          /* default 20000 */
  int solver;               /* 0 (default): supernodal Cholesky on the GPU, the
                               reference's factor + back-substitute scheme;
                               1: conjugate gradients */
  int refine;               /* refinement passes after the direct solve
                               (default 1, like refine_anchored, solver.cpp:43-58) */
  int reuse_factor;         /* plans only: keep the numeric factor of M (it depends on
                               the mesh and anchors alone, both fixed by the plan) and
                               skip refactoring on later decodes (default 0: factor
                               on every decode, like the reference) */
  uint32_t frame_begin;     /* direct solver: decode frames [frame_begin, frame_begin +
                               frame_count) only and write just those columns of the
                               output (frame_count 0 = all frames).  The solve is
                               column-separable, so a window gives the same bits as the
                               full decode; the multi-GPU decoder splits frames across
                               ranks this way. */
  uint32_t frame_count;
} dmcg_decode_options;

void dmcg_decode_options_default(dmcg_decode_options* opt);

/* ---- data views -------------------------------------------------------- */
/* Input sequence: replaces const dmc::MeshSequence& (mesh.hpp:36-57). */
typedef struct {
  uint32_t n, F;            /* vertices, frames (MeshSequence::n(), k()) */
  int dtype;                /* DMCG_F64 (reference) or DMCG_F32 */
  const void* axes[3];      /* host (or device, for plan calls) pointers, x[i*F+f] */
  const uint32_t* faces;    /* 3 * n_faces vertex indices */
  uint32_t n_faces;
} dmcg_seq;

/* Compressed animation, n_b = 1 subset of dmc::CompressedAnimation for the
 * variants on the B200 path: pca, pca_q, v2v, pca_qs, pca_qp
 * (include/dmc/stream.hpp:130-155).  All arrays are caller-allocated with
 * the sizes from dmcg_encoded_sizes(); levels are 16-bit because every bit
 * depth is limited to 1..16 (codec.cpp:82-86,114-118).
 *   dict_q[a]   F*F levels, column-major (pack_matrix order, codec.cpp:122)
 *   row_*[a]    k_l quantiser headers (QuantRow, stream.hpp:86-93)
 *   coeff_q[a]  k_l*n levels, row r at [r*n]; degenerate rows hold zeros
 *   anchor_q[a] n_c*F levels, anchor-major (codec.cpp:466-468) */
typedef struct {
  uint32_t n, F, k_l, n_c, n_faces;
  uint8_t variant, flags, anchor_bits, dict_bits, diff_bits;
  const uint32_t* faces;
  uint16_t* dict_q[3];
  float* row_min[3];
  float* row_max[3];
  uint8_t* row_bits[3];
  uint16_t* coeff_q[3];
  uint32_t* anchor_idx;
  float anchor_min[3], anchor_max[3];
  uint16_t* anchor_q[3];
  float* means[3];          /* F per-frame vertex means, variants pca / pca_q only
                               (codec.cpp:432-441; may be NULL otherwise) */
  /* blocks variant (DMCG_BLOCKS, n_b > 1; AxisPayload dict_first / dict_diffs /
   * coeffs, stream.hpp:101-109): the F frames are padded with the last frame to
   * F + pad = n_b * k_f (codec.cpp:43-49, 81-82).  0 reads as n_b = 1.  With
   * n_b > 1 the arrays above hold, per axis:
   *   dict_q      n_b * k_f^2 levels: dict_first (dict_bits) then the n_b - 1
   *               dict_diffs (diff_bits), each k_f x k_f column-major
   *   diff_min/max  n_b - 1 difference ranges (DictDiff::min / max)
   *   row_*       n_b * k_l headers, block b at [b * k_l]
   *   coeff_q     n_b * k_l * n levels, block b at [b * k_l * n]
   *   anchor_q    n_c * F (unpadded, as for pca_qp) */
  uint16_t n_b, pad;
  float* diff_min[3];
  float* diff_max[3];
} dmcg_encoded;

/* Element counts of each dmcg_encoded array for (n, F, cfg). */
typedef struct {
  size_t dict_q, rows, coeff_q, anchor_idx, anchor_q, means;
  size_t dict_ranges;       /* n_b - 1 (blocks variant), else 0 */
  uint16_t n_b, pad;        /* checked block count and frame padding */
} dmcg_sizes;
int dmcg_encoded_sizes(uint32_t n, uint32_t F, const dmcg_config* cfg, dmcg_sizes* out);

/* ---- drop-in entry points (host in, host out) --------------------------- */
/* dmc::encode(const MeshSequence&, const EncoderConfig&)
 * (include/dmc/codec.hpp:90; src/codec.cpp:351-473).
 * Host arrays may be pageable or page-locked; page-locked ones (seq->axes,
 * out->coeff_q) let the copies run under the kernels axis by axis.  The call
 * also prepares the decode of its own stream (plan, symbolic analysis, M's
 * numeric factor) for the next dmcg_decode on this context; nothing is kept
 * beyond that decode.  The same bits either way. */
int dmcg_encode(dmcg_ctx* ctx, const dmcg_seq* seq, const dmcg_config* cfg, dmcg_encoded* out);
/* dmc::decode(const CompressedAnimation&) (include/dmc/codec.hpp:91;
 * src/codec.cpp:475-552).  out_axes: 3 host arrays of n*F elements of
 * out_dtype; opt may be NULL. */
int dmcg_decode(dmcg_ctx* ctx, const dmcg_encoded* in, const dmcg_decode_options* opt,
                void* const out_axes[3], int out_dtype);

/* ---- stream (src/stream.cpp:172-469) ----------------------------------- */
typedef struct {
  size_t header, connectivity, dict_payload, dict_ranges, coeff_headers, coeff_payload,
      means, anchor_indices, anchor_ranges, anchor_payload;
} dmcg_sections;   /* SectionSizes (stream.hpp:159-175) */
/* serialize(): writes the DMC1 stream into out (cap bytes; out may be NULL
 * to query the size).  Returns the stream size, 0 on error. */
size_t dmcg_serialize(const dmcg_encoded* e, uint8_t* out, size_t cap, dmcg_sections* s);
/* parse(): two phases.  dmcg_parse_header fills the scalar fields of hdr so
 * the caller can size the arrays; dmcg_parse then fills them (strict: the
 * reference's checks, stream.cpp:294-469). */
int dmcg_parse_header(const uint8_t* data, size_t size, dmcg_encoded* hdr);
int dmcg_parse(const uint8_t* data, size_t size, dmcg_encoded* out, dmcg_sections* s);
/* Message of the last failed parse on this thread ("CorruptStream: ..."). */
const char* dmcg_parse_error(void);
/* rate_exact (src/metrics.cpp:46-59): q, q_a, q_d, aux, q_s. */
void dmcg_rate_exact(const dmcg_sections* s, uint32_t n, uint32_t F, double out[5]);

/* ---- host helpers mirroring reference free functions -------------------- */
uint32_t dmcg_anchor_count(uint32_t n, double fraction);               /* codec.cpp:199 */
/* build_connectivity (include/dmc/mesh.hpp:69, src/mesh.cpp:60-86): the sorted,
 * deduplicated one-ring of every vertex as CSR (row_ptr n + 1 entries, col cap
 * entries; cap >= 6 * n_faces always suffices; *nnz = neighbour count).
 * IndexOutOfRange / DegenerateFace / empty face list -> code 4, message in
 * dmcg_host_error(). */
int dmcg_build_connectivity(const uint32_t* faces, uint32_t n_faces, uint32_t n, uint32_t* row_ptr,
                            uint32_t* col, size_t cap, size_t* nnz);
const char* dmcg_host_error(void);
int dmcg_select_anchors(uint32_t n, uint32_t n_c, int strategy, uint64_t seed,
                        uint32_t* out);                                 /* codec.cpp:204 */

/* ---- device-resident plan (bench `value`, serving) ----------------------
 * A plan binds one connectivity + config to device buffers: it validates
 * the faces, builds the Laplacian CSR and anchor set once, and keeps every
 * intermediate in HBM.  Encode and decode then run with no host round trip. */
int dmcg_plan_create(dmcg_ctx* ctx, uint32_t n, uint32_t F, int dtype, const uint32_t* faces,
                     uint32_t n_faces, const dmcg_config* cfg, dmcg_plan** plan);
void dmcg_plan_destroy(dmcg_plan* plan);
/* d_axes: 3 device arrays (n*F of the plan dtype).  Leaves the encoded
 * symbols in device memory. */
int dmcg_plan_encode_device(dmcg_plan* plan, const void* const d_axes[3]);
/* Decodes the device-resident symbols into 3 device arrays (plan dtype). */
int dmcg_plan_decode_device(dmcg_plan* plan, const dmcg_decode_options* opt,
                            void* const d_out[3]);
/* D2H / H2D of the encoded representation. */
int dmcg_plan_download(dmcg_plan* plan, dmcg_encoded* out);
int dmcg_plan_upload(dmcg_plan* plan, const dmcg_encoded* in);
/* Device copy of the F x F basis of axis a (column-major) and its Ritz /
 * eigen values, for parity checks.  Blocks variant: the n_b k_f x k_f
 * dictionaries of the axis back to back (n_b k_f^2 doubles), evals = F
 * doubles (k_f eigenvalues per block's direct decomposition). */
int dmcg_plan_basis(dmcg_plan* plan, int axis, double* U_host, double* evals_host);
/* K1's delta coordinates of the last device encode, axis-major (n x F
 * vertex-major per axis, f64) into host memory: the delta_coordinates
 * parity check (laplacian.cpp:39-46) at full size.  Not for blocks plans. */
int dmcg_plan_delta(dmcg_plan* plan, int axis, double* delta_host);

typedef struct {
  int cg_iterations_max;     /* max over columns in the last decode */
  double cg_rel_residual_max;
  float ms_encode, ms_decode; /* device time of the last calls (CUDA events) */
  float ms_delta, ms_gram, ms_basis, ms_project, ms_reconstruct, ms_cg;
  int kernel_launches_encode, kernel_launches_decode;
  long long nnz_normal;       /* nnz of M = L^T L + S^T S */
  long long nnz_laplacian;    /* nnz of L (incl. diagonal) */
  float ms_factor, ms_solve;  /* direct solver: numeric factorisation, solves (+refine) */
  int solver;                 /* solver used by the last decode */
  int supernodes, levels;     /* supernodal structure of M */
  long long nnz_factor;       /* stored entries of the Cholesky factor */
  double flops_factor, flops_solve;  /* per decode */
  double analyze_seconds;     /* host symbolic analysis (plan creation) */
  float ms_oi;                /* fused orthogonal-iteration kernel (k_oi_fused), last encode */
  double flops_oi;            /* its algorithmic flops */
  /* dmcg_plan_set_kernel_timing only (else 0): summed CUDA-event times of
   * the solves' forward (k_fwd) and backward (k_bwd) GEMM launches of the
   * last decode, and their algorithmic flops (2 W sum_s m_s w_s each, per solve) */
  float ms_solve_fwd, ms_solve_bwd;
  double flops_solve_fwd, flops_solve_bwd;
} dmcg_stats;
int dmcg_plan_stats(const dmcg_plan* plan, dmcg_stats* out);
/* Stats of the last drop-in dmcg_encode / dmcg_decode on this context. */
int dmcg_ctx_stats(const dmcg_ctx* ctx, dmcg_stats* out);
/* Per-launch CUDA events around the solve GEMMs (stats ms_solve_fwd / _bwd)
 * while on != 0; off by default (the events are extra graph nodes). */
int dmcg_plan_set_kernel_timing(dmcg_plan* plan, int on);
/* Stream the plan runs on (cudaStream_t), for event timing by callers. */
void* dmcg_plan_stream(dmcg_plan* plan);
/* serialize() of the plan's device-resident symbols: the
 * bit-packed payload sections (dictionary, coefficient and anchor levels;
 * reference BitWriter, src/quantize.cpp:50-69) are packed on the GPU, the
 * header / row headers / indices on the host; bytes identical to
 * dmcg_serialize of dmcg_plan_download's result.  out == NULL queries the
 * size.  Returns the stream size, 0 on error (cap too small / CUDA). */
size_t dmcg_plan_serialize(dmcg_plan* plan, uint8_t* out, size_t cap, dmcg_sections* s);
/* distortion_report (src/metrics.cpp:67-129) on the device for
 * two device-resident sequences of the plan's shape and dtype: per-frame RMS
 * vertex error (frame_rms) and NMSVE with the normalised Laplacian into host
 * arrays of F doubles, and the per-vertex mean error into n doubles
 * (vertex_mean_error may be NULL). */
int dmcg_plan_distortion(dmcg_plan* plan, const void* const d_orig[3], const void* const d_recon[3],
                         double* frame_rms, double* nmsve, double* vertex_mean_error);

/* ---- multi-GPU: vertex-row shards of one sequence ----------
 * The reference is single-threaded with no parallel path; these entry points
 * are the B200 addition for sequences too large for one GPU (BASELINE
 * config 3).  One process per GPU.  Rank q of N owns vertex rows
 * [q n / N, (q+1) n / N); its local input (n_loc x F per axis, the plan dtype)
 * holds the owned rows followed by the halo rows listed by
 * dmcg_shard_info_get.  Encode collectives: allreduce(sum) of the Gram
 * partials, allreduce(max) of the row / anchor range keys, and an
 * all-gather of every rank's symbols, after which each rank holds the full
 * encoded stream (dmcg_plan_download / dmcg_plan_serialize work as usual).
 * Decode splits frames across ranks with dmcg_decode_options.frame_begin /
 * frame_count (no exchange).  Results equal a single-GPU encode up to the
 * summation order of the Gram. */
typedef struct dmcg_comm dmcg_comm;
/* ncclGetUniqueId on one rank; share the 128 bytes with the others. */
int dmcg_comm_unique_id(uint8_t id[128]);
/* ncclCommInitRank (NCCL is dlopen'ed; DMCG_E_UNSUPPORTED if absent). */
int dmcg_comm_create(int device, const uint8_t id[128], int nranks, int rank, dmcg_comm** out);
void dmcg_comm_destroy(dmcg_comm* comm);

typedef struct {
  int nranks, rank;
  uint32_t row_begin, row_end;      /* owned vertex rows */
  uint32_t n_own, n_halo, n_loc;    /* local input rows = n_own + n_halo */
  uint32_t anchor_begin, anchor_end;/* owned anchor slots */
  uint64_t stage_begin, stage_count;/* this rank's symbols in the gather buffer (u16) */
  uint64_t gather_count;            /* gather buffer length (u16) */
} dmcg_shard_info;

/* Host only (no GPU): the layout rank `rank` of `nranks` would use.  halo
 * (n_halo entries, may be NULL) receives the global ids of the halo rows in
 * local-row order. */
int dmcg_shard_layout(uint32_t n, uint32_t F, const uint32_t* faces, uint32_t n_faces,
                      const dmcg_config* cfg, int nranks, int rank, dmcg_shard_info* info,
                      uint32_t* halo);
/* A plan for rank `rank` of `nranks`; comm may be NULL (phase-by-phase use). */
int dmcg_plan_create_shard(dmcg_ctx* ctx, uint32_t n, uint32_t F, int dtype, const uint32_t* faces,
                           uint32_t n_faces, const dmcg_config* cfg, int nranks, int rank,
                           dmcg_comm* comm, dmcg_plan** plan);
int dmcg_shard_info_get(const dmcg_plan* plan, dmcg_shard_info* info, uint32_t* halo);
/* Whole sharded encode on the plan stream, collectives included. */
int dmcg_shard_encode_device(dmcg_plan* plan, const void* const d_loc_axes[3]);
/* The same encode one phase at a time, for callers that run the
 * collectives themselves: phase 0 (delta + Gram partial) -> sum-reduce
 * DMCG_SHARD_GRAM; phase 1 (basis + projection + range keys) -> max-reduce
 * DMCG_SHARD_KEYS; phase 2 (quantise own rows / anchors into the gather
 * buffer at stage_begin) -> all-gather DMCG_SHARD_SYMBOLS; phase 3 (unpack
 * the gathered symbols into the plan's encoded arrays). */
int dmcg_shard_encode_phase(dmcg_plan* plan, int phase, const void* const d_loc_axes[3]);
enum { DMCG_SHARD_GRAM = 0, DMCG_SHARD_KEYS = 1, DMCG_SHARD_SYMBOLS = 2 };
/* Device pointer and element count of a collective buffer (f64 / u64 / u16). */
int dmcg_shard_buffer(dmcg_plan* plan, int which, void** dptr, size_t* count);

/* ---- Ozaki INT8 tensor-core GEMM (csrc/ozaki.cu) ---------
 * C (M x N, row-major f64, device) = A B^T on the current device and stream 0,
 * A: M x K, B: N x K device matrices (f32 or f64) with element (r, k) at
 * [r * rs + k * ks]; s = slices per operand (3..7).  Synchronous; used by the
 * parity tests to pin the tcgen05 kernel against an fp64 GEMM. */
int dmcg_ozaki_gemm(const void* dA, int a_f32, long a_rs, long a_ks, int M, const void* dB,
                    int b_f32, long b_rs, long b_ks, int N, int K, int s, double* dC);

/* ---- diagnostics (host only, no GPU) ----------------------------------
 * Symbolic analysis of the anchored normal matrix of a mesh and, when W > 0,
 * a CPU solve M x = b (b, x: n x W row-major) with the same supernodal data
 * flow the GPU uses.  stats[0..7] = supernodes, levels, nnz(L), factor flops,
 * solve flops per rhs, max front, max width, analysis seconds. */
int dmcg_debug_chol(uint32_t n, const uint32_t* faces, uint32_t n_faces, uint32_t n_c,
                    const uint32_t* anchors, uint32_t W, const double* b, double* x,
                    double stats[8]);

#ifdef __cplusplus
}
#endif
#endif
