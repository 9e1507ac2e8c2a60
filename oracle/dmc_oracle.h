/*
 * dmc_oracle.h — CPU restatement of the reference dmc encode/decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or the timed CPU baseline — never as the product.
 *
 * The reference (/root/reference/proj, Eigen3-based C++) cannot be compiled
 * in this image: Eigen3 is required by CMakeLists.txt:11 and absent.  This
 * file restates, in plain C, each reference function on the pca_qp / n_b=1
 * path; every function cites the reference file:line it follows.  Where the
 * reference delegates to Eigen (SelfAdjointEigenSolver, SimplicialLDLT,
 * blocked GEMM), the published algorithm is restated (cyclic/round-robin
 * Jacobi, up-looking sparse LDL^T with nested-dissection ordering, plain
 * triple-loop GEMM); those results agree with Eigen to rounding, not bit for
 * bit.  Parity pins: SPEC.md's [OP] examples (tests/test_oracle_kat.py) and
 * numpy/scipy fixtures (tests/golden/, script tests/golden/make_golden.py).
 *
 * Compile with -ffp-contract=off: the reference Release build has no -march
 * (CMakeLists.txt:7-9), so Eigen's arithmetic has no FMA contraction.
 *
 * Layouts: a per-axis trajectory matrix is the reference's k x n column-major
 * Eigen::MatrixXd, i.e. n vertex rows of F contiguous frames (X[i*F + f]).
 * Dense F x F / F x p matrices are column-major.  Coefficient matrices are
 * row-major k_l x n (row r at C[r*n]), matching QuantRow order.
 */
#ifndef DMC_ORACLE_H
#define DMC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: the reference's dmc::Error codes (include/dmc/errors.hpp:43-61). */
enum {
  ORC_OK = 0,
  ORC_E_PARSE = 3,
  ORC_E_INDEX = 4,      /* IndexOutOfRange / DegenerateFace / ValidationError */
  ORC_E_CONFIG = 5,     /* DimensionMismatch / ConfigError / InvalidBits / InvalidCount */
  ORC_E_CORRUPT = 6,    /* CorruptPayload / CorruptStream */
  ORC_E_VERSION = 7,
  ORC_E_NUMERICAL = 9   /* ConvergenceFailure / RankDeficiency / SingularSystem */
};

/* ---- mesh.cpp ---------------------------------------------------------- */
/* build_connectivity (src/mesh.cpp:60-86): sorted, deduplicated one-ring
 * lists as CSR.  col must hold 6*m entries.  Returns nnz >= 0 or -code. */
long orc_build_connectivity(const uint32_t* faces, size_t m, uint32_t n,
                            uint32_t* row_ptr, uint32_t* col);
/* validate_sequence (src/mesh.cpp:108-136).  Returns a bitmask of issues:
 * 1 empty, 2 no faces, 4 isolated vertex, 8 not connected, 16 bad face,
 * 32/64/128 non-finite x/y/z.  0 = valid. */
int orc_validate(uint32_t n, uint32_t F, const uint32_t* faces, size_t m,
                 const double* ax, const double* ay, const double* az);

/* ---- laplacian.cpp ----------------------------------------------------- */
/* build_laplacian (src/laplacian.cpp:21-37), Combinatorial (kind 0) or
 * Normalized (kind 1).  lcol/lval hold n + nnz_adj entries; the diagonal
 * sits in its sorted column position. */
void orc_build_laplacian(uint32_t n, const uint32_t* adj_row, const uint32_t* adj_col,
                         int kind, uint32_t* lrow, uint32_t* lcol, double* lval);
/* delta_coordinates (src/laplacian.cpp:39-46): out = L * A^T (n x F,
 * vertex-major), accumulated in ascending column order per row, which is
 * the order of Eigen's column-major sparse x dense product. */
void orc_delta(uint32_t n, uint32_t F, const uint32_t* lrow, const uint32_t* lcol,
               const double* lval, const double* X, double* out);

/* ---- spectral.cpp ------------------------------------------------------ */
/* autocorrelation (src/spectral.cpp:35-39): R = 0.5*(A A^T + (A A^T)^T). */
void orc_autocorrelation(uint32_t n, uint32_t F, const double* X, double* R);
/* canonicalize_signs (src/spectral.cpp:41-47), column-major m x p. */
void orc_canonicalize_signs(uint32_t m, uint32_t p, double* U);
/* Symmetric eigensolver (round-robin Jacobi) — the restatement of Eigen's
 * SelfAdjointEigenSolver used by full_eigenbasis.  A (m x m, col-major) is
 * destroyed; V receives eigenvectors, w eigenvalues, both unsorted.
 * Returns sweeps used or -ORC_E_NUMERICAL. */
int orc_jacobi_eig(uint32_t m, double* A, double* V, double* w);
/* full_eigenbasis (src/spectral.cpp:49-67): descending order + canonical
 * signs. */
int orc_full_eigenbasis(uint32_t m, const double* R, double* U, double* evals);
/* orthogonal_iterations (src/spectral.cpp:69-104): t_max-1 rounds of
 * U <- Q(QR(R U)) with the RankDeficiency check; stop_tol < 0 = unset. */
int orc_orthogonal_iterations(uint32_t m, const double* R, const double* U_init,
                              int t_max, double stop_tol, double* U_out);
/* Thin Householder Q of an m x p matrix (m >= p); rank-safe (a vanishing
 * column gets tau = 0).  Restates Eigen::HouseholderQR::householderQ(). */
void orc_householder_q(uint32_t m, uint32_t p, const double* Z, double* Q);
/* Rank-k basis of the B200 path: seeded uniform start,
 * `rounds` orthogonal iterations on R, Rayleigh-Ritz, descending sort,
 * canonical signs, F x F completion.  rounds == 0 means the reference's
 * full_eigenbasis.  U is F x F, evals has F entries (Ritz values for the
 * first k; 0 for the completion). */
int orc_basis(uint32_t F, uint32_t k, const double* R, int rounds, uint64_t seed,
              double* U, double* evals);
/* subspace_angle (src/spectral.cpp:133-140): acos(sigma_min(U^T V)). */
double orc_subspace_angle(uint32_t m, uint32_t p, const double* U, const double* V);
/* OI start matrix shared with the GPU path: SplitMix64 stream, entry
 * = (next() >> 11) * 2^-52 - 1, uniform in [-1, 1) and exact in binary64
 * (no libm, so host and device agree bit for bit). */
void orc_start_matrix(uint64_t seed, size_t count, double* out);

/* ---- quantize.cpp / codec.cpp ----------------------------------------- */
void orc_widened_range(double lo, double hi, float* flo, float* fhi); /* codec.cpp:31-41 */
uint32_t orc_quantize(float mn, float mx, int bits, double x);      /* quantize.cpp:22-29 */
double orc_dequantize(float mn, float mx, int bits, uint32_t level); /* quantize.cpp:31-38 */
uint32_t orc_anchor_count(uint32_t n, double fraction);             /* codec.cpp:199-202 */
int orc_select_anchors(uint32_t n, uint32_t n_c, int strategy, uint64_t seed,
                       uint32_t* out);                               /* codec.cpp:204-242 */
/* quantize_rows (src/codec.cpp:244-265): C row-major (rows x n). */
void orc_quantize_rows(uint32_t k_l, uint32_t n, const double* C, const int* row_bits,
                       float* rmin, float* rmax, uint32_t* q);
/* dequantize_rows (src/codec.cpp:267-288) -> m x n row-major. */
int orc_dequantize_rows(uint32_t k_l, uint32_t m, uint32_t n, const float* rmin,
                        const float* rmax, const uint8_t* rbits, const uint32_t* q,
                        double* out);

/* ---- solver.cpp -------------------------------------------------------- */
/* solve_anchored, Parallel mode (src/solver.cpp:62-90): normal equations
 * L^T L + S^T S factored by sparse LDL^T, one refinement pass
 * (solver.cpp:43-58).  delta, X: n x W vertex-major; anchors: n_c x W.
 * nthreads > 1 splits the right-hand sides across threads. */
int orc_solve_anchored(uint32_t n, const uint32_t* lrow, const uint32_t* lcol,
                       const double* lval, uint32_t W, const double* delta,
                       uint32_t n_c, const uint32_t* idx, const double* anchors,
                       double* X, int nthreads);

/* ---- encode / decode (src/codec.cpp:351-552, pca_qp, n_b = 1) ----------- */
typedef struct {
  uint32_t n, F, k_l, n_c, n_faces;
  int anchor_bits, dict_bits, diff_bits;
  const uint32_t* faces;      /* 3 * n_faces */
  uint32_t* dict_q[3];        /* F*F, column-major (pack_matrix order) */
  float* row_min[3];          /* k_l */
  float* row_max[3];
  uint8_t* row_bits[3];
  uint32_t* coeff_q[3];       /* k_l*n, row r at [r*n]; degenerate rows all 0 */
  uint32_t* anchor_idx;       /* n_c */
  float anchor_min[3], anchor_max[3];
  uint32_t* anchor_q[3];      /* n_c*F anchor-major */
  int variant;                /* stream.hpp:60-68: 0 pca, 1 pca_q, 2 v2v, 3 pca_qs, 4 pca_qp */
  float* means[3];            /* F per-frame vertex means (pca / pca_q), else unused */
  /* blocks variant (5): n_b blocks of k_f = (F + pad) / n_b padded frames.
   * n_b == 0 reads as 1.  With n_b > 1: dict_q[a] holds n_b * k_f^2 levels
   * (first block at dict_bits, then n_b - 1 differences at diff_bits, each
   * column-major); diff_min / diff_max[a] the n_b - 1 difference ranges;
   * row_*[a] n_b * k_l headers and coeff_q[a] n_b * k_l * n levels, block b at
   * row offset b * k_l; anchor_q stays n_c * F (unpadded). */
  uint32_t n_b, pad;
  float* diff_min[3];
  float* diff_max[3];
} orc_encoded;

typedef struct {
  double t_connectivity, t_gram, t_eigen, t_delta, t_project, t_quantize, t_anchors;
  double t_dict_decode, t_reconstruct, t_solve;
} orc_timing;

/* encode: rounds == 0 is the reference path (full_eigenbasis); rounds > 0
 * is the B200 path's rank-k basis restated.  U_out (3*F*F) and evals_out
 * (3*F) may be NULL.  timing may be NULL. */
int orc_encode(uint32_t n, uint32_t F, const double* const axes[3], const uint32_t* faces,
               uint32_t n_faces, uint32_t k_l, const int* row_bits, double anchor_fraction,
               int anchor_bits, int dict_bits, int rounds, uint64_t basis_seed,
               orc_encoded* out, double* U_out, double* evals_out, orc_timing* timing,
               int nthreads);
int orc_decode(const orc_encoded* in, double* const axes_out[3], orc_timing* timing,
               int nthreads);
/* encode for any n_b = 1 variant 0-4 (codec.cpp:351-473): v2v projects the
 * trajectories instead of delta (codec.cpp:416-417); pca / pca_q store the
 * per-frame vertex means (codec.cpp:432-441) and no anchors; pca_qs codes like
 * pca_qp.  orc_encode == orc_encode_variant(4, ...). */
int orc_encode_variant(int variant, uint32_t n, uint32_t F, const double* const axes[3],
                       const uint32_t* faces, uint32_t n_faces, uint32_t k_l, const int* row_bits,
                       double anchor_fraction, int anchor_bits, int dict_bits, int rounds,
                       uint64_t basis_seed, orc_encoded* out, double* U_out, double* evals_out,
                       orc_timing* timing, int nthreads);
/* blocks variant (codec.cpp:351-473 with n_b > 1): frames padded with the
 * last frame (pad_frames, codec.cpp:43-49); per block the k_f x k_f
 * autocorrelation; block 0 full_eigenbasis, later blocks warm-started
 * orthogonal_iterations (t_max, stop_tol < 0 = none) falling back to
 * full_eigenbasis on RankDeficiency, then align_signs (block_dictionaries,
 * codec.cpp:149-172); encode_dictionaries with difference coding and
 * auto-realignment (codec.cpp:290-328); per block coeffs = dicts[b]^T delta_b^T
 * quantised by rows; anchors as pca_qp.  out->n_b / pad are set here; the
 * caller sizes the arrays (see orc_encoded).  U_out: 3 * n_b * k_f^2 (the
 * unquantised dictionaries) or NULL.  variant must be 5. */
int orc_encode_blocks(uint32_t n, uint32_t F, const double* const axes[3], const uint32_t* faces,
                      uint32_t n_faces, uint32_t n_b, uint32_t k_l, const int* row_bits,
                      double anchor_fraction, int anchor_bits, int dict_bits, int diff_bits,
                      int t_max, double stop_tol, orc_encoded* out, double* U_out, int nthreads);
/* decode_dictionaries (codec.cpp:330-349): the n_b decoded k_f x k_f
 * dictionaries of axis a (col-major, block b at b * k_f^2). */
int orc_decode_dictionaries(const orc_encoded* in, int a, double* out);
/* solve_mean_constrained (src/solver.cpp:105-133): vertex 0 pinned, normal
 * equations of L[:, 1:] by sparse LDL^T, one refinement, per-column mean
 * shift to means[c].  delta, X: n x W vertex-major. */
int orc_solve_mean_constrained(uint32_t n, const uint32_t* lrow, const uint32_t* lcol,
                               const double* lval, uint32_t W, const double* delta,
                               const double* means, double* X, int nthreads);

/* ---- stream.cpp / metrics.cpp ------------------------------------------ */
typedef struct {
  size_t header, connectivity, dict_payload, dict_ranges, coeff_headers, coeff_payload,
      means, anchor_indices, anchor_ranges, anchor_payload;
} orc_sections;
/* serialize (src/stream.cpp:172-292) for pca_qp, n_b = 1.  out may be NULL
 * (size query).  Returns the stream size. */
size_t orc_serialize(const orc_encoded* e, uint8_t* out, orc_sections* s);
/* rate_exact (src/metrics.cpp:46-59): q, q_a, q_d, aux, q_s. */
void orc_rate_exact(const orc_sections* s, uint32_t n, uint32_t F, double out[5]);
/* frame_rms (src/metrics.cpp:67-79). */
void orc_frame_rms(uint32_t n, uint32_t F, const double* const a[3], const double* const b[3],
                   double* out);

#ifdef __cplusplus
}
#endif
#endif
