// Host launchers of the dmcg sm_100a kernels (one per .cu translation unit
// group).  All launches go to the caller's stream; none synchronise.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace dmcg {

// ---- encode.cu (compiled with --fmad=false) -----------------------------
// K1: delta = L * A^T per axis (src/laplacian.cpp:39-46), bit-exact order.
// f32 selects float input.  flags[0] |= 1<<axis on non-finite input.
cudaError_t launch_delta(cudaStream_t s, int n, int F, const uint32_t* lap_rp,
                         const uint32_t* lap_ci, const void* const x[3], bool f32, double* delta,
                         int* flags, int axis = -1);
// flags[0] |= 1 << axis on a non-finite coordinate (v2v: no K1 pass).
cudaError_t launch_check_finite(cudaStream_t s, int n, int F, const void* const x[3], bool f32,
                                int* flags);
// Sum split-K Gram partials in split order and symmetrise (spectral.cpp:37-38).
cudaError_t launch_reduce_sym(cudaStream_t s, int F, int splits, int nbatch, const double* part,
                              double* R, bool lower_only = false);
// Sum of split-K partials (row-major M x N) into column-major out (M x N).
cudaError_t launch_reduce_sum(cudaStream_t s, int M, int N, int splits, int nbatch,
                              const double* part, double* out);
// Dictionary levels over [-1, 1] (codec.cpp:122-129, 300-301).
cudaError_t launch_quant_dict(cudaStream_t s, long count, int bits, const double* U, uint16_t* q);
cudaError_t launch_init_keys(cudaStream_t s, long rows, unsigned long long* keys);
// quantize_rows (codec.cpp:244-265) from the row min/max keys.
cudaError_t launch_quant_rows(cudaStream_t s, int k, int n, const unsigned long long* keys,
                              const uint8_t* bits_in, const double* C, float* rmin, float* rmax,
                              uint8_t* rbits, uint16_t* q, int axis = -1);
// Anchor quantisation (codec.cpp:444-471), one CTA per axis.
cudaError_t launch_anchors(cudaStream_t s, int n_c, int F, const uint32_t* idx,
                           const void* const x[3], bool f32, int bits, float* rng, uint16_t* q,
                           unsigned long long* keys);
// Vertex-row shards: anchor min/max keys of the rows[na] local
// anchor rows (keys: 3 x (min, max) ordered keys), then their levels with
// the (allreduced) global widened range -> rng (3 x 2), q (3 x na x F).
cudaError_t launch_anchor_keys(cudaStream_t s, int na, int F, const uint32_t* rows,
                               const void* const x[3], bool f32, unsigned long long* keys);
cudaError_t launch_anchor_quant(cudaStream_t s, int na, int F, const uint32_t* rows,
                                const void* const x[3], bool f32, int bits,
                                const unsigned long long* keys, float* rng, uint16_t* q);
// keys[2 r] = ~keys[2 r] for r < rows (min half <-> max-reducible).
cudaError_t launch_flip_min_keys(cudaStream_t s, long rows, unsigned long long* keys);

// DMC1 payload bit packing (stream.cpp BitWriter, MSB first) into a zeroed
// byte buffer viewed as 32-bit words; base_byte = the section's byte offset.
cudaError_t launch_pack_uniform(cudaStream_t s, const uint16_t* sym, long count, int bits,
                                unsigned long long base_byte, uint32_t* out);
// rows x n symbols; row r at bit row_bitoff[r] of the section (~0: no payload).
cudaError_t launch_pack_rows(cudaStream_t s, const uint16_t* sym, long n, int rows,
                             const uint8_t* row_bits, const unsigned long long* row_bitoff,
                             unsigned long long base_byte, uint32_t* out);

// ---- basis.cu --------------------------------------------------------------
// Round-robin Jacobi eigensolver of symmetric m x m A (col-major, per
// batch).  work: nbatch * max(2 * m2 * (m2 + 1), kJacobiBlkWork) doubles
// (m2 = m + m%2; the block-Jacobi cluster kernel pads to 256).  Writes V
// (m x m) and w (m).  flags[3] set on non-convergence.
constexpr size_t kJacobiBlkWork = 256 * 256;
cudaError_t launch_jacobi(cudaStream_t s, int nbatch, int m, const double* A, double* work,
                          double* V, double* w, int* flags);
// Stable descending order of w: Vs[:, j] = V[:, idx[j]], ws[j] = w[idx[j]];
// ld = leading dimension (rows) of V.
cudaError_t launch_sort_basis(cudaStream_t s, int nbatch, int m, int ncols_store, const double* V,
                              const double* w, double* Vs, long vs_batch_stride, double* ws,
                              long ws_batch_stride);
// canonicalize_signs (spectral.cpp:41-47) on columns [c0, c0+ncols) of
// m-row column-major U (batch stride bs).
cudaError_t launch_canon_signs(cudaStream_t s, int nbatch, int m, int c0, int ncols, double* U,
                               long bs);
// Fused orthogonal iterations (one CTA per axis): Q0 = qr(start), `rounds`
// x {Z = R Q; Q = qr(Z)}, then H = Q^T R Q (symmetrised); R Q is spread over a
// cluster of CTAs per axis (Q doubles as its L2 staging buffer).  work:
// nbatch * 2 (F|1) k doubles (used when the pair does not fit in shared memory).
// mirror: oi_mirror_doubles(F, nbatch) doubles (the published block
// reflectors, read by the other CTAs of the cluster from L2).
cudaError_t launch_oi_fused(cudaStream_t s, int nbatch, int F, int k, int rounds, const double* R,
                            const double* start, double* Q, double* H, double* work, double* scr,
                            double* mirror);
size_t oi_mirror_doubles(int F, int nbatch);
// Q (F x k per batch) = thin Householder Q of Z (same kernel as the fused
// OI, QR only): one round of the implicit X (X^T Q) iteration.
cudaError_t launch_qr_cluster(cudaStream_t s, int nbatch, int F, int k, const double* Z,
                              double* Q, double* mirror);
// U[:, k:F] = columns k..F-1 of the full Householder Q of U[:, :k].
cudaError_t launch_complete(cudaStream_t s, int nbatch, int F, int k, double* U, double* work,
                            double* scr, double* mirror = nullptr);
// Per-axis scratch (doubles) of the blocked QR used by the two kernels above.
size_t qr_scratch_doubles(int F, int k);
cudaError_t launch_fill_zero(cudaStream_t s, double* p, long count);

// ---- decode.cu ------------------------------------------------------------
// Dequantiser parameters per retained row (QParams of quantize.cpp:15-20).
cudaError_t launch_row_params(cudaStream_t s, int k, const float* rmin, const float* rmax,
                              const uint8_t* rbits, double* rowp);
// dequantize_rows of the 3 k retained rows (q: 3k x n levels) into f64 out
// (3k x n); decode_dictionaries of U~[:, :k] over frames [f0, f0 + Fw) into
// out (3 x k x Fw).  flags |= 1 on a level out of range (CorruptPayload).
cudaError_t launch_dequant_rows(cudaStream_t s, int rows, int n, const uint16_t* q,
                                const double* rowp, const uint8_t* rbits, int* flags, double* out);
cudaError_t launch_dequant_dict(cudaStream_t s, int F, int k, int f0, int Fw, const uint16_t* q,
                                int bits, int* flags, double* out);
// rhs = L^T delta~ + S^T a (solver.cpp:77-80) in the CG column-block layout.
cudaError_t launch_rhs(cudaStream_t s, int n, int F, int W, int nblk, const uint32_t* lap_rp,
                       const uint32_t* lap_ci, const int32_t* anchor_pos, int n_c,
                       const uint16_t* anchor_q, const float* anchor_rng, int anchor_bits,
                       const double* D, double* B, int* flags);
// Column-block CG on M = L^T L + S^T S (K7).
cudaError_t launch_cg(cudaStream_t s, int n, int W, int nblk, const uint32_t* m_rp,
                      const uint32_t* m_ci, const float* m_val, double* X, double* R, double* P,
                      double* Q, double rtol, int maxit, int* iters, double* res);
cudaError_t launch_output(cudaStream_t s, int n, int F, const double* X, void* const out[3],
                          bool f32);
// distortion_report terms (metrics.cpp:67-129) of orig a vs recon b (3 axes,
// vertex-major n x F, f32 or f64): per-frame RMS and NMSVE (normalised
// Laplacian), per-vertex mean error (vme may be null).  work: 3 n F doubles.
cudaError_t launch_distortion(cudaStream_t s, int n, int F, const uint32_t* lap_rp,
                              const uint32_t* lap_ci, const void* const a[3],
                              const void* const b[3], bool f32, double* work, double* rms,
                              double* nmsve, double* vme);
// Row-major (n x 3F) variants used by the direct solver.  F = frames in the
// decoded window [f_off, f_off + F) of the F_all-frame sequence (anchor
// levels and the output arrays are indexed with F_all).
cudaError_t launch_rhs_rm(cudaStream_t s, int n, int F, int F_all, int f_off,
                          const uint32_t* lap_rp, const uint32_t* lap_ci, const int32_t* anchor_pos,
                          int n_c, const uint16_t* anchor_q, const float* anchor_rng,
                          int anchor_bits, const double* D, double* B, int* flags);
cudaError_t launch_output_rm(cudaStream_t s, int n, int F, int F_all, int f_off, const double* X,
                             void* const out[3], bool f32, const double* shift = nullptr,
                             int F_out = -1);  // frames written per axis (< 0: F)
// Anchor-free variants (pca / pca_q): per-frame vertex means of the input
// (codec.cpp:432-441) -> means (3 x F floats); the per-column shift of the
// mean-constrained solution (solver.cpp:129-131) -> shift (3 Fw doubles).
// partial: scratch of 3 x 64 x max(F, 3 Fw) doubles.
cudaError_t launch_frame_means(cudaStream_t s, int n, int F, const void* const x[3], bool f32,
                               double* partial, float* means);
cudaError_t launch_mean_shift(cudaStream_t s, int n, int Fw, int F_all, int f0, const double* X,
                              const float* means, double* partial, double* shift);

// ---- blocks.cu (variant blocks, n_b > 1) ----------------------------------
// pad_frames (codec.cpp:43-49): out (3 x n x Fp, plan dtype) = x with the
// last frame repeated into frames F..Fp-1.
cudaError_t launch_pad_frames(cudaStream_t s, int n, int F, int Fp, const void* const x[3],
                              bool f32, void* out);
// block_dictionaries (codec.cpp:149-172) after the per-block eigenbases:
// per axis, block 0 = Ueig[0]; block b > 0 = orthogonal_iterations(R_b,
// U_{b-1}, t_max, tol) (spectral.cpp:69-104) or, on RankDeficiency,
// Ueig[b]; then align_signs against U_{b-1} (spectral.cpp:122-131).
// R, Ueig, U: 3 x nb x kf x kf col-major; work: 3 x block_work_doubles(kf).
// flags[0] += number of blocks that fell back to the eigenbasis.
cudaError_t launch_block_chain(cudaStream_t s, int nb, int kf, int t_max, double tol,
                               const double* R, const double* Ueig, double* U, double* work,
                               int* flags);
size_t block_work_doubles(int kf);
// encode_dictionaries (codec.cpp:290-328, auto_realign): q (3 x nb x kf^2)
// = first block at dict_bits, then the closed-loop differences at
// diff_bits; rng (3 x (nb-1) x 2) their widened ranges.
cudaError_t launch_dict_encode_blocks(cudaStream_t s, int nb, int kf, int dict_bits,
                                      int diff_bits, const double* U, double* work, uint16_t* q,
                                      float* rng);
// decode_dictionaries (codec.cpp:330-349): Ud (3 x nb x kf^2); flags |= 1 on
// a level out of range.
cudaError_t launch_dict_decode_blocks(cudaStream_t s, int nb, int kf, int dict_bits,
                                      int diff_bits, const uint16_t* q, const float* rng,
                                      int* flags, double* Ud);
// anchor levels (3 x n_c x Fp): columns F..Fp-1 = column F-1 (the decoder's
// anchor padding, codec.cpp:483-495).
cudaError_t launch_pad_anchor_levels(cudaStream_t s, int n_c, int F, int Fp, uint16_t* q);

}  // namespace dmcg
