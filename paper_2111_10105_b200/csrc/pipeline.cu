// Device orchestration of one plan: encode (K1 delta, K2 Gram, K3 basis,
// K4 projection + quantisation, K5 dictionary / anchors) and decode (K6
// dequantise + reconstruct + rhs, K7 CG), all on the context stream.
// Reference call stacks: src/codec.cpp:351-473 (encode), 475-552 (decode).
#include <cstring>
#include <string>

#include <functional>
#include "gemm.cuh"
#include "internal.h"
#include "ozaki.h"
#include "kernels.h"

namespace dmcg {

// DMCG_SYNC=1 synchronises after every launch so a fault names its kernel.
static bool debug_sync() {
  static const bool on = getenv("DMCG_SYNC") != nullptr;
  return on;
}

#define DMCG_TRY(expr)                                                            \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e == cudaSuccess && debug_sync()) _e = cudaDeviceSynchronize();          \
    if (_e != cudaSuccess)                                                        \
      return Status{DMCG_E_CUDA, std::string("CudaError: ") + cudaGetErrorString(_e) + \
                                     " at " #expr};                               \
  } while (0)

namespace {

// Event record that stays a timing point inside a CUDA graph capture.
cudaError_t record_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t err = cudaStreamIsCapturing(s, &cs);
  if (err != cudaSuccess) return err;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                             : cudaEventRecord(e, s);
}

// ---- GEMM operand loaders / epilogues specific to the codec --------------

// Projection epilogue (codec.cpp:420 + the row min/max of codec.cpp:253):
// C[b][m][n] row-major (k x n), per-row running min/max as ordered keys.
struct StoreCoeffMinMax {
  double* C;
  unsigned long long* keys;
  __device__ __forceinline__ void operator()(int b, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = mb + i * 8 + (lane >> 2);
      double lo = INFINITY, hi = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = nb + j * 8 + (lane & 3) * 2 + e;
          if (m < M && n < N) {
            const double v = wt.acc[i][j][e];
            C[((long)b * M + m) * N + n] = v;
            lo = fmin(lo, v);
            hi = fmax(hi, v);
          }
        }
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, 2));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, 2));
      if ((lane & 3) == 0 && m < M && lo <= hi) {
        atomicMin(&keys[2 * ((long)b * M + m)], ordered_key(lo));
        atomicMax(&keys[2 * ((long)b * M + m) + 1], ordered_key(hi));
      }
    }
  }
};

// Decode operand A(k = r, m = i) = dequantised coefficient c~(r, i) of axis
// b (dequantize_rows, codec.cpp:267-288).  Out-of-range levels set flag.
struct LoadCoeffDeq {
  static constexpr bool kKContig = false;
  const uint16_t* q;
  const double* rowp;
  const uint8_t* rbits;
  int* flags;
  int n, k;
  __device__ __forceinline__ double operator()(int b, int r, int i) const {
    const long row = (long)b * k + r;
    const uint32_t lv = q[row * n + i];
    const double min_ = rowp[2 * row], width = rowp[2 * row + 1];
    if (width == 0.0) return min_;
    if (lv >= (1u << rbits[row])) atomicOr(flags, 1);
    return dequantize_level(min_, width, false, lv);
  }
};

// Decode operand B(k = r, n = f) = U~(f, r), the dequantised dictionary
// (decode_dictionaries / unpack_matrix, codec.cpp:330-349, 131-142).
struct LoadDictDeq {
  static constexpr bool kKContig = false;
  const uint16_t* q;
  double width;
  uint32_t levels;
  int F;
  int* flags;
  int f0;  // first decoded frame (frame window, dmcg_decode_options)
  __device__ __forceinline__ double operator()(int b, int r, int f) const {
    const uint32_t lv = q[((long)b * F + r) * F + f0 + f];
    if (lv >= levels) atomicOr(flags, 1);
    return dequantize_level(-1.0, width, false, lv);
  }
};

// delta~ into the CG column-block layout: column c = b*F + f.
struct StoreCG {
  double* D;
  int n, F;
  __device__ __forceinline__ void operator()(int b, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int m = mb + r, f = nb + c;
          if (m < M && f < N) {
            const int col = b * F + f;
            D[((size_t)(col / kCB) * n + m) * kCB + col % kCB] = wt.acc[i][j][e];
          }
        }
  }
};

int pick_splits(int tiles, int nbatch, int K) {
  const int want = 2 * 148;
  int s = (want + tiles * nbatch - 1) / (tiles * nbatch);
  const int maxs = (K + kBK - 1) / kBK;
  if (s > maxs) s = maxs;
  if (s < 1) s = 1;
  return s;
}

template <typename T>
Status gram(dmcg_plan* p, const void* const x[3], int n) {
  cudaStream_t s = p->ctx->stream;
  const int F = (int)p->F;
  if (p->oz_slices) {
    // INT8 tensor cores, Ozaki slices (ozaki.h): exact int32 slice products,
    // fp64 combination; the partials go through the same ordered reduction
    int splits = 0;
    DMCG_TRY(oz_gram(s, x, std::is_same<T, float>::value, n, F, p->oz_slices, p->d_oz_q,
                     p->d_oz_max, p->d_part, &splits));
    // oz_gram computes the tiles that reach the lower triangle only (SYRK)
    DMCG_TRY(launch_reduce_sym(s, F, splits, 3, p->d_part, p->d_R, true));
    return Status::ok();
  }
  const int tiles = ((F + kBM - 1) / kBM) * ((F + kBN - 1) / kBN);
  int splits = pick_splits(tiles, 3, n);
  const long maxs = (long)(p->part_elems / (3L * F * F));
  if (splits > maxs) splits = (int)maxs;
  splits = gemm_splits(n, splits, nullptr);
  // R(f, g) = sum_i X(i, f) X(i, g): both operands X(k = i, m = f) = x[i*F + f].
  LoadDense3<T, false> la{(const T*)x[0], (const T*)x[1], (const T*)x[2], (long)F, 1L};
  DMCG_TRY(launch_gemm(s, 3, F, F, n, splits, la, la, StorePartial{p->d_part, 3}));
  DMCG_TRY(launch_reduce_sym(s, F, splits, 3, p->d_part, p->d_R));
  return Status::ok();
}

bool implicit_oi(const dmcg_plan* p) {
  return p->implicit && p->rounds > 0 && p->k > 0 && p->k < p->F;
}

// Algorithmic flops of the OI: explicit (rounds + 1) x {QR,
// R Q} + Q^T Z; implicit (rounds + 1) x {QR, X Q} + rounds x X^T P + P^T P
// over the plan's (or shard's) vertex rows.
double oi_flops(const dmcg_plan* p, double F, double k, double r, double qr) {
  if (!implicit_oi(p)) return 3.0 * ((r + 1.0) * (qr + 2.0 * F * F * k) + 2.0 * F * k * k);
  const double n = p->shard ? (double)p->shard->n_own : (double)p->n;
  return 3.0 * ((r + 1.0) * (qr + 2.0 * n * F * k) + r * 2.0 * n * F * k + 2.0 * n * k * k);
}

// The implicit orthogonal iterations (dmcg_config.oi_implicit; BASELINE
// config 3): R = X^T X is never formed.  Q0 = qr(start); every round
//   P = X Q (n x k, GEMM over frames),  Z = X^T P (F x k, split-K GEMM over
//   the vertex rows),  Q = qr(Z)  (k_oi_cluster in QR-only mode),
// then P = X Q and H = P^T P (= Q^T R Q, symmetrised like the oracle).  On a
// vertex-row shard X is the rank's rows and the Z / H partials are
// allreduced (sum) every round.  P lives in the coefficient buffer.
template <typename T>
Status implicit_oi(dmcg_plan* p, const void* const x[3], int nrows, dmcg_comm* comm, double* H) {
  cudaStream_t s = p->ctx->stream;
  const int F = (int)p->F, k = (int)p->k;
  const long Fk = (long)F * k, nk = (long)nrows * k;
  double* P = p->d_C;
  LoadDense3<T, true> lxk{(const T*)x[0], (const T*)x[1], (const T*)x[2], 1L, (long)F};   // X(i, f) by f
  LoadDense3<T, false> lxm{(const T*)x[0], (const T*)x[1], (const T*)x[2], (long)F, 1L};  // X(i, f) by i
  LoadDense<double, true> lq{p->d_Q, Fk, 1L, (long)F};
  LoadDense<double, true> lp{P, nk, 1L, (long)nrows};
  auto splits_for = [&](int M, int N) {
    const int tiles = ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
    long sp = pick_splits(tiles, 3, nrows);
    const long cap = (long)(p->part_elems / (3L * M * N));
    if (sp > cap) sp = cap;
    return gemm_splits(nrows, (int)(sp < 1 ? 1 : sp), nullptr);
  };
  DMCG_TRY(launch_qr_cluster(s, 3, F, k, p->d_start, p->d_Q, p->d_oi_mirror));
  for (int r = 0; r <= p->rounds; ++r) {
    // P = X Q: M = rows, N = k, K = F
    DMCG_TRY(launch_gemm(s, 3, nrows, k, F, 1, lxk, lq, StoreStrided{P, nk, 1L, (long)nrows}));
    if (r == p->rounds) break;
    // Z = X^T P: M = F, N = k, K = rows (split-K)
    const int sz = splits_for(F, k);
    DMCG_TRY(launch_gemm(s, 3, F, k, nrows, sz, lxm, lp, StorePartial{p->d_part, 3}));
    DMCG_TRY(launch_reduce_sum(s, F, k, sz, 3, p->d_part, p->d_Z));
    if (comm) {
      Status st = comm_allreduce_sum_f64(comm, p->d_Z, 3 * (size_t)Fk, s);
      if (!st.good()) return st;
    }
    DMCG_TRY(launch_qr_cluster(s, 3, F, k, p->d_Z, p->d_Q, p->d_oi_mirror));
  }
  // H = P^T P: M = N = k, K = rows (split-K), symmetrised
  const int sh = splits_for(k, k);
  DMCG_TRY(launch_gemm(s, 3, k, k, nrows, sh, lp, lp, StorePartial{p->d_part, 3}));
  DMCG_TRY(launch_reduce_sym(s, k, sh, 3, p->d_part, H));
  if (comm) return comm_allreduce_sum_f64(comm, H, 3 * (size_t)k * k, s);
  return Status::ok();
}

Status basis(dmcg_plan* p, const void* const x[3] = nullptr, int nrows = 0,
             dmcg_comm* comm = nullptr) {
  cudaStream_t s = p->ctx->stream;
  const int F = (int)p->F, k = (int)p->k;
  const long FF = (long)F * F;
  if (p->rounds <= 0 || k >= F || k == 0) {
    // Reference n_b = 1 path: full_eigenbasis (spectral.cpp:49-67).
    DMCG_TRY(launch_jacobi(s, 3, F, p->d_R, p->d_H, p->d_V, p->d_w, p->d_flags + 3));
    DMCG_TRY(launch_sort_basis(s, 3, F, F, p->d_V, p->d_w, p->d_U, FF, p->d_evals, F));
    DMCG_TRY(launch_canon_signs(s, 3, F, 0, F, p->d_U, FF));
    return Status::ok();
  }
  const long Fk = (long)F * k;
  // Q0 = qr(start); rounds x {Z = R Q; Q = qr(Z)}; H = Q^T R Q — one fused
  // kernel, one CTA per axis (basis.cu k_oi_fused).
  double* H = p->d_C;  // k x k scratch (coefficient buffer is free here)
  DMCG_TRY(record_event(p->ev[6], s));
  if (implicit_oi(p)) {
    H = p->d_Z;  // the coefficient buffer holds P; Z is dead after the last QR
    Status st = p->dtype == DMCG_F32 ? implicit_oi<float>(p, x, nrows, comm, H)
                                     : implicit_oi<double>(p, x, nrows, comm, H);
    if (!st.good()) return st;
  } else {
    DMCG_TRY(launch_oi_fused(s, 3, F, k, p->rounds, p->d_R, p->d_start, p->d_Q, H, p->d_H,
                             p->d_qr_scr, p->d_oi_mirror));
  }
  DMCG_TRY(record_event(p->ev[7], s));
  DMCG_TRY(launch_jacobi(s, 3, k, H, p->d_H, p->d_V, p->d_w, p->d_flags + 3));
  double* Ws = p->d_Z;  // k x k sorted Ritz vectors (Z is free)
  DMCG_TRY(launch_sort_basis(s, 3, k, k, p->d_V, p->d_w, Ws, (long)k * k, p->d_evals, F));
  // U[:, :k] = Q Ws: A(k = t, m = g) = Q[t*F + g], B(k = t, n = j) = Ws[j*k + t].
  LoadDense<double, false> lQm{p->d_Q, Fk, (long)F, 1L};
  LoadDense<double, true> lW{Ws, (long)k * k, 1L, (long)k};
  DMCG_TRY(launch_gemm(s, 3, F, k, k, 1, lQm, lW, StoreStrided{p->d_U, FF, 1L, (long)F}));
  DMCG_TRY(launch_canon_signs(s, 3, F, 0, k, p->d_U, FF));
  // Completion to F x F: columns k..F-1 of the full Householder Q of U_k, on
  // the side stream (it only feeds the dictionary levels; the projection
  // needs U_k alone).  enqueue_encode joins before quant_dict.
  cudaStream_t s2 = p->ctx->aux;
  DMCG_TRY(cudaEventRecord(p->ev_fork, s));
  DMCG_TRY(cudaStreamWaitEvent(s2, p->ev_fork, 0));
  DMCG_TRY(launch_complete(s2, 3, F, k, p->d_U, p->d_H, p->d_qr_scr, p->d_oi_mirror));
  DMCG_TRY(launch_canon_signs(s2, 3, F, k, F - k, p->d_U, FF));
  for (int a = 0; a < 3; ++a)
    DMCG_TRY(launch_fill_zero(s2, p->d_evals + (long)a * F + k, F - k));
  DMCG_TRY(cudaEventRecord(p->ev_join, s2));
  p->forked = true;
  return Status::ok();
}

}  // namespace

// Blocks variant operand: batch b = axis b / nb, block b % nb; element
// (k, i) of the block at p[axis] + block * off + k * sk + i * si.
template <typename T, bool KC>
struct LoadBlocks {
  static constexpr bool kKContig = KC;
  const T* p0;
  const T* p1;
  const T* p2;
  int nb;
  long off, sk, si;
  __device__ __forceinline__ const T* addr(int b, int k, int i) const {
    const int a = b / nb, blk = b - a * nb;
    return (a == 0 ? p0 : (a == 1 ? p1 : p2)) + blk * off + (long)k * sk + (long)i * si;
  }
  __device__ __forceinline__ double operator()(int b, int k, int i) const {
    return (double)*addr(b, k, i);
  }
};

// Blocks variant encode (codec.cpp:351-473 with n_b > 1): padded frames,
// every block's k_f x k_f autocorrelation and eigenbasis as batched
// launches over the 3 n_b blocks, the sequential warm-started OI chain and
// dictionary difference coder per axis, then the batched per-block
// projection + row quantisation and the anchors.
template <typename T>
static Status enqueue_encode_blocks_t(dmcg_plan* p, const void* const x[3]) {
  cudaStream_t s = p->ctx->stream;
  const int n = (int)p->n, Fp = (int)p->F, Fi = (int)p->F_in, nb = (int)p->nb, kf = (int)p->kf;
  const int kl = (int)p->k_l, k = (int)p->k, nbat = 3 * nb;
  const long kk = (long)kf * kf;
  const bool f32 = p->dtype == DMCG_F32;
  DMCG_TRY(cudaMemsetAsync(p->d_flags, 0, 8 * sizeof(int), s));
  DMCG_TRY(record_event(p->ev[0], s));
  const void* xs[3] = {x[0], x[1], x[2]};
  if (p->pad) {  // pad_frames (codec.cpp:43-49)
    DMCG_TRY(launch_pad_frames(s, n, Fi, Fp, x, f32, p->d_xpad));
    for (int a = 0; a < 3; ++a) xs[a] = (const T*)p->d_xpad + (size_t)a * n * Fp;
  }
  // delta of the padded trajectories (column-separable: block b's delta is
  // columns [b k_f, (b+1) k_f), codec.cpp:419)
  DMCG_TRY(launch_delta(s, n, Fp, p->d_lap_rp, p->d_lap_ci, xs, f32, p->d_delta, p->d_flags));
  DMCG_TRY(record_event(p->ev[1], s));
  // R_b = A_b A_b^T per block (spectral.cpp:35-39), split-K over vertices
  {
    const int tiles = ((kf + kBM - 1) / kBM) * ((kf + kBN - 1) / kBN);
    int splits = pick_splits(tiles, nbat, n);
    const long maxs = (long)(p->part_elems / ((long)nbat * kk));
    if (splits > maxs) splits = (int)maxs;
    splits = gemm_splits(n, splits, nullptr);
    LoadBlocks<T, false> lx{(const T*)xs[0], (const T*)xs[1], (const T*)xs[2], nb, (long)kf,
                            (long)Fp, 1L};
    DMCG_TRY(launch_gemm(s, nbat, kf, kf, n, splits, lx, lx, StorePartial{p->d_part, nbat}));
    DMCG_TRY(launch_reduce_sym(s, kf, splits, nbat, p->d_part, p->d_R));
  }
  DMCG_TRY(record_event(p->ev[2], s));
  // full_eigenbasis of every block (block 0's dictionary, the later blocks'
  // RankDeficiency fallback), then the OI chain + align_signs per axis
  DMCG_TRY(launch_jacobi(s, nbat, kf, p->d_R, p->d_H, p->d_V, p->d_w, p->d_flags + 3));
  DMCG_TRY(launch_sort_basis(s, nbat, kf, kf, p->d_V, p->d_w, p->d_bUeig, kk, p->d_evals, kf));
  DMCG_TRY(launch_canon_signs(s, nbat, kf, 0, kf, p->d_bUeig, kk));
  DMCG_TRY(launch_block_chain(s, nb, kf, p->t_max, p->oi_tol, p->d_R, p->d_bUeig, p->d_U,
                              p->d_bwork, p->d_flags + 5));
  DMCG_TRY(record_event(p->ev[3], s));
  // coeffs_b = dicts[b]^T delta_b^T, rows < k_l (codec.cpp:420), + quantize_rows
  if (kl > 0) {
    DMCG_TRY(launch_init_keys(s, 3L * k, p->d_keys));
    LoadDense<double, true> lU{p->d_U, kk, 1L, (long)kf};  // A(f, r) = U_b(f, r)
    const double* d = p->d_delta;
    const long nF = (long)n * Fp;
    LoadBlocks<double, true> lD{d, d + nF, d + 2 * nF, nb, (long)kf, 1L, (long)Fp};
    DMCG_TRY(launch_gemm(s, nbat, kl, n, kf, 1, lU, lD, StoreCoeffMinMax{p->d_C, p->d_keys}));
    if (!p->coeff_streamed)
      DMCG_TRY(launch_quant_rows(s, k, n, p->d_keys, p->d_row_bits + 3 * k, p->d_C, p->d_row_min,
                                 p->d_row_max, p->d_row_bits, p->d_coeff_q));
  }
  DMCG_TRY(record_event(p->ev[4], s));
  // anchors (codec.cpp:444-471): the padded frames repeat the last one, so
  // the range and the first F_in levels equal those of the unpadded input
  DMCG_TRY(launch_anchors(s, (int)p->n_c, Fp, p->d_anchor_idx, xs, f32, p->anchor_bits,
                          p->d_anchor_rng, p->d_anchor_q, p->d_keys + 6L * k));
  // encode_dictionaries (codec.cpp:290-328)
  DMCG_TRY(launch_dict_encode_blocks(s, nb, kf, p->dict_bits, p->diff_bits, p->d_U, p->d_bwork,
                                     p->d_dict_q, p->d_diff_rng));
  DMCG_TRY(record_event(p->ev[5], s));
  return Status::ok();
}

static Status enqueue_encode_blocks(dmcg_plan* p, const void* const x[3]) {
  return p->dtype == DMCG_F32 ? enqueue_encode_blocks_t<float>(p, x)
                              : enqueue_encode_blocks_t<double>(p, x);
}

// The decoder's numeric factor of M during the encode (see dmcg_plan::
// factor_pending): only once the plan's decode structures exist (after its
// first decode), for the direct solver of single-block, single-GPU plans.
static bool prefactor_on(const dmcg_plan* p) {
  static const bool off = getenv("DMCG_NO_PREFACTOR") != nullptr;
  return !off && p->decode_ready && p->nb == 1 && !p->shard && p->variant != DMCG_V2V &&
         p->cdev.P != nullptr;
}

// Fork: M's supernodal factor on the low-priority stream aux2 (it reads
// only the plan's mesh structures; the encode never touches F / Linv / P).
// after_stream = false: not ordered behind the plan stream (a fresh decode
// plan whose uploads went through aux2 itself: dmcg_encode's preparation).
static Status fork_prefactor(dmcg_plan* p, bool after_stream = true) {
  cudaStream_t s = p->ctx->stream, sf = p->ctx->aux2;
  if (after_stream) {
    DMCG_TRY(cudaEventRecord(p->ev_pf_fork, s));
    DMCG_TRY(cudaStreamWaitEvent(sf, p->ev_pf_fork, 0));
  }
  DMCG_TRY(cudaMemsetAsync(p->d_pf_flag, 0, sizeof(int), sf));
  DMCG_TRY(record_event(p->ev_pf0, sf));
  CholDev cd = p->cdev;
  cd.flags = p->d_pf_flag;
  DMCG_TRY(chol_factor_device(sf, cd, p->levels));
  DMCG_TRY(record_event(p->ev_pf1, sf));
  DMCG_TRY(cudaEventRecord(p->ev_pf_join, sf));
  return Status::ok();
}

Status plan_prefactor_async(dmcg_plan* p, bool after_stream) {
  if (!p->cdev.P || p->nb != 1 || p->shard) return Status{DMCG_E_UNSUPPORTED, "Unsupported: prefactor"};
  Status st = fork_prefactor(p, after_stream);
  if (!st.good()) return st;
  p->factor_pending = true;
  p->pf_unjoined = true;
  return Status::ok();
}

// Every kernel of one encode on the plan stream (no host synchronisation:
// capturable into a CUDA graph).
static Status enqueue_encode(dmcg_plan* p, const void* const x[3], bool prefactor) {
  if (p->nb > 1) {
    if (p->in_events)  // drop-in: the input axes arrive on the copy stream
      for (int a = 0; a < 3; ++a)
        DMCG_TRY(cudaStreamWaitEvent(p->ctx->stream, p->ctx->ev_in[a], 0));
    return enqueue_encode_blocks(p, x);
  }
  cudaStream_t s = p->ctx->stream;
  const int n = (int)p->n, F = (int)p->F, k = (int)p->k;
  const bool f32 = p->dtype == DMCG_F32;
  const long FF = (long)F * F;
  DMCG_TRY(cudaMemsetAsync(p->d_flags, 0, 8 * sizeof(int), s));
  DMCG_TRY(record_event(p->ev[0], s));
  if (prefactor) {
    Status st = fork_prefactor(p);
    if (!st.good()) return st;
  }
  Status st = Status::ok();
  if (p->in_events && p->oz_slices && variant_uses_delta(p->variant) && !implicit_oi(p)) {
    // drop-in encode, fp32 storage: K1 and the Gram slices / tiles of an axis
    // as soon as that axis has arrived (ctx->ev_in), under the next axis' H2D;
    // same kernels, K splits and partial slots as the batched calls below
    // (bit-identical delta and R).  ms_delta then covers these interleaved
    // launches and their waits, ms_gram the reduction.
    int splits = 0;
    for (int a = 0; a < 3; ++a) {
      DMCG_TRY(cudaStreamWaitEvent(s, p->ctx->ev_in[a], 0));
      DMCG_TRY(launch_delta(s, n, F, p->d_lap_rp, p->d_lap_ci, x, f32, p->d_delta, p->d_flags, a));
      DMCG_TRY(oz_gram_axis(s, a, x[a], f32, n, F, p->oz_slices, p->d_oz_q, p->d_oz_max,
                            p->d_part, &splits));
    }
    DMCG_TRY(record_event(p->ev[1], s));
    DMCG_TRY(launch_reduce_sym(s, F, splits, 3, p->d_part, p->d_R, true));
    DMCG_TRY(record_event(p->ev[2], s));
  } else {
    if (p->in_events)
      for (int a = 0; a < 3; ++a) DMCG_TRY(cudaStreamWaitEvent(s, p->ctx->ev_in[a], 0));
    // K1 delta coordinates (codec.cpp:419); v2v codes the trajectories.
    if (variant_uses_delta(p->variant))
      DMCG_TRY(launch_delta(s, n, F, p->d_lap_rp, p->d_lap_ci, x, f32, p->d_delta, p->d_flags));
    else
      DMCG_TRY(launch_check_finite(s, n, F, x, f32, p->d_flags));
    DMCG_TRY(record_event(p->ev[1], s));
    // K2 autocorrelation (spectral.cpp:35-39); the implicit OI never forms it.
    if (!implicit_oi(p)) st = f32 ? gram<float>(p, x, n) : gram<double>(p, x, n);
    if (!st.good()) return st;
    DMCG_TRY(record_event(p->ev[2], s));
  }
  // K3 basis.
  p->forked = false;
  st = basis(p, x, n);
  if (!st.good()) return st;
  DMCG_TRY(record_event(p->ev[3], s));
  // K4 projection coeffs = U_k^T delta^T (codec.cpp:420) + row min/max, then
  // quantize_rows (codec.cpp:426).
  if (k > 0) {
    DMCG_TRY(launch_init_keys(s, 3L * k, p->d_keys));
    LoadDense<double, true> lU{p->d_U, FF, 1L, (long)F};
    StoreCoeffMinMax ep{p->d_C, p->d_keys};
    if (variant_uses_delta(p->variant) && p->oz_proj_slices) {
      // INT8 tensor cores (Ozaki slices, ozaki.h): C[b](r, i) = sum_f U(f, r)
      // delta(i, f), the row ranges folded into the epilogue
      const int sp = p->oz_proj_slices;
      const long nF = (long)n * F;
      const double* d = p->d_delta;
      OzOperand A{{p->d_U, p->d_U + FF, p->d_U + 2 * FF}, false, (long)F, 1L, k, F, 3};
      OzOperand B{{d, d + nF, d + 2 * nF}, false, (long)F, 1L, n, F, 3};
      int8_t* qa = p->d_oz_q;
      int8_t* qb = qa + oz_slice_bytes(k, F, sp, 3);
      unsigned long long* ma = p->d_oz_max;
      unsigned long long* mb = ma + 3L * oz_rows_pad(k);
      OzStore out{p->d_C, (long)k * n, 0L, (long)n, 1L, p->d_keys};
      DMCG_TRY(oz_matmul(s, A, B, sp, qa, ma, qb, mb, out));
    } else if (variant_uses_delta(p->variant) && p->h_coeff_dst[0] && p->nb == 1) {
      // drop-in encode into page-locked arrays: projection and quantisation
      // axis by axis (same tiles and arithmetic as the batched launches), each
      // axis' symbols leaving on the copy stream under the next axis' GEMM
      const long kn = (long)k * n;
      for (int a = 0; a < 3; ++a) {
        LoadDense<double, true> lUa{p->d_U + a * FF, FF, 1L, (long)F};
        LoadDense<double, true> lDa{p->d_delta + (long)a * n * F, (long)n * F, 1L, (long)F};
        StoreCoeffMinMax epa{p->d_C + a * kn, p->d_keys + 2L * a * k};
        DMCG_TRY(launch_gemm(s, 1, k, n, F, 1, lUa, lDa, epa));
        DMCG_TRY(launch_quant_rows(s, k, n, p->d_keys, p->d_row_bits + 3 * k, p->d_C, p->d_row_min,
                                   p->d_row_max, p->d_row_bits, p->d_coeff_q, a));
        DMCG_TRY(cudaEventRecord(p->ctx->ev_q[a], s));
        DMCG_TRY(cudaStreamWaitEvent(p->ctx->copy, p->ctx->ev_q[a], 0));
        DMCG_TRY(cudaMemcpyAsync(p->h_coeff_dst[a], p->d_coeff_q + a * kn, kn * 2,
                                 cudaMemcpyDeviceToHost, p->ctx->copy));
      }
      DMCG_TRY(cudaEventRecord(p->ctx->ev_cp, p->ctx->copy));
      p->coeff_streamed = true;
    } else if (variant_uses_delta(p->variant)) {
      LoadDense<double, true> lD{p->d_delta, (long)n * F, 1L, (long)F};
      DMCG_TRY(launch_gemm(s, 3, k, n, F, 1, lU, lD, ep));
    } else if (f32) {  // v2v: coeffs = U^T traj (codec.cpp:416-417)
      LoadDense3<float, true> lX{(const float*)x[0], (const float*)x[1], (const float*)x[2], 1L,
                                 (long)F};
      DMCG_TRY(launch_gemm(s, 3, k, n, F, 1, lU, lX, ep));
    } else {
      LoadDense3<double, true> lX{(const double*)x[0], (const double*)x[1], (const double*)x[2],
                                  1L, (long)F};
      DMCG_TRY(launch_gemm(s, 3, k, n, F, 1, lU, lX, ep));
    }
    DMCG_TRY(launch_quant_rows(s, k, n, p->d_keys, p->d_row_bits + 3 * k, p->d_C, p->d_row_min,
                               p->d_row_max, p->d_row_bits, p->d_coeff_q));
  }
  DMCG_TRY(record_event(p->ev[4], s));
  // K5b anchors (codec.cpp:444-471) or the per-frame means (codec.cpp:432-441).
  if (p->n_c)
    DMCG_TRY(launch_anchors(s, (int)p->n_c, F, p->d_anchor_idx, x, f32, p->anchor_bits,
                            p->d_anchor_rng, p->d_anchor_q, p->d_keys + 6L * k));
  if (variant_uses_means(p->variant))
    DMCG_TRY(launch_frame_means(s, n, F, x, f32, p->d_colsum, p->d_means));
  // K5a dictionary levels (encode_dictionaries first block), after the
  // completion joined back from the side stream.
  if (p->forked) DMCG_TRY(cudaStreamWaitEvent(s, p->ev_join, 0));
  DMCG_TRY(launch_quant_dict(s, 3 * FF, p->dict_bits, p->d_U, p->d_dict_q));
  DMCG_TRY(record_event(p->ev[5], s));
  if (p->coeff_streamed)  // the plan stream's next wait covers the streamed symbols
    DMCG_TRY(cudaStreamWaitEvent(s, p->ctx->ev_cp, 0));
  if (prefactor) DMCG_TRY(cudaStreamWaitEvent(s, p->ev_pf_join, 0));  // join (graph capture)
  return Status::ok();
}

// CUDA graphs for plans that are reused (dmcg_plan_*): the ~50 encode and
// ~300 decode launches are replayed from one instantiated graph instead of
// being re-issued one by one (the stream launch rate, ~3.5 us per kernel on
// this host, would otherwise bound the small-kernel phases).  A graph is
// keyed by the caller's device pointers and options and re-captured when
// they change.  Off for the one-shot drop-in plans and under the debugging
// switches (DMCG_SYNC, DMCG_LEVEL_TIMING, DMCG_NO_GRAPH).
static bool graphs_allowed(const dmcg_plan* p) {
  static const bool env_off = getenv("DMCG_NO_GRAPH") || getenv("DMCG_SYNC") ||
                              getenv("DMCG_LEVEL_TIMING") || getenv("DMCG_DEBUG");
  return p->use_graphs && !env_off;
}

template <class Fn>
static Status run_graph(dmcg_plan* p, PlanGraph& g, const void* const key[4], long long opt_key,
                        const Fn& enqueue) {
  cudaStream_t s = p->ctx->stream;
  if (!graphs_allowed(p)) return enqueue();
  bool hit = g.exec != nullptr && g.opt_key == opt_key;
  for (int i = 0; i < 4 && hit; ++i) hit = g.key[i] == key[i];
  if (!hit) {
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    DMCG_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    Status st = enqueue();
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (!st.good()) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    DMCG_TRY(e);
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    DMCG_TRY(e);
    for (int i = 0; i < 4; ++i) g.key[i] = key[i];
    g.opt_key = opt_key;
  }
  DMCG_TRY(cudaGraphLaunch(g.exec, s));
  return Status::ok();
}

// Host-side wrapper used by host.cpp.
// between: host work to run after the launches are queued and before the
// stream is waited for (dmcg_encode prepares the next decode there).
Status plan_encode(dmcg_plan* p, const void* const x[3], const std::function<void()>* between) {
  p->rec_a_valid = false;  // the encode reuses the coefficient and slice buffers
  cudaStream_t s = p->ctx->stream;
  const int k = (int)p->k, F = (int)p->F;
  const void* key[4] = {x[0], x[1], x[2], nullptr};
  const bool pf = prefactor_on(p);
  PhaseTimer tm("plan_encode");
  {
    Status st = run_graph(p, p->g_encode, key, pf ? 1 : 0, [&] { return enqueue_encode(p, x, pf); });
    if (!st.good()) return st;
  }
  tm.lap("enqueue (host)");
  p->oi_timed = p->nb == 1 && p->rounds > 0 && k < F && k > 0;
  int flags[8];
  // (before the flags read-back: its pageable destination makes that copy wait
  // for the kernels on the host)
  if (between && *between) (*between)();
  DMCG_TRY(cudaMemcpyAsync(flags, p->d_flags, sizeof(flags), cudaMemcpyDeviceToHost, s));
  DMCG_TRY(cudaStreamSynchronize(s));
  float ms;
  cudaEventElapsedTime(&ms, p->ev[0], p->ev[5]);
  p->stats.ms_encode = ms;
  p->factor_pending = pf;
  if (pf) cudaEventElapsedTime(&p->ms_prefactor, p->ev_pf0, p->ev_pf1);
  cudaEventElapsedTime(&p->stats.ms_delta, p->ev[0], p->ev[1]);
  cudaEventElapsedTime(&p->stats.ms_gram, p->ev[1], p->ev[2]);
  cudaEventElapsedTime(&p->stats.ms_basis, p->ev[2], p->ev[3]);
  cudaEventElapsedTime(&p->stats.ms_project, p->ev[3], p->ev[4]);
  p->stats.ms_oi = 0.0f;
  p->stats.flops_oi = 0.0;
  if (p->oi_timed) {
    cudaEventElapsedTime(&p->stats.ms_oi, p->ev[6], p->ev[7]);
    // per axis: (rounds + 1) x {Householder factor 2Fk^2 - 2k^3/3, thin Q 2Fk^2 - 2k^3/3}
    // + (rounds + 1) x R Q (2F^2 k) + Q^T Z (2Fk^2)
    const double F = p->F, k = p->k, r = p->rounds;
    const double qr = 2.0 * (2.0 * F * k * k - 2.0 * k * k * k / 3.0);
    p->stats.flops_oi = oi_flops(p, F, k, r, qr);
    p->oi_timed = false;
  }
  p->stats.kernel_launches_encode =
      1 + 2 + (p->rounds > 0 && k < F ? 2 * p->rounds + 12 : 3) + 1 + (k > 0 ? 3 : 0) + 1;
  if (p->nb > 1) {
    p->stats.kernel_launches_encode = (p->pad ? 1 : 0) + 1 + 2 + 4 + (k > 0 ? 3 : 0) + 2;
    p->oi_fallbacks = flags[5];
  }
  if (flags[0]) {
    std::string axes;
    for (int a = 0; a < 3; ++a)
      if (flags[0] & (1 << a)) axes += (axes.empty() ? "" : ", ") + std::string(1, "xyz"[a]);
    return Status{DMCG_E_INDEX, "ValidationError: non-finite coordinate in axis " + axes};
  }
  if (flags[3])
    return Status{DMCG_E_NUMERICAL,
                  "ConvergenceFailure: symmetric eigendecomposition did not converge"};
  return Status::ok();
}


// ---- vertex-row shards (shard.cpp has the layout and NCCL) -----
// Phase 0: K1 delta of the owned rows (local CSR over owned + halo rows) and
// the symmetrised Gram partial of the owned rows into d_R.
// Phase 1: basis from the (allreduced) d_R, projection of the owned rows
// with per-row min / max keys, anchor keys; min halves complemented so one
// MAX allreduce combines every key.
// Phase 2: keys restored; owned rows and anchors quantised into this rank's
// slot of the gather buffer; dictionary levels.
// Phase 3: every rank's symbols (after the all-gather) unpacked into the
// plan's [3][k][n] / [3][n_c][F] encoded arrays; waits for the stream and
// checks the flags.
static Status shard_finish_stats(dmcg_plan* p);
Status shard_phase(dmcg_plan* p, int phase, const void* const x[3]) {
  ShardState& sh = *p->shard;
  cudaStream_t s = p->ctx->stream;
  const int F = (int)p->F, k = (int)p->k, n_own = (int)sh.n_own;
  const bool f32 = p->dtype == DMCG_F32;
  const long FF = (long)F * F;
  const long krows = 3L * k + 3;
  const int q = sh.rank;
  const int na = (int)(sh.a0[q + 1] - sh.a0[q]);
  switch (phase) {
    case 0: {
      DMCG_TRY(cudaMemsetAsync(p->d_flags, 0, 8 * sizeof(int), s));
      DMCG_TRY(record_event(p->ev[0], s));
      if (variant_uses_delta(p->variant))
        DMCG_TRY(launch_delta(s, n_own, F, sh.d_loc_rp, sh.d_loc_ci, x, f32, p->d_delta,
                              p->d_flags));
      else
        DMCG_TRY(launch_check_finite(s, n_own, F, x, f32, p->d_flags));
      DMCG_TRY(record_event(p->ev[1], s));
      if (implicit_oi(p)) return Status::ok();
      Status st = f32 ? gram<float>(p, x, n_own) : gram<double>(p, x, n_own);
      if (!st.good()) return st;
      return Status::ok();
    }
    case 1: {
      DMCG_TRY(record_event(p->ev[2], s));
      p->forked = false;
      if (implicit_oi(p) && !sh.comm && sh.nranks > 1)
        return Status{DMCG_E_CONFIG,
                      "ConfigError: the implicit OI allreduces every round: shard it with a "
                      "communicator (dmcg_shard_encode_device)"};
      Status st = basis(p, x, n_own, sh.comm);
      if (!st.good()) return st;
      DMCG_TRY(record_event(p->ev[3], s));
      DMCG_TRY(launch_init_keys(s, krows, sh.d_keys));
      if (k > 0) {
        LoadDense<double, true> lU{p->d_U, FF, 1L, (long)F};
        StoreCoeffMinMax ep{p->d_C, sh.d_keys};
        if (variant_uses_delta(p->variant)) {
          LoadDense<double, true> lD{p->d_delta, (long)n_own * F, 1L, (long)F};
          DMCG_TRY(launch_gemm(s, 3, k, n_own, F, 1, lU, lD, ep));
        } else if (f32) {  // v2v: the owned rows of the trajectories
          LoadDense3<float, true> lX{(const float*)x[0], (const float*)x[1], (const float*)x[2],
                                     1L, (long)F};
          DMCG_TRY(launch_gemm(s, 3, k, n_own, F, 1, lU, lX, ep));
        } else {
          LoadDense3<double, true> lX{(const double*)x[0], (const double*)x[1],
                                      (const double*)x[2], 1L, (long)F};
          DMCG_TRY(launch_gemm(s, 3, k, n_own, F, 1, lU, lX, ep));
        }
      }
      DMCG_TRY(launch_anchor_keys(s, na, F, sh.d_loc_anchor, x, f32, sh.d_keys + 6L * k));
      DMCG_TRY(launch_flip_min_keys(s, krows, sh.d_keys));
      return Status::ok();
    }
    case 2: {
      DMCG_TRY(launch_flip_min_keys(s, krows, sh.d_keys));
      uint16_t* stage = sh.d_gather + sh.stage_off[q];
      if (k > 0)
        DMCG_TRY(launch_quant_rows(s, k, n_own, sh.d_keys, p->d_row_bits + 3 * k, p->d_C,
                                   p->d_row_min, p->d_row_max, p->d_row_bits, stage));
      DMCG_TRY(launch_anchor_quant(s, na, F, sh.d_loc_anchor, x, f32, p->anchor_bits,
                                   sh.d_keys + 6L * k, p->d_anchor_rng,
                                   stage + 3L * k * n_own));
      DMCG_TRY(record_event(p->ev[4], s));
      if (p->forked) DMCG_TRY(cudaStreamWaitEvent(s, p->ev_join, 0));
      DMCG_TRY(launch_quant_dict(s, 3 * FF, p->dict_bits, p->d_U, p->d_dict_q));
      return Status::ok();
    }
    case 3: {
      const size_t n = p->n, n_c = p->n_c;
      for (int r = 0; r < sh.nranks; ++r) {
        const size_t own = sh.r0[r + 1] - sh.r0[r], nar = sh.a0[r + 1] - sh.a0[r];
        const uint16_t* src = sh.d_gather + sh.stage_off[r];
        if (k > 0 && own)
          DMCG_TRY(cudaMemcpy2DAsync(p->d_coeff_q + sh.r0[r], n * 2, src, own * 2, own * 2,
                                     3 * (size_t)k, cudaMemcpyDeviceToDevice, s));
        if (nar)
          DMCG_TRY(cudaMemcpy2DAsync(p->d_anchor_q + (size_t)sh.a0[r] * F, n_c * F * 2,
                                     src + 3 * (size_t)k * own, nar * F * 2, nar * F * 2, 3,
                                     cudaMemcpyDeviceToDevice, s));
      }
      DMCG_TRY(record_event(p->ev[5], s));
      return shard_finish_stats(p);
    }
  }
  return Status{DMCG_E_CONFIG, "ConfigError: bad shard phase"};
}

static Status shard_finish_stats(dmcg_plan* p) {
  cudaStream_t s = p->ctx->stream;
  int flags[8];
  DMCG_TRY(cudaMemcpyAsync(flags, p->d_flags, sizeof(flags), cudaMemcpyDeviceToHost, s));
  DMCG_TRY(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&p->stats.ms_encode, p->ev[0], p->ev[5]);
  cudaEventElapsedTime(&p->stats.ms_delta, p->ev[0], p->ev[1]);
  cudaEventElapsedTime(&p->stats.ms_gram, p->ev[1], p->ev[2]);    // incl. the allreduce
  cudaEventElapsedTime(&p->stats.ms_basis, p->ev[2], p->ev[3]);
  cudaEventElapsedTime(&p->stats.ms_project, p->ev[3], p->ev[4]); // incl. the key allreduce
  const bool oi = p->rounds > 0 && p->k < p->F && p->k > 0;
  p->stats.ms_oi = 0.0f;
  p->stats.flops_oi = 0.0;
  if (oi) {
    cudaEventElapsedTime(&p->stats.ms_oi, p->ev[6], p->ev[7]);
    const double F = p->F, k = p->k, r = p->rounds;
    const double qr = 2.0 * (2.0 * F * k * k - 2.0 * k * k * k / 3.0);
    p->stats.flops_oi = oi_flops(p, F, k, r, qr);
  }
  p->stats.kernel_launches_encode = 1 + 2 + (oi ? 10 : 3) + 1 + (p->k > 0 ? 2 : 0) + 1 + 2 + 1 + 1;
  if (flags[0])
    return Status{DMCG_E_INDEX, "ValidationError: non-finite coordinate in the local rows"};
  if (flags[3])
    return Status{DMCG_E_NUMERICAL,
                  "ConvergenceFailure: symmetric eigendecomposition did not converge"};
  return Status::ok();
}

Status shard_encode(dmcg_plan* p, const void* const x[3]) {
  ShardState& sh = *p->shard;
  cudaStream_t s = p->ctx->stream;
  const size_t FF = (size_t)p->F * p->F;
  Status st = shard_phase(p, 0, x);
  if (st.good() && !implicit_oi(p)) st = comm_allreduce_sum_f64(sh.comm, p->d_R, 3 * FF, s);
  if (st.good()) st = shard_phase(p, 1, x);
  if (st.good()) st = comm_allreduce_max_u64(sh.comm, sh.d_keys, (3ull * p->k + 3) * 2, s);
  if (st.good()) st = shard_phase(p, 2, x);
  if (st.good()) st = comm_allgatherv_u16(sh.comm, sh.d_gather, sh.stage_off.data(), s);
  if (st.good()) st = shard_phase(p, 3, x);
  return st;
}

// Direct decode: K6 into the row-major n x 3F layout, rhs, supernodal
// Cholesky factor + solve + refinement (solver.cpp:43-58, 82-90).
// Frames [f0, f0 + Fw) only (the solve is column-separable: each frame
// column's result does not depend on the others, so a window decodes to the
// same bits as the full decode).
static Status enqueue_decode_direct(dmcg_plan* p, int refine, bool factor, bool pre,
                                    void* const out[3], int f0, int Fw) {
  cudaStream_t s = p->ctx->stream;
  const int n = (int)p->n, F = Fw, F_all = (int)p->F, k = (int)p->k, W = 3 * Fw;
  CholDev cdev = p->cdev;
  cdev.W = (uint32_t)W;
  const bool f32 = p->dtype == DMCG_F32;
  DMCG_TRY(cudaMemsetAsync(p->d_flags, 0, 8 * sizeof(int), s));
  DMCG_TRY(record_event(p->ev[0], s));
  const size_t nW = (size_t)n * W;
  // The right-hand sides (dequantise + reconstruct + L^T delta~ + S^T a) do
  // not depend on the factor of M: they run on the side stream while the
  // main stream factors, and join before the solves.
  cudaStream_t s1 = s;
  s = p->ctx->aux;
  DMCG_TRY(cudaEventRecord(p->ev_fork, s1));
  DMCG_TRY(cudaStreamWaitEvent(s, p->ev_fork, 0));
  if (k > 0 && p->nb > 1) {
    // blocks: decode_dictionaries (closed-loop sums), dequantize_rows of
    // every block, then delta~(:, block b) = (U~_b c~_b)^T as one batched
    // GEMM over the 3 n_b blocks (codec.cpp:527-533)
    const int nb = (int)p->nb, kf = (int)p->kf, kl = (int)p->k_l;
    const long kk = (long)kf * kf;
    DMCG_TRY(launch_row_params(s, 3 * k, p->d_row_min, p->d_row_max, p->d_row_bits, p->d_rowp));
    DMCG_TRY(launch_dequant_rows(s, 3 * k, n, p->d_coeff_q, p->d_rowp, p->d_row_bits,
                                 p->d_flags + 1, p->d_C));
    DMCG_TRY(launch_dict_decode_blocks(s, nb, kf, p->dict_bits, p->diff_bits, p->d_dict_q,
                                       p->d_diff_rng, p->d_flags + 1, p->d_bUd));
    LoadDense<double, false> la{p->d_C, (long)kl * n, (long)n, 1L};  // A(r, i) = c~_b(r, i)
    LoadDense<double, false> lb{p->d_bUd, kk, (long)kf, 1L};         // B(r, f) = U~_b(f, r)
    DMCG_TRY(launch_gemm(s, 3 * nb, n, kf, kl, 1, la, lb,
                         StoreStrided{p->d_rm_delta, (long)kf, (long)W, 1L}));
  } else if (k > 0) {
    DMCG_TRY(launch_row_params(s, 3 * k, p->d_row_min, p->d_row_max, p->d_row_bits, p->d_rowp));
    // dequantised coefficients (3 k x n, into the encode's coefficient
    // buffer) and U~[:, :k] over the window, then a plain f64 GEMM
    double* Cd = p->d_C;
    double* Ud = p->d_Ud;
    // a later frame window of the same upload (the drop-in decode's second
    // window): the dequantised coefficients and their slices are in place
    const bool a_ready = p->rec_a_valid && p->oz_rec_slices && !p->use_graphs;
    const bool per_axis = p->coeff_events && p->oz_rec_slices && !a_ready && !p->use_graphs;
    if (p->coeff_events && !per_axis) {  // the symbols arrive on the copy stream
      for (int a = 0; a < 3; ++a) DMCG_TRY(cudaStreamWaitEvent(s, p->ctx->ev_in[a], 0));
      p->coeff_events = false;
    }
    if (!a_ready && !per_axis)
      DMCG_TRY(launch_dequant_rows(s, 3 * k, n, p->d_coeff_q, p->d_rowp, p->d_row_bits,
                                   p->d_flags + 1, Cd));
    DMCG_TRY(launch_dequant_dict(s, F_all, k, f0, F, p->d_dict_q, p->dict_bits, p->d_flags + 1, Ud));
    if (per_axis) {
      // dequantise, slice and multiply axis a as soon as its symbols are in
      // (same slices and tiles as the batched oz_matmul below: same bits)
      const int sr = p->oz_rec_slices;
      const long kn = (long)k * n, kF = (long)k * F;
      OzSlices sa, sb;
      sa.rows = n;
      sa.rows_pad = oz_rows_pad(n);
      sa.K = k;
      sa.K_pad = oz_k_pad(k);
      sa.s = sr;
      sa.batch = 1;
      sb = sa;
      sb.rows = F;
      sb.rows_pad = oz_rows_pad(F);
      int8_t* qa = p->d_oz_q;
      int8_t* qb = qa + oz_slice_bytes(n, k, sr, 3);
      unsigned long long* ma = p->d_oz_max;
      unsigned long long* mb = ma + 3L * oz_rows_pad(n);
      for (int a = 0; a < 3; ++a) {
        DMCG_TRY(cudaStreamWaitEvent(s, p->ctx->ev_in[a], 0));
        DMCG_TRY(launch_dequant_rows(s, k, n, p->d_coeff_q + a * kn, p->d_rowp + 2L * a * k,
                                     p->d_row_bits + a * k, p->d_flags + 1, Cd + a * kn));
        OzOperand A{{Cd + a * kn, nullptr, nullptr}, false, 1L, (long)n, n, k, 1};
        OzOperand B{{Ud + a * kF, nullptr, nullptr}, false, 1L, (long)F, F, k, 1};
        sa.q = qa + (size_t)a * sr * sa.rows_pad * sa.K_pad;
        sa.maxbits = ma + (size_t)a * sa.rows_pad;
        sb.q = qb + (size_t)a * sr * sb.rows_pad * sb.K_pad;
        sb.maxbits = mb + (size_t)a * sb.rows_pad;
        DMCG_TRY(oz_slice(s, A, sa));
        DMCG_TRY(oz_slice(s, B, sb));
        OzStore outa{p->d_rm_delta + (long)a * F, 0L, 0L, (long)W, 1L};
        int used = 0;
        DMCG_TRY(oz_gemm(s, sa, sb, outa, 1, &used));
        if (used != 1) return Status{DMCG_E_CUDA, "CudaError: reconstruction split"};
      }
      p->rec_a_valid = true;
      p->coeff_events = false;
    } else if (p->oz_rec_slices) {
      // INT8 tensor cores (Ozaki slices): delta~(i, b F + f) = sum_r c~(b, r, i) U~(f, r)
      const int sr = p->oz_rec_slices;
      const long kn = (long)k * n, kF = (long)k * F;
      OzOperand A{{Cd, Cd + kn, Cd + 2 * kn}, false, 1L, (long)n, n, k, 3};
      OzOperand B{{Ud, Ud + kF, Ud + 2 * kF}, false, 1L, (long)F, F, k, 3};
      int8_t* qa = p->d_oz_q;
      int8_t* qb = qa + oz_slice_bytes(n, k, sr, 3);
      unsigned long long* ma = p->d_oz_max;
      unsigned long long* mb = ma + 3L * oz_rows_pad(n);
      OzStore out{p->d_rm_delta, (long)F, 0L, (long)W, 1L};
      DMCG_TRY(oz_matmul(s, A, B, sr, qa, ma, qb, mb, out, a_ready));
      p->rec_a_valid = !p->use_graphs;
    } else {
      LoadDense<double, false> la{Cd, (long)k * n, (long)n, 1L};   // A(r, i) = c~(r, i)
      LoadDense<double, false> lb{Ud, (long)k * F, (long)F, 1L};   // B(r, f) = U~(f0 + f, r)
      // delta~ (i, a*F + f): batch b = axis, rows = vertices, cols = frames
      DMCG_TRY(launch_gemm(s, 3, n, F, k, 1, la, lb,
                           StoreStrided{p->d_rm_delta, (long)F, (long)W, 1L}));
    }
  } else {
    DMCG_TRY(cudaMemsetAsync(p->d_rm_delta, 0, nW * sizeof(double), s));
  }
  if (p->variant == DMCG_V2V) {  // axes = U~ c~ (codec.cpp:520-524): no solve
    DMCG_TRY(record_event(p->ev[1], s));
    DMCG_TRY(cudaEventRecord(p->ev_join, s));
    s = s1;
    DMCG_TRY(cudaStreamWaitEvent(s, p->ev_join, 0));
    for (int e : {2, 5, 3}) DMCG_TRY(record_event(p->ev[e], s));
    DMCG_TRY(launch_output_rm(s, n, F, F_all, f0, p->d_rm_delta, out, f32));
    DMCG_TRY(record_event(p->ev[4], s));
    return Status::ok();
  }
  // rhs = L^T delta~ (+ S^T a): every row of L delta~ (anchor slots -1 on the
  // anchor-free variants, whose reduced system uses rows 1.. only).
  DMCG_TRY(launch_rhs_rm(s, n, F, F_all, f0, p->d_lap_rp, p->d_lap_ci, p->d_anchor_pos, (int)p->n_c,
                         p->d_anchor_q, p->d_anchor_rng, p->anchor_bits, p->d_rm_delta, p->d_rm_b,
                         p->d_flags + 1));
  DMCG_TRY(record_event(p->ev[1], s));
  DMCG_TRY(cudaEventRecord(p->ev_join, s));
  s = s1;
  if (factor) DMCG_TRY(chol_factor_device(s, cdev, p->levels));
  DMCG_TRY(record_event(p->ev[2], s));
  DMCG_TRY(cudaStreamWaitEvent(s, p->ev_join, 0));
  DMCG_TRY(record_event(p->ev[5], s));
  // solve_anchored (solver.cpp:62-90) on all n rows, or solve_mean_constrained
  // (solver.cpp:105-133): vertex 0 pinned, unknowns = rows 1.. (offset W).
  if (pre && !factor) {  // the overlapped factor: joined here if launched outside a graph
    if (p->pf_unjoined) DMCG_TRY(cudaStreamWaitEvent(s, p->ev_pf_join, 0));
    DMCG_TRY(cudaMemcpyAsync(p->d_flags + 4, p->d_pf_flag, sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  const bool mc = variant_uses_means(p->variant);
  const int nm = (int)cdev.n;
  const size_t o = mc ? (size_t)W : 0;
  const size_t evl = 4 * (size_t)p->levels.nlevels;
  if (p->kernel_timing && p->solve_ev.size() < (size_t)(1 + refine) * evl) {
    const size_t have = p->solve_ev.size();
    p->solve_ev.resize((size_t)(1 + refine) * evl);
    for (size_t e = have; e < p->solve_ev.size(); ++e) cudaEventCreate(&p->solve_ev[e]);
  }
  auto tev = [&](int pass) {
    SolveEvents t;
    if (p->kernel_timing) t.ev = p->solve_ev.data() + (size_t)pass * evl;
    return t;
  };
  const SolveEvents tev0 = tev(0);
  DMCG_TRY(chol_solve_device(s, cdev, p->levels, p->d_rm_b + o, p->d_rm_y, p->d_rm_xp,
                             p->d_rm_x + o, false, &tev0));
  for (int r = 0; r < refine; ++r) {
    DMCG_TRY(normal_residual(s, nm, W, p->d_m_rp, p->d_m_ci, p->d_m_val, p->d_rm_b + o,
                             p->d_rm_x + o, p->d_rm_r));
    const SolveEvents tevr = tev(1 + r);
    DMCG_TRY(chol_solve_device(s, cdev, p->levels, p->d_rm_r, p->d_rm_y, p->d_rm_xp,
                               p->d_rm_x + o, true, &tevr));
  }
  DMCG_TRY(record_event(p->ev[3], s));
  const double* shift = nullptr;
  if (mc) {  // x = [0; z], each column moved to its stored mean
    DMCG_TRY(cudaMemsetAsync(p->d_rm_x, 0, (size_t)W * sizeof(double), s));
    double* sh = p->d_colsum + 64 * (size_t)W;  // after the (<= 64) row-chunk partials
    DMCG_TRY(launch_mean_shift(s, n, F, F_all, f0, p->d_rm_x, p->d_means, p->d_colsum, sh));
    shift = sh;
  }
  if (p->nb > 1)  // strip the padding (codec.cpp:549)
    DMCG_TRY(launch_output_rm(s, n, F, (int)p->F_in, 0, p->d_rm_x, out, f32, nullptr,
                              (int)p->F_in));
  else
    DMCG_TRY(launch_output_rm(s, n, F, F_all, f0, p->d_rm_x, out, f32, shift));
  DMCG_TRY(record_event(p->ev[4], s));
  return Status::ok();
}

static Status plan_decode_direct(dmcg_plan* p, const dmcg_decode_options* opt,
                                 void* const out[3]) {
  cudaStream_t s = p->ctx->stream;
  const int k = (int)p->k;
  const int refine = opt ? opt->refine : 1;
  // the factor of M left by the last encode (overlapped with it), else the
  // caller's reuse_factor, else factor now
  const bool pre = p->factor_pending;
  const bool factor = !(pre || (opt && opt->reuse_factor && p->factor_valid));
  uint32_t f0 = opt ? opt->frame_begin : 0, Fw = opt ? opt->frame_count : 0;
  if (p->nb > 1) {  // blocks: one stacked solve over all padded frames
    if (f0 != 0 || (Fw != 0 && Fw != p->F_in))
      return Status{DMCG_E_UNSUPPORTED, "Unsupported: frame windows of a blocks stream"};
    Fw = 0;
  }
  if (Fw == 0) {
    f0 = 0;
    Fw = p->F;
  }
  if (f0 >= p->F || Fw > p->F - f0)
    return Status{DMCG_E_CONFIG, "DimensionMismatch: frame window outside the sequence"};
  const int W = 3 * (int)Fw;
  const void* key[4] = {out[0], out[1], out[2], nullptr};
  {
    const long long okey = ((long long)f0 << 40) | ((long long)Fw << 16) | (refine * 8) |
                           (p->kernel_timing ? 4 : 0) | (pre ? 2 : 0) | (factor ? 1 : 0);
    Status st = run_graph(p, p->g_decode, key, okey, [&] {
      return enqueue_decode_direct(p, refine, factor, pre, out, (int)f0, (int)Fw);
    });
    if (!st.good()) return st;
  }
  int flags[8];
  DMCG_TRY(cudaMemcpyAsync(flags, p->d_flags, sizeof(flags), cudaMemcpyDeviceToHost, s));
  DMCG_TRY(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&p->stats.ms_decode, p->ev[0], p->ev[4]);
  // reconstruct (side stream) and factor (main stream) both start at ev0
  cudaEventElapsedTime(&p->stats.ms_reconstruct, p->ev[0], p->ev[1]);
  cudaEventElapsedTime(&p->stats.ms_factor, p->ev[0], p->ev[2]);
  cudaEventElapsedTime(&p->stats.ms_solve, p->ev[5], p->ev[3]);
  p->stats.ms_cg = 0.0f;
  p->stats.solver = 0;
  p->stats.cg_iterations_max = 0;
  p->stats.cg_rel_residual_max = 0.0;
  const CholLevels& lv = p->levels;
  int nl = 0;  // factor: assemble, panels + trailing, inverse (2), P (2) per level
  for (uint32_t l = 0; l < lv.nlevels; ++l) nl += 5 + (int)((lv.maxw[l] + 31) / 32) * 2;
  // gather, forward, backward per level (the leaf level has no gather pass)
  const int per_solve = (int)lv.nlevels * 3 - (lv.nlevels ? 1 : 0);
  p->stats.kernel_launches_decode = (k > 0 ? 2 : 0) + 1 + (factor ? nl : 0) +
                                    (1 + refine) * per_solve + refine + 1;
  p->stats.flops_solve = (1 + refine) * p->chol.flops_solve_per_rhs * W;
  p->stats.ms_solve_fwd = p->stats.ms_solve_bwd = 0.0f;
  p->stats.flops_solve_fwd = p->stats.flops_solve_bwd = 0.0;
  if (p->kernel_timing) {  // the events completed with the stream sync above
    const size_t evl = 4 * (size_t)lv.nlevels;
    for (int pass = 0; pass <= refine; ++pass)
      for (uint32_t l = 0; l < lv.nlevels; ++l) {
        const cudaEvent_t* e = p->solve_ev.data() + pass * evl + 4 * l;
        float a = 0.0f, b = 0.0f;
        cudaEventElapsedTime(&a, e[0], e[1]);
        cudaEventElapsedTime(&b, e[2], e[3]);
        p->stats.ms_solve_fwd += a;
        p->stats.ms_solve_bwd += b;
      }
    p->stats.flops_solve_fwd = p->stats.flops_solve_bwd = 0.5 * p->stats.flops_solve;
  }
  if (flags[1]) return Status{DMCG_E_CORRUPT, "CorruptPayload: packed value out of range"};
  if (flags[4]) {
    p->factor_valid = false;
    return Status{DMCG_E_NUMERICAL,
                  "SingularSystem: anchored normal equations are not positive definite"};
  }
  if (pre && p->pf_unjoined) cudaEventElapsedTime(&p->ms_prefactor, p->ev_pf0, p->ev_pf1);
  p->factor_pending = false;
  p->pf_unjoined = false;
  p->factor_valid = true;
  // overlapped factor: its own time on aux2 during the encode
  if (!factor) p->stats.ms_factor = pre ? p->ms_prefactor : 0.0f;
  return Status::ok();
}

Status plan_decode(dmcg_plan* p, const dmcg_decode_options* opt, void* const out[3]) {
  if (opt && opt->solver != 0 && p->nb > 1)
    return Status{DMCG_E_UNSUPPORTED,
                  "Unsupported: the CG solver serves the n_b = 1 anchored variants only"};
  if (opt && opt->solver != 0 && !variant_uses_anchors(p->variant))
    return Status{DMCG_E_UNSUPPORTED,
                  "Unsupported: the CG solver serves the anchored variants only (pca_qp, pca_qs)"};
  if (!opt || opt->solver == 0) {
    Status st = plan_prepare_decode(p);
    if (!st.good()) return st;
    return plan_decode_direct(p, opt, out);
  }
  cudaStream_t s = p->ctx->stream;
  const int n = (int)p->n, F = (int)p->F, k = (int)p->k;
  const bool f32 = p->dtype == DMCG_F32;
  if (!p->d_cg_x) {  // CG vectors are allocated on first use
    const size_t vec = (size_t)p->nblk * n * kCB * 8;
    p->d_cg_x = (double*)plan_alloc(p, vec);
    p->d_cg_r = (double*)plan_alloc(p, vec);
    p->d_cg_p = (double*)plan_alloc(p, vec);
    p->d_cg_q = (double*)plan_alloc(p, vec);
    if (!p->d_cg_x || !p->d_cg_r || !p->d_cg_p || !p->d_cg_q)
      return Status{DMCG_E_CUDA, "CudaError: device allocation failed"};
  }
  p->stats.solver = 1;
  {
    Status sn = plan_prepare_normal(p);
    if (!sn.good()) return sn;
  }
  DMCG_TRY(cudaMemsetAsync(p->d_flags, 0, 8 * sizeof(int), s));
  DMCG_TRY(record_event(p->ev[0], s));
  // K6: dequantise + reconstruct delta~ = (U~ c~)^T (codec.cpp:528-533)
  // straight into the CG layout; rows >= k_l are exactly zero in the
  // reference, so the contraction runs over r < k_l only.
  const size_t vec = (size_t)p->nblk * n * kCB;
  DMCG_TRY(cudaMemsetAsync(p->d_cg_q, 0, vec * sizeof(double), s));
  if (k > 0) {
    DMCG_TRY(launch_row_params(s, 3 * k, p->d_row_min, p->d_row_max, p->d_row_bits, p->d_rowp));
    LoadCoeffDeq la{p->d_coeff_q, p->d_rowp, p->d_row_bits, p->d_flags + 1, n, k};
    const uint32_t levels = 1u << p->dict_bits;
    LoadDictDeq lb{p->d_dict_q, 2.0 / (double)levels, levels, F, p->d_flags + 1};
    DMCG_TRY(launch_gemm(s, 3, n, F, k, 1, la, lb, StoreCG{p->d_cg_q, n, F}));
  }
  // rhs = L^T delta~ + S^T a (solver.cpp:77-80) -> r
  DMCG_TRY(launch_rhs(s, n, F, (int)p->W, (int)p->nblk, p->d_lap_rp, p->d_lap_ci, p->d_anchor_pos,
                      (int)p->n_c, p->d_anchor_q, p->d_anchor_rng, p->anchor_bits, p->d_cg_q,
                      p->d_cg_r, p->d_flags + 1));
  DMCG_TRY(record_event(p->ev[1], s));
  // K7 CG.
  const double rtol = opt ? opt->cg_rtol : 1e-10;
  const int maxit = opt ? opt->cg_max_iter : 20000;
  DMCG_TRY(launch_cg(s, n, (int)p->W, (int)p->nblk, p->d_m_rp, p->d_m_ci, p->d_m_val, p->d_cg_x,
                     p->d_cg_r, p->d_cg_p, p->d_cg_q, rtol, maxit, p->d_cg_iters, p->d_cg_res));
  DMCG_TRY(record_event(p->ev[2], s));
  DMCG_TRY(launch_output(s, n, F, p->d_cg_x, out, f32));
  DMCG_TRY(record_event(p->ev[3], s));
  int flags[8];
  DMCG_TRY(cudaMemcpyAsync(flags, p->d_flags, sizeof(flags), cudaMemcpyDeviceToHost, s));
  std::vector<int> iters(p->W);
  std::vector<double> res(p->W);
  DMCG_TRY(cudaMemcpyAsync(iters.data(), p->d_cg_iters, p->W * sizeof(int), cudaMemcpyDeviceToHost, s));
  DMCG_TRY(cudaMemcpyAsync(res.data(), p->d_cg_res, p->W * sizeof(double), cudaMemcpyDeviceToHost, s));
  DMCG_TRY(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&p->stats.ms_decode, p->ev[0], p->ev[3]);
  cudaEventElapsedTime(&p->stats.ms_reconstruct, p->ev[0], p->ev[1]);
  cudaEventElapsedTime(&p->stats.ms_cg, p->ev[1], p->ev[2]);
  p->stats.kernel_launches_decode = (k > 0 ? 2 : 0) + 3;
  int itmax = 0;
  double resmax = 0.0;
  for (uint32_t c = 0; c < p->W; ++c) {
    itmax = iters[c] > itmax ? iters[c] : itmax;
    resmax = res[c] > resmax ? res[c] : resmax;
  }
  p->stats.cg_iterations_max = itmax;
  p->stats.cg_rel_residual_max = resmax;
  if (flags[1]) return Status{DMCG_E_CORRUPT, "CorruptPayload: packed value out of range"};
  if (!(resmax <= rtol))
    return Status{DMCG_E_NUMERICAL, "SingularSystem: anchored solve did not converge (residual " +
                                        std::to_string(resmax) + ")"};
  return Status::ok();
}

}  // namespace dmcg
