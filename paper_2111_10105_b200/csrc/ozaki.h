// FP64-accurate GEMMs on the sm_100a INT8 tensor cores (tcgen05.mma
// kind::i8, TMEM accumulators, TMA-fed shared-memory tiles): the Ozaki
// splitting scheme.
//
// sm_100a has no tcgen05 kind::f64; its FP64 tensor
// path is legacy DMMA at ~37 TFLOP/s.  The int8 tensor cores run at
// ~4.5 POPS dense and their int32 accumulation is EXACT, so a matrix product
// whose operands are cut into s signed 7-bit slices,
//
//   x = 2^e(row) * sum_{p=1..s} a_p 2^(-7p),    a_1 in [-127, 127],
//   a_p in [-64, 64] for p > 1 (balanced, round-to-nearest digits),
//
// is recovered as  C = 2^(eA + eB) sum_{d=2}^{s+1} 2^(-7d) D_d,
//   D_d = sum_{p+q=d} A_p B_q^T   (exact int32 GEMMs, one TMEM accumulator
// per diagonal d, combined in fp64 in the epilogue).  The dropped terms
// (p + q > s + 1, both digits balanced) and the rounded slice tails bound the
// error by about 2^(-7s) |x|_max |y|_max per product term, zero-mean, so
// the error of a K-term sum grows like sqrt(K) — s = 5 (35 bits) covers fp32
// inputs with headroom, s = 7 (49 bits) approaches fp64.
//
// Operands are "rows x K" views of fp32 / fp64 matrices with arbitrary
// strides; oz_slice() writes the int8 slices K-major ([batch][s][rows][K],
// zero padded) plus one exponent per row, oz_gemm() multiplies two sliced
// operands.  Reference contractions this serves: the Gram A A^T
// (src/spectral.cpp:35-39), the projection U^T delta^T (src/codec.cpp:420)
// and the implicit OI products X Q, X^T P.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dmcg {

constexpr int kOzBM = 128;   // UMMA M (TMEM lanes)
constexpr int kOzBN = 64;    // UMMA N per diagonal accumulator
constexpr int kOzBK = 32;    // one kind::i8 MMA consumes K = 32 bytes
constexpr int kOzMaxS = 7;
constexpr int kOzKChunk = 16384;  // K per split: |D_d| <= S * 127 * 64 * K < 2^31

// A batch (<= 3) of "rows x K" matrices: element (r, k) of batch b at
// base[b][r * row_stride + k * k_stride], fp32 or fp64.
struct OzOperand {
  const void* base[3];
  bool f32;
  long row_stride, k_stride;
  int rows, K, batch;
};

// Sliced operand in device memory.
struct OzSlices {
  int8_t* q = nullptr;          // [batch][s][rows_pad][K_pad]
  unsigned long long* maxbits = nullptr;  // [batch][rows_pad] bits of max |x| (double; exponents derive from it)
  int rows = 0, rows_pad = 0, K = 0, K_pad = 0, s = 0, batch = 0;
  size_t bytes() const { return (size_t)batch * s * rows_pad * K_pad; }
};

// rows_pad / K_pad of an operand (rows to a multiple of 128, K of 32).
inline int oz_rows_pad(int rows) { return (rows + kOzBM - 1) / kOzBM * kOzBM; }
inline int oz_k_pad(int K) { return (K + kOzBK - 1) / kOzBK * kOzBK; }

// Row maxima, then the s slices (zero padded).  sl.q / sl.maxbits must be
// allocated for (batch, s, rows_pad, K_pad).
cudaError_t oz_slice(cudaStream_t st, const OzOperand& op, OzSlices& sl);

// Epilogue: C(b, split, m, n) at C + b*sb + split*ssplit + m*sm + n*sn (fp64).
// keys (optional, one split only): per-row running (min, max) as ordered
// keys at keys[2 (b M + m)], [.. + 1] (the projection's row ranges).
struct OzStore {
  double* C;
  long sb, ssplit, sm, sn;
  unsigned long long* keys = nullptr;
};

// C[b](m, n) = sum_k A[b](m, k) B[b](n, k) over M = A.rows, N = B.rows,
// K = A.K (= B.K), split over ceil(K_pad / kOzKChunk) K ranges (or `splits`
// if larger) written to separate partial slots.  Returns the split count via
// *splits_out.  A and B may be the same OzSlices (the Gram).
// syrk (A and B the same slices): tiles entirely above the diagonal are
// skipped; the caller reads the lower triangle only.
cudaError_t oz_gemm(cudaStream_t st, const OzSlices& A, const OzSlices& B, const OzStore& out,
                    int min_splits, int* splits_out, bool syrk = false);

// C[b] = A[b] B[b]^T for two operand views (one K split: K_pad <= kOzKChunk),
// slicing both into qa / qb (oz_slice_bytes each) and maxa / maxb
// (batch x oz_rows_pad(rows) each): the projection U_k^T delta^T
// (codec.cpp:420, with out.keys = the row ranges) and the reconstruction
// U~ c~ (codec.cpp:531-532) of fp32-storage plans.
inline size_t oz_slice_bytes(int rows, int K, int s, int batch) {
  return (size_t)batch * s * oz_rows_pad(rows) * oz_k_pad(K);
}
// a_sliced: qa / maxa already hold A's slices (an earlier call on the same A).
cudaError_t oz_matmul(cudaStream_t st, const OzOperand& A, const OzOperand& B, int s, int8_t* qa,
                      unsigned long long* maxa, int8_t* qb, unsigned long long* maxb,
                      const OzStore& out, bool a_sliced = false);

// Splits oz_gemm will use for (A, B, min_splits).
int oz_splits(const OzSlices& A, int min_splits);

// The Gram R = X^T X of a batch of 3 n x F fp32 / fp64 axis matrices
// (x[i*F + f]; rows = frames, K = vertex rows): slices X into q / maxbits
// (3 x s x oz_rows_pad(F) x oz_k_pad(n) bytes, 3 x oz_rows_pad(F)) and writes
// the split-K partials part[(split * 3 + b) F^2 + f F + g]; returns the
// split count in *splits.  oz_gram_splits() = that count (for sizing part).
int oz_gram_splits(int F, int n, int s);
cudaError_t oz_gram(cudaStream_t st, const void* const x[3], bool f32, int n, int F, int s,
                    int8_t* q, unsigned long long* maxbits, double* part, int* splits);
// Axis a alone, into the same buffers and partial slots (bit-identical R).
cudaError_t oz_gram_axis(cudaStream_t st, int a, const void* xa, bool f32, int n, int F, int s,
                         int8_t* q, unsigned long long* maxbits, double* part, int* splits);

}  // namespace dmcg
