// Ozaki-scheme FP64-accurate GEMM on the sm_100a INT8 tensor cores
// (ozaki.h).  Three kernels:
//
//   k_oz_rowmax_*  max |x| per operand row (the slice exponent),
//   k_oz_slice     the s signed 7-bit slices, K-major int8, zero padded,
//   k_oz_gemm      warp-specialised tcgen05 GEMM: warp 0 issues the TMA loads
//                  of one 32-byte K step of every slice of A (128 rows) and B
//                  (64 rows) per pipeline stage (SWIZZLE_32B tiles, mbarrier
//                  complete_tx), warp 1 allocates TMEM and issues
//                  tcgen05.mma.cta_group::1.kind::i8 for every slice pair
//                  p + q <= s + 1 into the int32 accumulator of its diagonal
//                  (s accumulators of 128 x 64 in TMEM), tcgen05.commit frees
//                  the stage; warps 2-5 drain TMEM (tcgen05.ld 32x32b) and
//                  combine the diagonals in fp64.
#include "ozaki.h"

#include "common.cuh"

#include <cudaTypedefs.h>

#include <cmath>
#include <type_traits>
#include <mutex>
#include <vector>

namespace dmcg {
namespace {

// ---- slicing ------------------------------------------------------------------

// Slice exponent of a row with max |x| = mx: the smallest e with
// mx 2^-e < 127.5 / 128, so the first balanced digit rint(128 x 2^-e) stays
// within [-127, 127] and every later digit (a remainder in [-1/2, 1/2]
// scaled by 128) within [-64, 64].  Rounded (balanced) digits make the
// truncation and the dropped diagonals (p, q >= 2 only) zero-mean, so their
// errors cancel like fp64 rounding instead of accumulating with n.
__device__ __forceinline__ int oz_exp(double mx) {
  if (!(mx > 0.0)) return 0;
  int e;
  const double f = frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  return f >= 127.5 / 128.0 ? e + 1 : e;
}

template <typename T>
__device__ __forceinline__ double oz_ld(const OzOperand& op, int b, long r, long k) {
  const T* base = (const T*)op.base[b];
  return (double)base[r * op.row_stride + k * op.k_stride];
}

// One warp per row, K contiguous (k_stride == 1).
template <typename T>
__global__ void k_oz_rowmax_kcontig(OzOperand op, unsigned long long* maxbits, int rows_pad) {
  const int row = (int)((blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  if (row >= rows_pad) return;
  double m = 0.0;
  if (row < op.rows) {
    const T* p = (const T*)op.base[b] + (long)row * op.row_stride;
    for (int k = lane; k < op.K; k += 32) m = fmax(m, fabs((double)p[k]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) maxbits[(long)b * rows_pad + row] = (unsigned long long)__double_as_longlong(m);
}

// One thread per row over a K chunk (any strides; coalesced when row_stride
// == 1), atomicMax of the non-negative double bits.
template <typename T>
__global__ void k_oz_rowmax_rows(OzOperand op, unsigned long long* maxbits, int rows_pad, int kchunk) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.z;
  if (row >= op.rows) return;
  const long k0 = (long)blockIdx.y * kchunk;
  const long k1 = k0 + kchunk < op.K ? k0 + kchunk : op.K;
  // eight independent loads in flight per thread (the dependent one-load loop
  // ran at 29 % of HBM)
  double m8[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) m8[u] = 0.0;
  long k = k0;
  for (; k + 8 <= k1; k += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = oz_ld<T>(op, b, row, k + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) m8[u] = fmax(m8[u], fabs(v[u]));
  }
  for (; k < k1; ++k) m8[0] = fmax(m8[0], fabs(oz_ld<T>(op, b, row, k)));
  double m = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) m = fmax(m, m8[u]);
  atomicMax(maxbits + (long)b * rows_pad + row, (unsigned long long)__double_as_longlong(m));
}

// 64 rows x 64 K tile per 256-thread CTA: load (coalesced along the
// contiguous dimension) into shared memory, then each thread slices 16
// consecutive K of one row into s 16-byte stores.
template <typename T, bool KCONTIG>
__global__ void __launch_bounds__(256) k_oz_slice(OzOperand op, OzSlices sl) {
  __shared__ double tile[64][65];
  const int b = blockIdx.z, r0 = blockIdx.y * 64;
  const long k0 = (long)blockIdx.x * 64;
  const int t = threadIdx.x;
  {  // all sixteen loads of the thread in flight, then the stores
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = t + 256 * j;
      const int r = KCONTIG ? i / 64 : i % 64, k = KCONTIG ? i % 64 : i / 64;
      const long gr = r0 + r, gk = k0 + k;
      v[j] = (gr < op.rows && gk < op.K) ? oz_ld<T>(op, b, gr, gk) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = t + 256 * j;
      const int r = KCONTIG ? i / 64 : i % 64, k = KCONTIG ? i % 64 : i / 64;
      tile[r][k] = v[j];
    }
  }
  __syncthreads();
  const int r = t >> 2, kq = (t & 3) * 16;
  const long gk = k0 + kq;
  if (gk >= sl.K_pad) return;
  const int e = oz_exp(__longlong_as_double((long long)sl.maxbits[(long)b * sl.rows_pad + r0 + r]));
  uint32_t w[kOzMaxS][4];
#pragma unroll
  for (int p = 0; p < kOzMaxS; ++p) w[p][0] = w[p][1] = w[p][2] = w[p][3] = 0u;
  if constexpr (std::is_same<T, float>::value) {
    // fp32 storage: the same digits in fp32 arithmetic.  x 2^-e, the products
    // by 128 and the remainders are exact in fp32 (a 24-bit value loses 7 bits
    // per digit), rint is the round-to-nearest-even of adding 1.5 * 2^23, and
    // the digit's two's complement sits in the sum's low mantissa byte: no
    // fp64 pipe and no XU conversions (which bound the fp64 loop below).
    // Values that would be fp32 denormals after scaling are below every digit.
    const float scale = (e > -127 && e < 127) ? __int_as_float((127 - e) << 23) : 0.0f;
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = (float)tile[r][kq + j];
      float y = scale != 0.0f ? __fmul_rn(x, scale) : ldexpf(x, -e);
#pragma unroll
      for (int p = 0; p < kOzMaxS; ++p) {
        if (p < sl.s) {
          y = __fmul_rn(y, 128.0f);
          const float m = __fadd_rn(y, kMagic);
          const float a = __fsub_rn(m, kMagic);
          y = __fsub_rn(y, a);
          w[p][j >> 2] |= ((uint32_t)__float_as_int(m) & 0xffu) << (8 * (j & 3));
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      double y = ldexp(tile[r][kq + j], -e);  // |y| < 127.5 / 128, exact
#pragma unroll
      for (int p = 0; p < kOzMaxS; ++p) {
        if (p < sl.s) {
          y *= 128.0;
          const double a = rint(y);  // balanced digits: |a_1| <= 127, |a_p| <= 64 (p > 1)
          y -= a;                    // exact, |y| <= 1/2
          w[p][j >> 2] |= (uint32_t)(uint8_t)(int8_t)(int)a << (8 * (j & 3));
        }
      }
    }
  }
  const long row = r0 + r;
#pragma unroll
  for (int p = 0; p < kOzMaxS; ++p)
    if (p < sl.s) {
      int8_t* dst = sl.q + (((long)b * sl.s + p) * sl.rows_pad + row) * sl.K_pad + gk;
      *reinterpret_cast<uint4*>(dst) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
    }
}

// ---- tcgen05 / TMA / mbarrier primitives ----------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// K-major SWIZZLE_32B shared-memory matrix descriptor (sm100 version 1):
// rows of 32 bytes, 8-row core groups 256 B apart (SBO); LBO unused.
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;   // SBO = 256 B
  d |= (uint64_t)1 << 46;            // descriptor version (Blackwell)
  d |= (uint64_t)6 << 61;            // SWIZZLE_32B
  return d;
}
// Instruction descriptor: s32 accumulate, signed int8 A and B, K-major both.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// ---- the GEMM ---------------------------------------------------------------------

struct OzGemmArgs {
  int M, N, tiles_m, tiles_n, splits, kb_total, kb_per_split;
  int a_rows_pad, b_rows_pad;
  int syrk;  // A == B (Gram): only the tiles that reach the lower triangle are computed
  const unsigned long long* a_max;
  const unsigned long long* b_max;
  OzStore out;
};

template <int S>
struct OzCfg {
  static constexpr int kA = kOzBM * kOzBK;                 // bytes of one A slice tile
  static constexpr int kB = kOzBN * kOzBK;                 // bytes of one B slice tile
  static constexpr int kStage = S * (kA + kB);
  // S <= 4: the accumulators fit 256 TMEM columns, so two CTAs share an SM
  // (one's epilogue under the other's MMAs) with four stages each
  static constexpr int kCtasPerSm = S <= 4 ? 2 : 1;
  static constexpr int kStages = S <= 4 ? 4 : ((196608 / kStage) < 8 ? (196608 / kStage) : 8);
  static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/ + 4 * kOzBN;
  static constexpr int kCols = S * kOzBN <= 256 ? 256 : 512;  // TMEM allocation (power of 2)
};

template <int S>
__global__ void __launch_bounds__(192, OzCfg<S>::kCtasPerSm)
    k_oz_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
              OzGemmArgs g) {
  using C = OzCfg<S>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + C::kStages * C::kStage);
  // bars[0 .. kStages): full, [kStages .. 2 kStages): empty, [2 kStages]: tmem_full
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * C::kStages + 1);
  int* col_exp = (int*)(tmem_slot + 4);  // kOzBN column exponents of this tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work unit: batch, tile_m, tile_n, split
  int u = blockIdx.x;
  const int sp = u % g.splits;
  u /= g.splits;
  const int tn = u % g.tiles_n;
  u /= g.tiles_n;
  const int tm = u % g.tiles_m;
  const int b = u / g.tiles_m;
  const int kb0 = sp * g.kb_per_split;
  const int kb1 = min(g.kb_total, kb0 + g.kb_per_split);
  const int nkb = kb1 - kb0;
  // Gram: the slice products are exact integers and the fp64 combination is
  // the same expression for (f, g) and (g, f), so the partial is bitwise
  // symmetric; a tile entirely above the diagonal is never read
  // (k_reduce_sym, lower_only) and exits before any setup
  if (g.syrk && tn * kOzBN > tm * kOzBM + (kOzBM - 1)) return;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(smem_u32(&bars[i]), 1);
      mbar_init(smem_u32(&bars[C::kStages + i]), 1);
    }
    mbar_init(smem_u32(&bars[2 * C::kStages]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0 && nkb > 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&ta) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tb) : "memory");
      for (int it = 0; it < nkb; ++it) {
        const int st = it % C::kStages;
        const uint32_t ph = (uint32_t)(it / C::kStages) & 1u;
        mbar_wait(smem_u32(&bars[C::kStages + st]), ph ^ 1u);
        const uint32_t full = smem_u32(&bars[st]);
        mbar_expect_tx(full, (uint32_t)C::kStage);
        const uint32_t sa = smem_u32(smem + st * C::kStage);
        const uint32_t sb = sa + S * C::kA;
        const int kc = (kb0 + it) * kOzBK;
#pragma unroll
        for (int p = 0; p < S; ++p) {
          tma_load_3d(sa + p * C::kA, &ta, full, kc, tm * kOzBM, b * S + p);
          tma_load_3d(sb + p * C::kB, &tb, full, kc, tn * kOzBN, b * S + p);
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    constexpr uint32_t idesc = idesc_i8(kOzBM, kOzBN);
    for (int it = 0; it < nkb; ++it) {
      const int st = it % C::kStages;
      const uint32_t ph = (uint32_t)(it / C::kStages) & 1u;
      mbar_wait(smem_u32(&bars[st]), ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t sa = smem_u32(smem + st * C::kStage);
        const uint32_t sb = sa + S * C::kA;
#pragma unroll
        for (int d = 2; d <= S + 1; ++d) {
          const int p0 = d - S > 1 ? d - S : 1, p1 = d - 1 < S ? d - 1 : S;
#pragma unroll
          for (int p = p0; p <= p1; ++p) {
            // the first product of diagonal d in the first K step overwrites
            const uint32_t acc = (it > 0 || p != p0) ? 1u : 0u;
            mma_i8(tbase + (uint32_t)((d - 2) * kOzBN), sw32_desc(sa + (p - 1) * C::kA),
                   sw32_desc(sb + (d - p - 1) * C::kB), idesc, acc);
          }
        }
        mma_commit(smem_u32(&bars[C::kStages + st]));  // frees the stage when these MMAs finish
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(smem_u32(&bars[2 * C::kStages]));
    __syncwarp();
  } else {
    // ===== epilogue: warps 2..5 own TMEM lanes 32 (warp % 4) .. +31 =====
    const int quarter = warp & 3;
    const int mrow = tm * kOzBM + quarter * 32 + lane;
    const int ea = oz_exp(__longlong_as_double(
        (long long)g.a_max[(long)b * g.a_rows_pad + min(mrow, g.a_rows_pad - 1)]));
    {  // the tile's column exponents, once (epilogue warps 2..5 = threads 64..191)
      const int t = threadIdx.x - 64;
      if (t < kOzBN) {
        const int ncol = min(tn * kOzBN + t, g.b_rows_pad - 1);
        col_exp[t] = oz_exp(__longlong_as_double((long long)g.b_max[(long)b * g.b_rows_pad + ncol]));
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the four epilogue warps only
    }
    const uint32_t lane_addr = tbase + ((uint32_t)(quarter * 32) << 16);
    if (nkb > 0) {
      mbar_wait(smem_u32(&bars[2 * C::kStages]), 0u);
      tc_fence_after();
    }
    double lo = INFINITY, hi = -INFINITY;
    // Unit-stride outputs go through shared memory (the operand stages are
    // free once tmem_full has fired): a lane holds one ROW of the tile, so
    // direct stores are 32 scattered 8-byte pieces per instruction; staged,
    // the warp writes each row's 64 doubles as two contiguous 256-byte stores.
    constexpr int kStgLd = kOzBN + 1;
    static_assert(4 * 32 * kStgLd * 8 <= C::kStages * C::kStage, "staging fits the operand stages");
    const bool staged = g.out.sn == 1;
    double* stg = reinterpret_cast<double*>(smem) + quarter * (32 * kStgLd);
#pragma unroll 1
    for (int c = 0; c < kOzBN / 16; ++c) {
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.0;
      if (nkb > 0) {
#pragma unroll
        for (int d = S + 1; d >= 2; --d) {  // smallest weight first
          int32_t raw[16];
          tmem_ld16(lane_addr + (uint32_t)((d - 2) * kOzBN + c * 16), raw);
          tmem_wait_ld();
          const double wd = ldexp(1.0, -7 * d);  // exact: (double) raw * wd is exact
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = fma((double)raw[j], wd, v[j]);
        }
      }
      if (mrow < g.M) {
        double* dst = g.out.C + b * g.out.sb + sp * g.out.ssplit + (long)mrow * g.out.sm;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int ncol = tn * kOzBN + c * 16 + j;
          if (ncol < g.N) {
            const double r = ldexp(v[j], ea + col_exp[c * 16 + j]);
            if (staged)
              stg[lane * kStgLd + c * 16 + j] = r;
            else
              dst[(long)ncol * g.out.sn] = r;
            lo = fmin(lo, r);
            hi = fmax(hi, r);
          }
        }
      }
    }
    if (staged) {
      __syncwarp();
      const int m0 = tm * kOzBM + quarter * 32;
#pragma unroll 4
      for (int rr = 0; rr < 32; ++rr) {
        if (m0 + rr >= g.M) break;
        double* dst = g.out.C + b * g.out.sb + sp * g.out.ssplit + (long)(m0 + rr) * g.out.sm +
                      tn * kOzBN;
#pragma unroll
        for (int h = 0; h < kOzBN / 32; ++h) {
          const int col = lane + 32 * h;
          if (tn * kOzBN + col < g.N) dst[col] = stg[rr * kStgLd + col];
        }
      }
    }
    if (g.out.keys && mrow < g.M && lo <= hi) {
      unsigned long long* kp = g.out.keys + 2 * ((long)b * g.M + mrow);
      atomicMin(kp, ordered_key(lo));
      atomicMax(kp + 1, ordered_key(hi));
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(C::kCols));
  }
}

// ---- host ----------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)f;
  }();
  return fn;
}

// 3-D map over the slices: (K_pad bytes, rows_pad, batch * s), box (32, box_rows, 1), SWIZZLE_32B.
bool make_map(CUtensorMap* map, const OzSlices& sl, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)sl.K_pad, (cuuint64_t)sl.rows_pad, (cuuint64_t)sl.batch * sl.s};
  const cuuint64_t strides[2] = {(cuuint64_t)sl.K_pad, (cuuint64_t)sl.K_pad * sl.rows_pad};
  const cuuint32_t box[3] = {(cuuint32_t)kOzBK, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)sl.q, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int S>
cudaError_t launch_gemm_s(cudaStream_t st, const CUtensorMap& ma, const CUtensorMap& mb,
                          const OzGemmArgs& g, int units) {
  using C = OzCfg<S>;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(k_oz_gemm<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  if (attr != cudaSuccess) return attr;
  k_oz_gemm<S><<<units, 192, C::kSmem, st>>>(ma, mb, g);
  return cudaGetLastError();
}

}  // namespace

cudaError_t oz_slice(cudaStream_t st, const OzOperand& op, OzSlices& sl) {
  if (sl.s < 1 || sl.s > kOzMaxS || op.batch != sl.batch) return cudaErrorInvalidValue;
  const long maxn = (long)sl.batch * sl.rows_pad;
  cudaError_t e = cudaMemsetAsync(sl.maxbits, 0, maxn * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (op.k_stride == 1) {
    dim3 grid((unsigned)((sl.rows_pad * 32L + 255) / 256), sl.batch);
    if (op.f32) k_oz_rowmax_kcontig<float><<<grid, 256, 0, st>>>(op, sl.maxbits, sl.rows_pad);
    else k_oz_rowmax_kcontig<double><<<grid, 256, 0, st>>>(op, sl.maxbits, sl.rows_pad);
  } else {
    const int kchunk = 1024;
    dim3 grid((op.rows + 255) / 256, (op.K + kchunk - 1) / kchunk, sl.batch);
    if (op.f32) k_oz_rowmax_rows<float><<<grid, 256, 0, st>>>(op, sl.maxbits, sl.rows_pad, kchunk);
    else k_oz_rowmax_rows<double><<<grid, 256, 0, st>>>(op, sl.maxbits, sl.rows_pad, kchunk);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid((sl.K_pad + 63) / 64, sl.rows_pad / 64, sl.batch);
  const bool kc = op.k_stride == 1;
  if (op.f32) {
    if (kc) k_oz_slice<float, true><<<grid, 256, 0, st>>>(op, sl);
    else k_oz_slice<float, false><<<grid, 256, 0, st>>>(op, sl);
  } else {
    if (kc) k_oz_slice<double, true><<<grid, 256, 0, st>>>(op, sl);
    else k_oz_slice<double, false><<<grid, 256, 0, st>>>(op, sl);
  }
  return cudaGetLastError();
}

int oz_splits(const OzSlices& A, int min_splits) {
  const int kb_total = A.K_pad / kOzBK;
  const int kb_chunk = kOzKChunk / kOzBK;
  int splits = (kb_total + kb_chunk - 1) / kb_chunk;
  if (min_splits > splits) splits = min_splits < kb_total ? min_splits : kb_total;
  return splits < 1 ? 1 : splits;
}

static int gram_min_splits(int F) {
  const int tiles = ((F + kOzBM - 1) / kOzBM) * ((F + kOzBN - 1) / kOzBN);
  return (2 * 148 + 3 * tiles - 1) / (3 * tiles);
}

int oz_gram_splits(int F, int n, int s) {
  OzSlices sl;
  sl.K = n;
  sl.K_pad = oz_k_pad(n);
  sl.s = s;
  return oz_splits(sl, gram_min_splits(F));
}

cudaError_t oz_gram(cudaStream_t st, const void* const x[3], bool f32, int n, int F, int s,
                    int8_t* q, unsigned long long* maxbits, double* part, int* splits) {
  OzOperand op{{x[0], x[1], x[2]}, f32, 1L, (long)F, F, n, 3};
  OzSlices sl;
  sl.q = q;
  sl.maxbits = maxbits;
  sl.rows = F;
  sl.rows_pad = oz_rows_pad(F);
  sl.K = n;
  sl.K_pad = oz_k_pad(n);
  sl.s = s;
  sl.batch = 3;
  cudaError_t e = oz_slice(st, op, sl);
  if (e != cudaSuccess) return e;
  const long FF = (long)F * F;
  OzStore out{part, FF, 3 * FF, (long)F, 1L};
  return oz_gemm(st, sl, sl, out, gram_min_splits(F), splits, true);
}

// One axis of oz_gram (the drop-in encode runs an axis as soon as its input has
// arrived): same slices, same K splits and the same partial slots as the
// batched call, so the reduced R is bit-identical.
cudaError_t oz_gram_axis(cudaStream_t st, int a, const void* xa, bool f32, int n, int F, int s,
                         int8_t* q, unsigned long long* maxbits, double* part, int* splits) {
  OzOperand op{{xa, nullptr, nullptr}, f32, 1L, (long)F, F, n, 1};
  OzSlices sl;
  sl.rows = F;
  sl.rows_pad = oz_rows_pad(F);
  sl.K = n;
  sl.K_pad = oz_k_pad(n);
  sl.s = s;
  sl.batch = 1;
  sl.q = q + (size_t)a * s * sl.rows_pad * sl.K_pad;
  sl.maxbits = maxbits + (size_t)a * sl.rows_pad;
  cudaError_t e = oz_slice(st, op, sl);
  if (e != cudaSuccess) return e;
  const long FF = (long)F * F;
  OzStore out{part + a * FF, FF, 3 * FF, (long)F, 1L};
  return oz_gemm(st, sl, sl, out, oz_gram_splits(F, n, s), splits, true);
}

cudaError_t oz_matmul(cudaStream_t st, const OzOperand& A, const OzOperand& B, int s, int8_t* qa,
                      unsigned long long* maxa, int8_t* qb, unsigned long long* maxb,
                      const OzStore& out, bool a_sliced) {
  if (A.K != B.K || A.batch != B.batch || oz_k_pad(A.K) > kOzKChunk) return cudaErrorInvalidValue;
  OzSlices sa, sb;
  sa.q = qa;
  sa.maxbits = maxa;
  sa.rows = A.rows;
  sa.rows_pad = oz_rows_pad(A.rows);
  sa.K = A.K;
  sa.K_pad = oz_k_pad(A.K);
  sa.s = s;
  sa.batch = A.batch;
  sb = sa;
  sb.q = qb;
  sb.maxbits = maxb;
  sb.rows = B.rows;
  sb.rows_pad = oz_rows_pad(B.rows);
  cudaError_t e = a_sliced ? cudaSuccess : oz_slice(st, A, sa);
  if (e == cudaSuccess) e = oz_slice(st, B, sb);
  if (e != cudaSuccess) return e;
  int used = 0;
  e = oz_gemm(st, sa, sb, out, 1, &used);
  return (e == cudaSuccess && used != 1) ? cudaErrorInvalidValue : e;
}

cudaError_t oz_gemm(cudaStream_t st, const OzSlices& A, const OzSlices& B, const OzStore& out,
                    int min_splits, int* splits_out, bool syrk) {
  if (A.s != B.s || A.K_pad != B.K_pad || A.batch != B.batch) return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, kOzBM) || !make_map(&mb, B, kOzBN)) return cudaErrorInvalidValue;
  OzGemmArgs g;
  g.M = A.rows;
  g.N = B.rows;
  g.tiles_m = (A.rows + kOzBM - 1) / kOzBM;
  g.tiles_n = (B.rows + kOzBN - 1) / kOzBN;
  g.kb_total = A.K_pad / kOzBK;
  g.splits = oz_splits(A, min_splits);
  g.kb_per_split = (g.kb_total + g.splits - 1) / g.splits;
  g.syrk = (syrk && A.q == B.q) ? 1 : 0;
  g.a_rows_pad = A.rows_pad;
  g.b_rows_pad = B.rows_pad;
  g.a_max = A.maxbits;
  g.b_max = B.maxbits;
  g.out = out;
  if (splits_out) *splits_out = g.splits;
  const int units = A.batch * g.tiles_m * g.tiles_n * g.splits;
  switch (A.s) {
    case 3: return launch_gemm_s<3>(st, ma, mb, g, units);
    case 4: return launch_gemm_s<4>(st, ma, mb, g, units);
    case 5: return launch_gemm_s<5>(st, ma, mb, g, units);
    case 6: return launch_gemm_s<6>(st, ma, mb, g, units);
    case 7: return launch_gemm_s<7>(st, ma, mb, g, units);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dmcg

extern "C" int dmcg_ozaki_gemm(const void* dA, int a_f32, long a_rs, long a_ks, int M, const void* dB,
                               int b_f32, long b_rs, long b_ks, int N, int K, int s, double* dC) {
  using namespace dmcg;
  if (M <= 0 || N <= 0 || K <= 0 || s < 3 || s > kOzMaxS) return 5;
  OzOperand a{{dA, nullptr, nullptr}, a_f32 != 0, a_rs, a_ks, M, K, 1};
  OzOperand b{{dB, nullptr, nullptr}, b_f32 != 0, b_rs, b_ks, N, K, 1};
  OzSlices sa, sb;
  sa.rows = M; sa.rows_pad = oz_rows_pad(M); sa.K = K; sa.K_pad = oz_k_pad(K); sa.s = s; sa.batch = 1;
  sb.rows = N; sb.rows_pad = oz_rows_pad(N); sb.K = K; sb.K_pad = sa.K_pad; sb.s = s; sb.batch = 1;
  cudaError_t e = cudaSuccess;
  void* mem = nullptr;
  const size_t qa = sa.bytes(), qb = sb.bytes();
  const int splits = oz_splits(sa, 1);
  const size_t part = (size_t)splits * M * N;
  e = cudaMalloc(&mem, qa + qb + 8 * (size_t)(sa.rows_pad + sb.rows_pad) + 8 * part);
  if (e != cudaSuccess) return 10;
  uint8_t* m8 = (uint8_t*)mem;
  sa.q = (int8_t*)m8;
  sb.q = (int8_t*)(m8 + qa);
  sa.maxbits = (unsigned long long*)(m8 + qa + qb);
  sb.maxbits = sa.maxbits + sa.rows_pad;
  double* P = (double*)(sb.maxbits + sb.rows_pad);
  if ((e = oz_slice(0, a, sa)) == cudaSuccess && (e = oz_slice(0, b, sb)) == cudaSuccess) {
    OzStore st{splits > 1 ? P : dC, 0, (long)M * N, (long)N, 1};
    int used = 0;
    e = oz_gemm(0, sa, sb, st, 1, &used);
    if (e == cudaSuccess && used > 1) {
      std::vector<double> h((size_t)used * M * N), c((size_t)M * N, 0.0);
      e = cudaMemcpy(h.data(), P, h.size() * 8, cudaMemcpyDeviceToHost);
      for (int q = 0; q < used; ++q)
        for (size_t i = 0; i < c.size(); ++i) c[i] += h[(size_t)q * M * N + i];
      if (e == cudaSuccess) e = cudaMemcpy(dC, c.data(), c.size() * 8, cudaMemcpyHostToDevice);
    }
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(mem);
  return e == cudaSuccess ? 0 : 10;
}
