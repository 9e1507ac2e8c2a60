// Device view of a CholPlan (chol.h) and the launchers of chol.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace dmcg {

struct CholDev {
  uint32_t n = 0, nsup = 0, W = 0;
  const uint32_t* first = nullptr;
  const unsigned long long* str_ptr = nullptr;
  const uint32_t* str_idx = nullptr;
  const uint32_t* child_ptr = nullptr;
  const uint32_t* child_idx = nullptr;
  const unsigned long long* rel_ptr = nullptr;
  const uint32_t* rel_idx = nullptr;
  const unsigned long long* a_ptr = nullptr;
  const uint32_t* a_pos = nullptr;
  const float* a_val = nullptr;
  const unsigned long long* front_off = nullptr;
  const unsigned long long* inv_off = nullptr;
  const unsigned long long* rhs_off = nullptr;
  const unsigned long long* op_off = nullptr;
  const uint32_t* perm = nullptr;
  const uint32_t* level_sup = nullptr;
  const uint32_t* level_ptr = nullptr;  // nlevels + 1 offsets into level_sup
  const uint32_t* pull_ptr = nullptr;   // extend-add pull lists (chol.h)
  const uint32_t* pull_src = nullptr;
  uint32_t nlevels = 0;
  double* F = nullptr;     // fronts (factor in place)
  double* Linv = nullptr;  // L11^{-1}, row-major per front
  double* P = nullptr;     // solve operators [L11^{-1}; -L21 L11^{-1}], m_s x w_s column-major
  double* R = nullptr;     // per-front update rows (rows w_s .. m_s of an m_s x W panel)
  double* scratch = nullptr;  // blocked-inverse tiles (chol_scratch_doubles)
  unsigned long long linv_doubles = 0;
  int* flags = nullptr;    // [0] non-positive pivot
};

// Host-side per-level launch geometry.
struct CholLevels {
  uint32_t nlevels = 0;
  std::vector<uint32_t> offset, count, maxw, maxm, maxu;
};

cudaError_t chol_factor_device(cudaStream_t s, const CholDev& d, const CholLevels& lv);
// Doubles of scratch the blocked L11 inverse needs (CholDev::scratch).
size_t chol_scratch_doubles(const CholLevels& lv);
// b: n x W row-major in the original order; y, x: n x W in the permuted order.
// Optional per-launch timing: ev[4 l + 0 / 1] around level l's forward
// GEMM, ev[4 l + 2 / 3] around its backward GEMM (4 nlevels events).
struct SolveEvents {
  cudaEvent_t* ev = nullptr;
};
// out (original order, n x W) = x unpermuted (accumulate: out += x), written
// by the backward pass itself.
cudaError_t chol_solve_device(cudaStream_t s, const CholDev& d, const CholLevels& lv,
                              const double* b, double* y, double* x, double* out, bool accumulate,
                              const SolveEvents* tev = nullptr);
// r = b - M x for n x W row-major blocks (original order).
cudaError_t normal_residual(cudaStream_t s, int n, int W, const uint32_t* rp, const uint32_t* ci,
                            const float* val, const double* b, const double* x, double* r);

}  // namespace dmcg
