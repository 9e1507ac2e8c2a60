// Supernodal multifrontal Cholesky of the anchored normal matrix
// M = L^T L + S^T S (reference: SimplicialLDLT in src/solver.cpp:62-90,
// factored once and back-substituted for every frame column).
//
// Host analysis (chol_symbolic.cpp): nested-dissection ordering, elimination
// tree, postorder, column counts, fundamental + relaxed supernodes, front
// row structures, level schedule, extend-add index maps and the scatter list
// of M into the fronts.  Device numerics (chol.cu): per level, assemble the
// fronts, partial dense Cholesky (DMMA trailing updates), invert L11; the
// multi-RHS solves are then pure batched GEMMs per level.
#pragma once
#include <cstdint>
#include <map>
#include <utility>
#include <vector>

namespace dmcg {

struct CholPlan {
  uint32_t n = 0;
  std::vector<uint32_t> perm, iperm;      // perm[new] = old
  uint32_t nsup = 0;
  std::vector<uint32_t> first;            // nsup + 1: supernode s owns new columns [first[s], first[s+1])
  std::vector<uint64_t> str_ptr;          // nsup + 1
  std::vector<uint32_t> str_idx;          // rows (new numbering), own columns first
  std::vector<int32_t> parent;            // supernode parent, -1 at roots
  std::vector<uint32_t> child_ptr, child_idx;
  std::vector<uint32_t> level_ptr, level_sup;  // supernodes grouped by level (leaves first)
  std::vector<uint64_t> front_off;        // nsup + 1, m_s^2 doubles each
  std::vector<uint64_t> inv_off;          // nsup + 1, w_s^2 doubles each
  std::vector<uint64_t> rhs_off;          // nsup + 1, m_s rows each (times W columns)
  std::vector<uint64_t> op_off;           // nsup + 1, m_s x w_s doubles each (solve operator P_s)
  std::vector<uint64_t> rel_ptr;          // nsup + 1 (indexed by child)
  std::vector<uint32_t> rel_idx;          // child update row -> local row in the parent
  // "pull" form of the extend-add for the solves: front row g (global
  // numbering rhs_off[s] + r) sums the child update rows pull_src[pull_ptr[g]
  // .. pull_ptr[g+1]) (global rows), children in order: every row can be
  // formed independently and deterministically.
  std::vector<uint32_t> pull_ptr, pull_src;
  std::vector<uint64_t> a_ptr;            // nsup + 1
  std::vector<uint32_t> a_pos;            // local index (col * m + row) in the front
  std::vector<float> a_val;               // value of M
  // statistics
  uint64_t nnz_l = 0;                     // stored entries of L (dense fronts, lower)
  double flops_factor = 0.0, flops_solve_per_rhs = 0.0;
  uint32_t max_front = 0, max_width = 0, nlevels = 0;

  uint32_t w(uint32_t s) const { return first[s + 1] - first[s]; }
  uint32_t m(uint32_t s) const { return (uint32_t)(str_ptr[s + 1] - str_ptr[s]); }
};

// M given as a symmetric CSR (rows sorted, diagonal present).
// g_rp / g_ci (optional): the 1-ring graph whose square is M's pattern (the
// mesh Laplacian's structure), used for a cheaper nested-dissection ordering.
// pre (optional): the ordering of chol_order_graph on the same 1-ring graph,
// computed ahead (it does not need M, so a caller can run it beside the
// normal-matrix build).
struct CholOrdering {
  std::vector<uint32_t> perm0;  // elimination order before the postorder
  std::map<uint64_t, std::pair<uint32_t, uint32_t>> splits;  // dissection ranges (see .cpp)
};
void chol_order_graph(uint32_t n, const std::vector<uint32_t>& g_rp,
                      const std::vector<uint32_t>& g_ci, CholOrdering* out);
void chol_analyze(uint32_t n, const std::vector<uint32_t>& rp, const std::vector<uint32_t>& ci,
                  const std::vector<float>& val, CholPlan* plan,
                  const std::vector<uint32_t>* g_rp = nullptr,
                  const std::vector<uint32_t>* g_ci = nullptr, CholOrdering* pre = nullptr);

// CPU reference numerics over the same structures (tests / debugging).
// F: front_off[nsup] doubles, Linv: inv_off[nsup] doubles.  Returns false if
// a pivot is not positive.
bool chol_factor_cpu(const CholPlan& p, std::vector<double>* F, std::vector<double>* Linv);
// x = M^{-1} b for W columns; b, x are n x W row-major in the ORIGINAL order.
void chol_solve_cpu(const CholPlan& p, const std::vector<double>& F,
                    const std::vector<double>& Linv, uint32_t W, const double* b, double* x);

}  // namespace dmcg
