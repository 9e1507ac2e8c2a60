// dmc/codec.hpp — Eigen-free C++ drop-in for the reference encoder/decoder
// API (reference include/dmc/codec.hpp:28-91, include/dmc/stream.hpp:130-155,
// include/dmc/mesh.hpp:36-57, include/dmc/errors.hpp:24-61), header-only over
// the libdmcg C ABI (include/dmcg.h).  Link with -ldmcg.
//
// Differences from the reference, all forced by the environment / scope:
//   * dmc::Matrix replaces Eigen::MatrixXd (column-major, rows()/cols()/
//     data()/operator()) because Eigen3 is unavailable (reference
//     CMakeLists.txt:11); the memory layout is identical, so a reference
//     caller can pass Eigen::MatrixXd::data() buffers straight through.
//   * CompressedAnimation holds the quantised-payload fields of the variants
//     pca, pca_q, v2v, pca_qs, pca_qp and blocks; the coefficient blocks of
//     an axis are one flat row list (block b at rows [b k_l, (b+1) k_l)).
//   * EncoderConfig::oi_tolerance is a double (< 0 = unset) instead of
//     std::optional<double>.
//   * EncoderConfig gains oi_rounds / oi_seed (B200 rank-k basis) and
//     decode() takes optional CG controls.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../dmcg.h"

namespace dmc {

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what)
      : std::runtime_error(what), code_(code), kind_(what.substr(0, what.find(':'))) {}
  int code() const { return code_; }
  const std::string& kind() const { return kind_; }

 private:
  int code_;
  std::string kind_;
};

// Column-major dense matrix (the Eigen::MatrixXd layout).
class Matrix {
 public:
  Matrix() = default;
  Matrix(int64_t r, int64_t c) : r_(r), c_(c), d_((size_t)(r * c), 0.0) {}
  int64_t rows() const { return r_; }
  int64_t cols() const { return c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(int64_t i, int64_t j) { return d_[(size_t)(j * r_ + i)]; }
  double operator()(int64_t i, int64_t j) const { return d_[(size_t)(j * r_ + i)]; }

 private:
  int64_t r_ = 0, c_ = 0;
  std::vector<double> d_;
};

using Face = std::array<uint32_t, 3>;

// Reference MeshSequence (mesh.hpp:36-57): three k x n axis matrices.
class MeshSequence {
 public:
  MeshSequence() = default;
  MeshSequence(std::vector<Face> faces, std::array<Matrix, 3> axes)
      : faces_(std::move(faces)), axes_(std::move(axes)) {
    for (int a = 1; a < 3; ++a)
      if (axes_[a].rows() != axes_[0].rows() || axes_[a].cols() != axes_[0].cols())
        throw Error(5, "DimensionMismatch: axis matrices must share one k x n shape");
  }
  int n() const { return (int)axes_[0].cols(); }
  int k() const { return (int)axes_[0].rows(); }
  const std::vector<Face>& faces() const { return faces_; }
  const Matrix& axis(int a) const { return axes_[a]; }

 private:
  std::vector<Face> faces_;
  std::array<Matrix, 3> axes_;
};

enum class Variant : uint8_t { Pca = 0, PcaQ = 1, V2v = 2, PcaQs = 3, PcaQp = 4, Blocks = 5,
                               PerMeshGft = 6 };
enum class AnchorStrategy : uint8_t { Stride = 0, SeededRandom = 1 };

struct EncoderConfig {  // reference codec.hpp:30-49 (+ B200 basis controls)
  Variant variant = Variant::PcaQp;
  uint32_t k_l = 20;
  std::vector<int> row_bits;
  uint16_t n_b = 1;
  int t_max = 4;
  double anchor_fraction = 0.01;
  int anchor_bits = 16;
  int dict_bits = 16;
  int diff_bits = 8;
  AnchorStrategy anchor_strategy = AnchorStrategy::Stride;
  uint64_t seed = 0;
  bool raw_payload = false;
  int oi_rounds = 0;       // 0 = full eigenbasis (reference n_b = 1 path)
  uint64_t oi_seed = 0;
  int oi_implicit = 0;
  double oi_tolerance = -1.0;  // blocks: principal-angle stop (< 0 = unset)
};

struct QuantRow {  // stream.hpp:86-93
  float min = 0.0f, max = 0.0f;
  uint8_t bits = 0;
  std::vector<uint32_t> q;  // empty when min == max
};

struct DictDiff {  // stream.hpp:95-101
  float min = 0.0f, max = 0.0f;
  std::vector<uint32_t> q;  // k_f * k_f levels at diff_bits, column-major
};

struct CompressedAnimation {  // stream.hpp:130-155, quantised payloads of variants 0-5
  Variant variant = Variant::PcaQp;
  uint32_t n = 0, k = 0, k_l = 0, n_c = 0;
  uint16_t n_b = 1, pad = 0;
  uint8_t anchor_bits = 16, dict_bits = 16, diff_bits = 8;
  std::vector<Face> faces;
  std::array<std::vector<uint32_t>, 3> dict_first;   // k_f*k_f levels, column-major
  std::array<std::vector<DictDiff>, 3> dict_diffs;   // blocks 2..n_b
  std::array<std::vector<QuantRow>, 3> coeffs;       // n_b * k_l rows per axis
  uint32_t k_f() const { return (k + pad) / n_b; }
  std::vector<uint32_t> anchor_indices;
  std::array<float, 3> anchor_min{}, anchor_max{};
  std::array<std::vector<uint32_t>, 3> anchor_q;     // n_c*k, anchor-major
  std::array<std::vector<float>, 3> means;           // k per-frame means (pca / pca_q)
};

namespace detail {
struct Ctx {
  dmcg_ctx* c = nullptr;
  Ctx() {
    int rc = dmcg_create(&c, 0);
    if (rc) throw Error(rc, "CudaError: dmcg_create failed");
  }
  ~Ctx() { dmcg_destroy(c); }
  static Ctx& get() {
    thread_local Ctx ctx;  // one context (stream + pool) per calling thread
    return ctx;
  }
};
inline void check(int rc) {
  if (rc) throw Error(rc, dmcg_last_error(Ctx::get().c));
}
}  // namespace detail

inline uint32_t anchor_count(uint32_t n, double fraction) { return dmcg_anchor_count(n, fraction); }

inline std::vector<uint32_t> select_anchors(uint32_t n, uint32_t n_c, AnchorStrategy s,
                                            uint64_t seed) {
  std::vector<uint32_t> out(n_c);
  int rc = dmcg_select_anchors(n, n_c, (int)s, seed, out.data());
  if (rc) throw Error(rc, "InvalidCount: anchor count outside 1..n");
  return out;
}

// dmc::encode (reference codec.hpp:90).
inline CompressedAnimation encode(const MeshSequence& s, const EncoderConfig& cfg) {
  dmcg_config c;
  dmcg_config_default(&c);
  c.variant = (int)cfg.variant;
  c.k_l = cfg.k_l;
  c.row_bits = cfg.row_bits.empty() ? nullptr : cfg.row_bits.data();
  c.n_row_bits = (uint32_t)cfg.row_bits.size();
  c.n_b = cfg.n_b;
  c.t_max = cfg.t_max;
  c.anchor_fraction = cfg.anchor_fraction;
  c.anchor_bits = cfg.anchor_bits;
  c.dict_bits = cfg.dict_bits;
  c.diff_bits = cfg.diff_bits;
  c.anchor_strategy = (int)cfg.anchor_strategy;
  c.seed = cfg.seed;
  c.raw_payload = cfg.raw_payload;
  c.oi_rounds = cfg.oi_rounds;
  c.oi_seed = cfg.oi_seed;
  c.oi_implicit = cfg.oi_implicit;
  c.oi_tolerance = cfg.oi_tolerance;
  const uint32_t n = (uint32_t)s.n(), F = (uint32_t)s.k();
  dmcg_sizes sz;
  detail::check(dmcg_encoded_sizes(n, F, &c, &sz));
  std::vector<uint32_t> faces;
  faces.reserve(s.faces().size() * 3);
  for (const Face& f : s.faces()) faces.insert(faces.end(), f.begin(), f.end());
  std::array<std::vector<uint16_t>, 3> dq, cq, aq;
  std::array<std::vector<float>, 3> rmin, rmax;
  std::array<std::vector<uint8_t>, 3> rbits;
  std::array<std::vector<float>, 3> dmin, dmax;
  CompressedAnimation out;
  out.anchor_indices.resize(sz.anchor_idx);
  dmcg_encoded e{};
  for (int a = 0; a < 3; ++a) {
    dmin[a].resize(sz.dict_ranges + 1);
    dmax[a].resize(sz.dict_ranges + 1);
    e.diff_min[a] = dmin[a].data();
    e.diff_max[a] = dmax[a].data();
    out.means[a].resize(sz.means);
    e.means[a] = sz.means ? out.means[a].data() : nullptr;
    dq[a].resize(sz.dict_q);
    cq[a].resize(sz.coeff_q + 1);
    aq[a].resize(sz.anchor_q);
    rmin[a].resize(sz.rows + 1);
    rmax[a].resize(sz.rows + 1);
    rbits[a].resize(sz.rows + 1);
    e.dict_q[a] = dq[a].data();
    e.coeff_q[a] = cq[a].data();
    e.anchor_q[a] = aq[a].data();
    e.row_min[a] = rmin[a].data();
    e.row_max[a] = rmax[a].data();
    e.row_bits[a] = rbits[a].data();
  }
  e.anchor_idx = out.anchor_indices.data();
  e.faces = faces.data();
  dmcg_seq q{n, F, DMCG_F64, {s.axis(0).data(), s.axis(1).data(), s.axis(2).data()},
             faces.data(), (uint32_t)s.faces().size()};
  detail::check(dmcg_encode(detail::Ctx::get().c, &q, &c, &e));
  out.variant = cfg.variant;
  out.n = n;
  out.k = F;
  out.k_l = cfg.k_l;
  out.n_b = sz.n_b;
  out.pad = sz.pad;
  out.n_c = e.n_c;
  out.anchor_bits = e.anchor_bits;
  out.dict_bits = e.dict_bits;
  out.diff_bits = e.diff_bits;
  out.faces = s.faces();
  const size_t kk = (size_t)out.k_f() * out.k_f(), rows = (size_t)out.n_b * cfg.k_l;
  for (int a = 0; a < 3; ++a) {
    out.dict_first[a].assign(dq[a].begin(), dq[a].begin() + kk);
    for (uint32_t b = 1; b < out.n_b; ++b) {
      DictDiff d;
      d.min = dmin[a][b - 1];
      d.max = dmax[a][b - 1];
      d.q.assign(dq[a].begin() + b * kk, dq[a].begin() + (b + 1) * kk);
      out.dict_diffs[a].push_back(std::move(d));
    }
    out.anchor_q[a].assign(aq[a].begin(), aq[a].end());
    out.anchor_min[a] = e.anchor_min[a];
    out.anchor_max[a] = e.anchor_max[a];
    out.coeffs[a].resize(rows);
    for (uint32_t r = 0; r < rows; ++r) {
      QuantRow& row = out.coeffs[a][r];
      row.min = rmin[a][r];
      row.max = rmax[a][r];
      row.bits = rbits[a][r];
      if (!(row.min == row.max))
        row.q.assign(cq[a].begin() + (size_t)r * n, cq[a].begin() + (size_t)(r + 1) * n);
    }
  }
  return out;
}

// dmc::decode (reference codec.hpp:91).
inline MeshSequence decode(const CompressedAnimation& c, double cg_rtol = 1e-10) {
  const uint32_t n = c.n, F = c.k;
  std::vector<uint32_t> faces;
  for (const Face& f : c.faces) faces.insert(faces.end(), f.begin(), f.end());
  std::array<std::vector<uint16_t>, 3> dq, cq, aq;
  std::array<std::vector<float>, 3> rmin, rmax;
  std::array<std::vector<uint8_t>, 3> rbits;
  std::array<std::vector<float>, 3> dmin, dmax;
  std::vector<uint32_t> idx(c.anchor_indices);
  const uint32_t nb = c.n_b ? c.n_b : 1;
  const size_t kk = (size_t)((F + c.pad) / nb) * ((F + c.pad) / nb), rows = (size_t)nb * c.k_l;
  dmcg_encoded e{};
  e.n = n;
  e.F = F;
  e.k_l = c.k_l;
  e.n_b = (uint16_t)nb;
  e.pad = c.pad;
  e.n_c = c.n_c;
  e.n_faces = (uint32_t)c.faces.size();
  e.variant = (uint8_t)c.variant;
  e.anchor_bits = c.anchor_bits;
  e.dict_bits = c.dict_bits;
  e.diff_bits = c.diff_bits;
  e.faces = faces.data();
  e.anchor_idx = idx.data();
  for (int a = 0; a < 3; ++a) {
    if (c.dict_first[a].size() != kk || c.dict_diffs[a].size() != nb - 1 ||
        c.coeffs[a].size() != rows ||
        c.anchor_q[a].size() != (size_t)c.n_c * F ||
        ((c.variant == Variant::Pca || c.variant == Variant::PcaQ) && c.means[a].size() != F))
      throw Error(6, "CorruptPayload: payload has wrong element count");
    e.means[a] = c.means[a].empty() ? nullptr : const_cast<float*>(c.means[a].data());
    dq[a].assign(c.dict_first[a].begin(), c.dict_first[a].end());
    dmin[a].resize(nb);
    dmax[a].resize(nb);
    for (uint32_t b = 1; b < nb; ++b) {
      const DictDiff& d = c.dict_diffs[a][b - 1];
      if (d.q.size() != kk) throw Error(6, "CorruptPayload: dictionary payload has wrong element count");
      dq[a].insert(dq[a].end(), d.q.begin(), d.q.end());
      dmin[a][b - 1] = d.min;
      dmax[a][b - 1] = d.max;
    }
    e.diff_min[a] = dmin[a].data();
    e.diff_max[a] = dmax[a].data();
    aq[a].assign(c.anchor_q[a].begin(), c.anchor_q[a].end());
    cq[a].assign(rows * n + 1, 0);
    rmin[a].resize(rows + 1);
    rmax[a].resize(rows + 1);
    rbits[a].resize(rows + 1);
    for (uint32_t r = 0; r < rows; ++r) {
      const QuantRow& row = c.coeffs[a][r];
      rmin[a][r] = row.min;
      rmax[a][r] = row.max;
      rbits[a][r] = row.bits;
      if (!(row.min == row.max)) {
        if (row.q.size() != n) throw Error(6, "CorruptPayload: row payload has wrong element count");
        for (uint32_t i = 0; i < n; ++i) {
          if (row.q[i] >= (1u << row.bits)) throw Error(6, "CorruptPayload: packed value out of range");
          cq[a][(size_t)r * n + i] = (uint16_t)row.q[i];
        }
      }
    }
    e.dict_q[a] = dq[a].data();
    e.coeff_q[a] = cq[a].data();
    e.anchor_q[a] = aq[a].data();
    e.row_min[a] = rmin[a].data();
    e.row_max[a] = rmax[a].data();
    e.row_bits[a] = rbits[a].data();
    e.anchor_min[a] = c.anchor_min[a];
    e.anchor_max[a] = c.anchor_max[a];
  }
  std::array<Matrix, 3> axes{Matrix(F, n), Matrix(F, n), Matrix(F, n)};
  void* outs[3] = {axes[0].data(), axes[1].data(), axes[2].data()};
  dmcg_decode_options opt;
  dmcg_decode_options_default(&opt);
  opt.cg_rtol = cg_rtol;
  detail::check(dmcg_decode(detail::Ctx::get().c, &e, &opt, outs, DMCG_F64));
  return MeshSequence(c.faces, std::move(axes));
}

}  // namespace dmc
