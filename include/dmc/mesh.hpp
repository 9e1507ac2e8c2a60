// dmc/mesh.hpp — Eigen-free mirror of the reference include/dmc/mesh.hpp
// (MeshSequence :36-57, Connectivity :60-65, build_connectivity :69,
// is_connected :72, validate_sequence :81).
//
// dmc::Matrix stands in for Eigen::MatrixXd (Eigen3 is absent, reference
// CMakeLists.txt:11): column-major with rows()/cols()/data()/operator()/row()
// — the same memory layout, so MeshSequence::axis(a).data() is exactly the
// vertex-major n x F buffer libdmcg reads (x[i*F + f]) and a reference caller
// can copy Eigen::MatrixXd::data() straight in.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <deque>
#include <string>
#include <vector>

#include "../dmcg.h"
#include "errors.hpp"

namespace dmc {

// Column-major dense matrix (the Eigen::MatrixXd layout).
class Matrix {
 public:
  Matrix() = default;
  Matrix(int64_t r, int64_t c) : r_(r), c_(c), d_((size_t)(r * c), 0.0) {}
  int64_t rows() const { return r_; }
  int64_t cols() const { return c_; }
  int64_t size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(int64_t i, int64_t j) { return d_[(size_t)(j * r_ + i)]; }
  double operator()(int64_t i, int64_t j) const { return d_[(size_t)(j * r_ + i)]; }
  std::vector<double> row(int64_t i) const {
    std::vector<double> out((size_t)c_);
    for (int64_t j = 0; j < c_; ++j) out[(size_t)j] = (*this)(i, j);
    return out;
  }
  bool allFinite() const {
    for (double v : d_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }

 private:
  int64_t r_ = 0, c_ = 0;
  std::vector<double> d_;
};

using Face = std::array<uint32_t, 3>;

enum class Axis : int { X = 0, Y = 1, Z = 2 };

/// An animation of k frames over a fixed triangle connectivity (reference
/// mesh.hpp:33-57): three k x n axis matrices whose row f holds frame f.
class MeshSequence {
 public:
  MeshSequence() = default;
  MeshSequence(std::vector<Face> faces, std::array<Matrix, 3> axes)
      : faces_(std::move(faces)), axes_(std::move(axes)) {
    for (int a = 1; a < 3; ++a)
      if (axes_[a].rows() != axes_[0].rows() || axes_[a].cols() != axes_[0].cols())
        throw DimensionMismatch("axis matrices must share one k x n shape");
  }

  // Builds the axis-major storage from per-frame n x 3 matrices (mesh.cpp:36-47).
  static MeshSequence from_frames(std::vector<Face> faces, const std::vector<Matrix>& frames) {
    if (frames.empty()) throw DimensionMismatch("no frames");
    const int64_t n = frames[0].rows(), k = (int64_t)frames.size();
    std::array<Matrix, 3> axes{Matrix(k, n), Matrix(k, n), Matrix(k, n)};
    for (int64_t f = 0; f < k; ++f) {
      if (frames[(size_t)f].rows() != n || frames[(size_t)f].cols() != 3)
        throw DimensionMismatch("every frame must be n x 3");
      for (int a = 0; a < 3; ++a)
        for (int64_t i = 0; i < n; ++i) axes[a](f, i) = frames[(size_t)f](i, a);
    }
    return MeshSequence(std::move(faces), std::move(axes));
  }

  int n() const { return static_cast<int>(axes_[0].cols()); }
  int k() const { return static_cast<int>(axes_[0].rows()); }
  const std::vector<Face>& faces() const { return faces_; }
  const Matrix& axis(Axis a) const { return axes_[static_cast<int>(a)]; }
  const Matrix& axis(int a) const { return axes_[a]; }
  Matrix frame(int f) const {
    Matrix out(n(), 3);
    for (int a = 0; a < 3; ++a)
      for (int i = 0; i < n(); ++i) out(i, a) = axes_[a](f, i);
    return out;
  }
  bool operator==(const MeshSequence& o) const { return faces_ == o.faces_ && axes_ == o.axes_; }

 private:
  std::vector<Face> faces_;
  std::array<Matrix, 3> axes_;  // each k x n
};

/// First-ring vertex adjacency: sorted, deduplicated neighbour lists.
struct Connectivity {
  int n = 0;
  std::vector<std::vector<uint32_t>> neighbors;
  int degree(int i) const { return static_cast<int>(neighbors[i].size()); }
};

inline std::vector<uint32_t> flat_faces(const std::vector<Face>& faces) {
  std::vector<uint32_t> out;
  out.reserve(faces.size() * 3);
  for (const Face& f : faces) out.insert(out.end(), f.begin(), f.end());
  return out;
}

// build_connectivity (reference mesh.hpp:69): IndexOutOfRange / DegenerateFace
// on bad faces.  libdmcg's dmcg_build_connectivity does the work.
inline Connectivity build_connectivity(const std::vector<Face>& faces, int n) {
  const std::vector<uint32_t> flat = flat_faces(faces);
  std::vector<uint32_t> rp((size_t)n + 1), col(6 * faces.size() + 1);
  size_t nnz = 0;
  int rc = dmcg_build_connectivity(flat.data(), (uint32_t)faces.size(), (uint32_t)n, rp.data(),
                                   col.data(), col.size(), &nnz);
  if (rc) detail::raise(rc, dmcg_host_error());
  Connectivity c;
  c.n = n;
  c.neighbors.resize((size_t)n);
  for (int i = 0; i < n; ++i) c.neighbors[(size_t)i].assign(col.begin() + rp[i], col.begin() + rp[i + 1]);
  return c;
}

// is_connected (mesh.hpp:72): BFS over the neighbour lists.
inline bool is_connected(const Connectivity& c) {
  if (c.n == 0) return true;
  std::vector<char> seen((size_t)c.n, 0);
  std::deque<uint32_t> q{0};
  seen[0] = 1;
  int visited = 1;
  while (!q.empty()) {
    const uint32_t v = q.front();
    q.pop_front();
    for (uint32_t w : c.neighbors[v])
      if (!seen[w]) {
        seen[w] = 1;
        ++visited;
        q.push_back(w);
      }
  }
  return visited == c.n;
}

struct ValidationReport {
  std::vector<std::string> issues;
  bool ok() const { return issues.empty(); }
};

// validate_sequence (mesh.hpp:81, mesh.cpp:108-136): at least one face, no
// isolated vertex, a connected vertex graph, finite coordinates.
inline ValidationReport validate_sequence(const MeshSequence& s) {
  ValidationReport r;
  if (s.faces().empty()) {
    r.issues.push_back("face list is empty");
    return r;
  }
  const Connectivity c = build_connectivity(s.faces(), s.n());
  for (int i = 0; i < c.n; ++i)
    if (c.degree(i) == 0) {
      r.issues.push_back("vertex " + std::to_string(i) + " is isolated");
      break;
    }
  if (!is_connected(c)) r.issues.push_back("graph not connected");
  static const char* names[3] = {"x", "y", "z"};
  for (int a = 0; a < 3; ++a)
    if (!s.axis(a).allFinite()) r.issues.push_back(std::string("non-finite coordinate on axis ") + names[a]);
  return r;
}

inline const Matrix& sequence_axis_matrix(const MeshSequence& s, Axis axis) { return s.axis(axis); }

}  // namespace dmc
