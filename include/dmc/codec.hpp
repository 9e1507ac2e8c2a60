// dmc/codec.hpp — Eigen-free C++ drop-in for the reference encoder/decoder
// API (reference include/dmc/codec.hpp:28-91), header-only over the libdmcg C
// ABI (include/dmcg.h).  Link with -ldmcg.  Together with dmc/errors.hpp,
// dmc/mesh.hpp, dmc/stream.hpp and dmc/metrics.hpp it keeps the reference's
// type names, member names and signatures, so a reference caller recompiles
// against it unchanged:
//
//   dmc::CompressedAnimation c = dmc::encode(seq, cfg);      // codec.hpp:90
//   c.axes[a].coeffs[0].rows[r].q; c.anchors[a].min;           // stream.hpp:130-155
//   std::vector<uint8_t> bytes = dmc::serialize(c);            // stream.hpp:177
//   dmc::MeshSequence out = dmc::decode(dmc::parse(bytes));    // codec.hpp:91
//   double bvpv = dmc::rate_exact(c).q_s;                      // metrics.hpp:50-51
//
// Differences from the reference, forced by the environment or the scope:
//   * dmc::Matrix replaces Eigen::MatrixXd (same column-major layout).
//   * EncoderConfig gains the B200 basis controls oi_rounds / oi_seed /
//     oi_implicit (0 rounds = the reference's full eigenbasis), and decode()
//     takes optional solver controls (DecodeOptions).
//   * Variants pca, pca_q, v2v, pca_qs, pca_qp and blocks run on the GPU;
//     per_mesh_gft, raw payloads and the normalized Laplacian throw
//     dmc::Unsupported (code 11).
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "../dmcg.h"
#include "errors.hpp"
#include "mesh.hpp"
#include "metrics.hpp"
#include "stream.hpp"

namespace dmc {

enum class LaplacianKind : uint8_t { Combinatorial = 0, Normalized = 1 };  // laplacian.hpp:26-29
enum class AnchorStrategy : uint8_t { Stride = 0, SeededRandom = 1 };

struct EncoderConfig {  // reference codec.hpp:30-49 (+ B200 basis controls)
  Variant variant = Variant::PcaQp;
  uint32_t k_l = 20;
  std::vector<int> row_bits;  // one entry per retained row; empty = all 16
  uint16_t n_b = 1;           // > 1 requires variant blocks
  int t_max = 4;
  double anchor_fraction = 0.01;
  int anchor_bits = 16;
  int dict_bits = 16;
  int diff_bits = 8;
  AnchorStrategy anchor_strategy = AnchorStrategy::Stride;
  uint64_t seed = 0;
  LaplacianKind laplacian = LaplacianKind::Combinatorial;
  bool raw_payload = false;
  std::optional<double> oi_tolerance;
  // B200 basis (dmcg_config): 0 = the reference's full F x F eigenbasis
  // (codec.cpp:158-159); N > 0 = rank-k_l orthogonal iterations (N rounds).
  int oi_rounds = 0;
  uint64_t oi_seed = 0;
  bool oi_implicit = false;  // never form R = X^T X: Z = X^T (X Q) per round
};

// B200 decoder controls (dmcg_decode_options); defaults = the reference's
// factor + solve + one refinement (solver.cpp:62-90).
struct DecodeOptions {
  double cg_rtol = 1e-10;
  int solver = 0;  // 0 supernodal Cholesky, 1 conjugate gradients
  int refine = 1;
};

namespace detail {
struct Ctx {
  dmcg_ctx* c = nullptr;
  Ctx() {
    int rc = dmcg_create(&c, 0);
    if (rc) throw CudaError("dmcg_create failed");
  }
  ~Ctx() { dmcg_destroy(c); }
  static Ctx& get() {
    thread_local Ctx ctx;  // one context (stream + pool) per calling thread
    return ctx;
  }
};
inline void check(int rc) {
  if (rc) raise(rc, dmcg_last_error(Ctx::get().c));
}
inline dmcg_config to_c(const EncoderConfig& cfg) {
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
  c.laplacian = (int)cfg.laplacian;
  c.raw_payload = cfg.raw_payload;
  c.oi_rounds = cfg.oi_rounds;
  c.oi_seed = cfg.oi_seed;
  c.oi_implicit = cfg.oi_implicit ? 1 : 0;
  c.oi_tolerance = cfg.oi_tolerance ? *cfg.oi_tolerance : -1.0;
  return c;
}
}  // namespace detail

// max(1, round(fraction * n)) (codec.cpp:199-202).
inline uint32_t anchor_count(uint32_t n, double fraction) { return dmcg_anchor_count(n, fraction); }

// select_anchors (codec.cpp:204-238): sorted indices.
inline std::vector<uint32_t> select_anchors(uint32_t n, uint32_t n_c, AnchorStrategy s, uint64_t seed) {
  std::vector<uint32_t> out(n_c ? n_c : 1);
  int rc = dmcg_select_anchors(n, n_c, (int)s, seed, out.data());
  if (rc) throw InvalidCount("anchor count " + std::to_string(n_c) + " outside 1.." + std::to_string(n));
  out.resize(n_c);
  return out;
}

// dmc::encode (reference codec.hpp:90; src/codec.cpp:351-473).
inline CompressedAnimation encode(const MeshSequence& s, const EncoderConfig& cfg) {
  if (cfg.laplacian != LaplacianKind::Combinatorial)
    throw Unsupported("the normalized Laplacian is outside the B200 path");
  const dmcg_config c = detail::to_c(cfg);
  const uint32_t n = (uint32_t)s.n(), F = (uint32_t)s.k();
  dmcg_sizes sz;
  detail::check(dmcg_encoded_sizes(n, F, &c, &sz));
  detail::CBuffers b;
  b.allocate(n, F, cfg.k_l, (uint32_t)sz.anchor_idx, (uint32_t)s.faces().size(), sz.n_b, sz.pad);
  b.faces = flat_faces(s.faces());
  b.bind();
  dmcg_seq q{n, F, DMCG_F64, {s.axis(0).data(), s.axis(1).data(), s.axis(2).data()},
             b.faces.data(), (uint32_t)s.faces().size()};
  detail::check(dmcg_encode(detail::Ctx::get().c, &q, &c, &b.e));
  b.e.variant = (uint8_t)cfg.variant;
  b.e.k_l = cfg.k_l;
  b.e.n_b = sz.n_b;
  b.e.pad = sz.pad;
  return b.store();
}

// dmc::decode (reference codec.hpp:91; src/codec.cpp:475-552).
inline MeshSequence decode(const CompressedAnimation& c, const DecodeOptions& o) {
  detail::CBuffers b;
  b.load(c);
  const uint32_t n = c.n, F = c.k;
  std::array<Matrix, 3> axes{Matrix(F, n), Matrix(F, n), Matrix(F, n)};
  void* outs[3] = {axes[0].data(), axes[1].data(), axes[2].data()};
  dmcg_decode_options opt;
  dmcg_decode_options_default(&opt);
  opt.cg_rtol = o.cg_rtol;
  opt.solver = o.solver;
  opt.refine = o.refine;
  detail::check(dmcg_decode(detail::Ctx::get().c, &b.e, &opt, outs, DMCG_F64));
  return MeshSequence(c.faces, std::move(axes));
}
inline MeshSequence decode(const CompressedAnimation& c) { return decode(c, DecodeOptions{}); }

}  // namespace dmc
