// dmc/stream.hpp — Eigen-free mirror of the reference include/dmc/stream.hpp
// (Variant :60-68, QuantRow :86-93, CoeffBlock :95-100, DictDiff :102-108,
// AxisPayload :110-119, AnchorAxis :121-128, CompressedAnimation :130-155,
// SectionSizes :159-175, serialize / parse :177-182) over the libdmcg C ABI
// (dmcg_serialize / dmcg_parse, the DMC1 byte format of src/stream.cpp:172-469).
//
// Same member names and nesting as the reference, so reference callers
// (`c.axes[a].coeffs[0].rows[r].q`, `c.anchors[a].min`, `c.anchor_indices`)
// compile unchanged.  The raw-payload debug members (dict_raw, CoeffBlock::raw,
// means_raw, AnchorAxis::raw) exist for source compatibility; the B200 path
// never fills them and refuses streams that carry kFlagRawPayload
// (dmc::Unsupported), as it refuses per_mesh_gft.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "../dmcg.h"
#include "errors.hpp"
#include "mesh.hpp"

namespace dmc {

enum class Variant : uint8_t {
  Pca = 0,
  PcaQ = 1,
  V2v = 2,
  PcaQs = 3,
  PcaQp = 4,
  Blocks = 5,
  PerMeshGft = 6,
};

constexpr uint16_t kStreamVersion = 1;
constexpr uint8_t kFlagRawPayload = 0x01;
constexpr uint8_t kFlagNormalizedLaplacian = 0x02;

inline const char* variant_name(Variant v) {
  switch (v) {
    case Variant::Pca: return "pca";
    case Variant::PcaQ: return "pca_q";
    case Variant::V2v: return "v2v";
    case Variant::PcaQs: return "pca_qs";
    case Variant::PcaQp: return "pca_qp";
    case Variant::Blocks: return "blocks";
    case Variant::PerMeshGft: return "per_mesh_gft";
  }
  return "unknown";
}
inline std::optional<Variant> variant_from_name(const std::string& name) {
  for (int v = 0; v <= 6; ++v)
    if (name == variant_name((Variant)v)) return (Variant)v;
  return std::nullopt;
}
inline bool variant_uses_anchors(Variant v) {
  return v == Variant::PcaQs || v == Variant::PcaQp || v == Variant::Blocks;
}
inline bool variant_uses_means(Variant v) {
  return v == Variant::Pca || v == Variant::PcaQ || v == Variant::PerMeshGft;
}
inline bool variant_uses_delta(Variant v) { return v != Variant::V2v; }

struct QuantRow {
  float min = 0.0f;
  float max = 0.0f;
  uint8_t bits = 0;
  std::vector<uint32_t> q;  // empty when min == max
  bool operator==(const QuantRow& o) const {
    return min == o.min && max == o.max && bits == o.bits && q == o.q;
  }
};

struct CoeffBlock {
  std::vector<QuantRow> rows;  // quantized path, k_l entries
  Matrix raw;                  // raw path (unused on the B200 path)
  bool operator==(const CoeffBlock& o) const { return rows == o.rows && raw == o.raw; }
};

struct DictDiff {
  float min = 0.0f;
  float max = 0.0f;
  std::vector<uint32_t> q;
  bool operator==(const DictDiff& o) const { return min == o.min && max == o.max && q == o.q; }
};

struct AxisPayload {
  std::vector<uint32_t> dict_first;  // k_f*k_f levels at dict_bits, column-major
  std::vector<DictDiff> dict_diffs;  // blocks 2..n_b
  std::vector<Matrix> dict_raw;      // raw path (unused)
  std::vector<CoeffBlock> coeffs;    // n_b entries
  std::vector<float> means;          // k entries (pca / pca_q)
  std::vector<double> means_raw;     // raw path (unused)
  bool operator==(const AxisPayload& o) const {
    return dict_first == o.dict_first && dict_diffs == o.dict_diffs && dict_raw == o.dict_raw &&
           coeffs == o.coeffs && means == o.means && means_raw == o.means_raw;
  }
};

struct AnchorAxis {
  float min = 0.0f;
  float max = 0.0f;
  std::vector<uint32_t> q;  // n_c*k levels, anchor-major
  std::vector<double> raw;  // raw path (unused)
  bool operator==(const AnchorAxis& o) const {
    return min == o.min && max == o.max && q == o.q && raw == o.raw;
  }
};

struct CompressedAnimation {
  uint16_t version = kStreamVersion;
  Variant variant = Variant::Pca;
  uint8_t flags = 0;
  uint32_t n = 0;
  uint32_t k = 0;
  uint16_t n_b = 1;
  uint16_t pad = 0;
  uint32_t k_l = 0;
  uint32_t n_c = 0;
  uint8_t anchor_bits = 16;
  uint8_t dict_bits = 16;
  uint8_t diff_bits = 8;
  std::vector<Face> faces;
  std::array<AxisPayload, 3> axes;
  std::vector<uint32_t> anchor_indices;
  std::array<AnchorAxis, 3> anchors;

  uint32_t k_padded() const { return k + pad; }
  uint32_t k_f() const { return k_padded() / n_b; }
  uint32_t coeff_width() const { return variant == Variant::PerMeshGft ? k : n; }
  bool raw_payload() const { return (flags & kFlagRawPayload) != 0; }
  bool normalized_laplacian() const { return (flags & kFlagNormalizedLaplacian) != 0; }
  bool operator==(const CompressedAnimation& o) const {
    return version == o.version && variant == o.variant && flags == o.flags && n == o.n &&
           k == o.k && n_b == o.n_b && pad == o.pad && k_l == o.k_l && n_c == o.n_c &&
           anchor_bits == o.anchor_bits && dict_bits == o.dict_bits && diff_bits == o.diff_bits &&
           faces == o.faces && axes == o.axes && anchor_indices == o.anchor_indices &&
           anchors == o.anchors;
  }
};

/// Byte extents of each stream section (stream.hpp:159-175).
struct SectionSizes {
  size_t header = 0;
  size_t connectivity = 0;
  size_t dict_payload = 0;
  size_t dict_ranges = 0;
  size_t coeff_headers = 0;
  size_t coeff_payload = 0;
  size_t means = 0;
  size_t anchor_indices = 0;
  size_t anchor_ranges = 0;
  size_t anchor_payload = 0;
  size_t total() const {
    return header + connectivity + dict_payload + dict_ranges + coeff_headers + coeff_payload +
           means + anchor_indices + anchor_ranges + anchor_payload;
  }
};

namespace detail {

inline SectionSizes from_c(const dmcg_sections& s) {
  SectionSizes o;
  o.header = s.header;
  o.connectivity = s.connectivity;
  o.dict_payload = s.dict_payload;
  o.dict_ranges = s.dict_ranges;
  o.coeff_headers = s.coeff_headers;
  o.coeff_payload = s.coeff_payload;
  o.means = s.means;
  o.anchor_indices = s.anchor_indices;
  o.anchor_ranges = s.anchor_ranges;
  o.anchor_payload = s.anchor_payload;
  return o;
}

// The flat 16-bit arrays libdmcg reads and writes (dmcg_encoded), owned here.
// Level counts follow dmcg.h: dict n_b k_f^2, rows n_b k_l, coefficients
// n_b k_l n, anchors n_c k, means k per axis.
struct CBuffers {
  dmcg_encoded e{};
  std::vector<uint32_t> faces, anchor_idx;
  std::array<std::vector<uint16_t>, 3> dq, cq, aq;
  std::array<std::vector<float>, 3> rmin, rmax, dmin, dmax, means;
  std::array<std::vector<uint8_t>, 3> rbits;

  void allocate(uint32_t n, uint32_t F, uint32_t k_l, uint32_t n_c, uint32_t n_faces, uint16_t n_b,
                uint16_t pad) {
    const size_t nb = n_b ? n_b : 1, kf = (F + pad) / nb, rows = nb * k_l;
    faces.assign(3 * (size_t)n_faces, 0);
    anchor_idx.assign((size_t)n_c + 1, 0);
    for (int a = 0; a < 3; ++a) {
      dq[a].assign(nb * kf * kf + 1, 0);
      cq[a].assign(rows * n + 1, 0);
      aq[a].assign((size_t)n_c * F + 1, 0);
      rmin[a].assign(rows + 1, 0.0f);
      rmax[a].assign(rows + 1, 0.0f);
      rbits[a].assign(rows + 1, 0);
      dmin[a].assign(nb, 0.0f);
      dmax[a].assign(nb, 0.0f);
      means[a].assign((size_t)F + 1, 0.0f);
    }
    e.n = n;
    e.F = F;
    e.k_l = k_l;
    e.n_c = n_c;
    e.n_faces = n_faces;
    e.n_b = (uint16_t)nb;
    e.pad = pad;
    bind();
  }
  void bind() {
    e.faces = faces.data();
    e.anchor_idx = anchor_idx.data();
    for (int a = 0; a < 3; ++a) {
      e.dict_q[a] = dq[a].data();
      e.coeff_q[a] = cq[a].data();
      e.anchor_q[a] = aq[a].data();
      e.row_min[a] = rmin[a].data();
      e.row_max[a] = rmax[a].data();
      e.row_bits[a] = rbits[a].data();
      e.diff_min[a] = dmin[a].data();
      e.diff_max[a] = dmax[a].data();
      e.means[a] = means[a].data();
    }
  }

  // CompressedAnimation -> flat arrays, with the reference decoder's payload
  // checks (CorruptPayload on a wrong element count or a level >= 2^bits,
  // codec.cpp:133-134,283) done before any value is narrowed to 16 bits.
  void load(const CompressedAnimation& c) {
    if (c.raw_payload()) throw Unsupported("raw payload streams are outside the B200 path");
    if (c.variant == Variant::PerMeshGft) throw Unsupported("per_mesh_gft is outside the B200 path");
    const uint32_t nb = c.n_b ? c.n_b : 1, n = c.n, F = c.k;
    allocate(n, F, c.k_l, c.n_c, (uint32_t)c.faces.size(), (uint16_t)nb, c.pad);
    e.variant = (uint8_t)c.variant;
    e.flags = c.flags;
    e.anchor_bits = c.anchor_bits;
    e.dict_bits = c.dict_bits;
    e.diff_bits = c.diff_bits;
    for (size_t t = 0; t < c.faces.size(); ++t)
      for (int j = 0; j < 3; ++j) faces[3 * t + j] = c.faces[t][j];
    if (c.anchor_indices.size() != c.n_c) throw CorruptPayload("anchor index count differs from n_c");
    for (uint32_t t = 0; t < c.n_c; ++t) anchor_idx[t] = c.anchor_indices[t];
    const size_t kf = c.k_f(), kk = kf * kf;
    auto narrow = [](const std::vector<uint32_t>& src, int bits, uint16_t* dst, const char* what) {
      const uint32_t lim = bits >= 32 ? 0xffffffffu : (1u << bits);
      for (size_t i = 0; i < src.size(); ++i) {
        if (src[i] >= lim) throw CorruptPayload(std::string(what) + " level out of range");
        dst[i] = (uint16_t)src[i];
      }
    };
    for (int a = 0; a < 3; ++a) {
      const AxisPayload& ax = c.axes[a];
      if (ax.dict_first.size() != kk || ax.dict_diffs.size() != nb - 1 || ax.coeffs.size() != nb)
        throw CorruptPayload("dictionary or coefficient payload has wrong element count");
      narrow(ax.dict_first, c.dict_bits, dq[a].data(), "dictionary");
      for (uint32_t b = 1; b < nb; ++b) {
        const DictDiff& d = ax.dict_diffs[b - 1];
        if (d.q.size() != kk) throw CorruptPayload("dictionary difference has wrong element count");
        narrow(d.q, c.diff_bits, dq[a].data() + b * kk, "dictionary difference");
        dmin[a][b - 1] = d.min;
        dmax[a][b - 1] = d.max;
      }
      for (uint32_t b = 0; b < nb; ++b) {
        const CoeffBlock& blk = ax.coeffs[b];
        if (blk.rows.size() != c.k_l) throw CorruptPayload("coefficient block has wrong row count");
        for (uint32_t r = 0; r < c.k_l; ++r) {
          const QuantRow& row = blk.rows[r];
          const size_t rr = (size_t)b * c.k_l + r;
          rmin[a][rr] = row.min;
          rmax[a][rr] = row.max;
          rbits[a][rr] = row.bits;
          if (row.min == row.max) continue;  // degenerate rows carry no payload
          if (row.q.size() != c.coeff_width()) throw CorruptPayload("row payload has wrong element count");
          narrow(row.q, row.bits, cq[a].data() + rr * n, "coefficient");
        }
      }
      if (variant_uses_means(c.variant)) {
        if (ax.means.size() != F) throw CorruptPayload("means payload has wrong element count");
        std::copy(ax.means.begin(), ax.means.end(), means[a].begin());
      }
      const AnchorAxis& an = c.anchors[a];
      if (an.q.size() != (size_t)c.n_c * F) throw CorruptPayload("anchor payload has wrong element count");
      narrow(an.q, c.anchor_bits, aq[a].data(), "anchor");
      e.anchor_min[a] = an.min;
      e.anchor_max[a] = an.max;
    }
    if (!variant_uses_means(c.variant))
      for (int a = 0; a < 3; ++a) e.means[a] = nullptr;
  }

  // flat arrays -> CompressedAnimation (after an encode or a parse)
  CompressedAnimation store() const {
    CompressedAnimation c;
    c.variant = (Variant)e.variant;
    c.flags = e.flags;
    c.n = e.n;
    c.k = e.F;
    c.n_b = e.n_b ? e.n_b : 1;
    c.pad = e.pad;
    c.k_l = e.k_l;
    c.n_c = e.n_c;
    c.anchor_bits = e.anchor_bits;
    c.dict_bits = e.dict_bits;
    c.diff_bits = e.diff_bits;
    c.faces.resize(e.n_faces);
    for (size_t t = 0; t < c.faces.size(); ++t)
      c.faces[t] = {faces[3 * t], faces[3 * t + 1], faces[3 * t + 2]};
    c.anchor_indices.assign(anchor_idx.begin(), anchor_idx.begin() + e.n_c);
    const size_t kf = c.k_f(), kk = kf * kf, n = c.n;
    for (int a = 0; a < 3; ++a) {
      AxisPayload& ax = c.axes[a];
      ax.dict_first.assign(dq[a].begin(), dq[a].begin() + kk);
      for (uint32_t b = 1; b < c.n_b; ++b) {
        DictDiff d;
        d.min = dmin[a][b - 1];
        d.max = dmax[a][b - 1];
        d.q.assign(dq[a].begin() + b * kk, dq[a].begin() + (b + 1) * kk);
        ax.dict_diffs.push_back(std::move(d));
      }
      ax.coeffs.resize(c.n_b);
      for (uint32_t b = 0; b < c.n_b; ++b) {
        ax.coeffs[b].rows.resize(c.k_l);
        for (uint32_t r = 0; r < c.k_l; ++r) {
          const size_t rr = (size_t)b * c.k_l + r;
          QuantRow& row = ax.coeffs[b].rows[r];
          row.min = rmin[a][rr];
          row.max = rmax[a][rr];
          row.bits = rbits[a][rr];
          if (!(row.min == row.max)) row.q.assign(cq[a].begin() + rr * n, cq[a].begin() + (rr + 1) * n);
        }
      }
      if (variant_uses_means(c.variant)) ax.means.assign(means[a].begin(), means[a].begin() + c.k);
      AnchorAxis& an = c.anchors[a];
      an.min = e.anchor_min[a];
      an.max = e.anchor_max[a];
      an.q.assign(aq[a].begin(), aq[a].begin() + (size_t)c.n_c * c.k);
    }
    return c;
  }
};

}  // namespace detail

// serialize (stream.hpp:177; src/stream.cpp:172-292): the DMC1 byte stream.
inline std::vector<uint8_t> serialize(const CompressedAnimation& c, SectionSizes* sizes = nullptr) {
  detail::CBuffers b;
  b.load(c);
  dmcg_sections s{};
  const size_t size = dmcg_serialize(&b.e, nullptr, 0, &s);
  if (size == 0) throw CorruptPayload("stream could not be framed");
  std::vector<uint8_t> out(size);
  dmcg_serialize(&b.e, out.data(), out.size(), &s);
  if (sizes) *sizes = detail::from_c(s);
  return out;
}

// parse (stream.hpp:181-182; src/stream.cpp:294-469): strict, throws
// CorruptStream / VersionMismatch like the reference.
inline CompressedAnimation parse(const uint8_t* data, size_t size, SectionSizes* sizes = nullptr) {
  dmcg_encoded hdr{};
  int rc = dmcg_parse_header(data, size, &hdr);
  if (rc) detail::raise(rc, dmcg_parse_error());
  detail::CBuffers b;
  b.allocate(hdr.n, hdr.F, hdr.k_l, hdr.n_c, hdr.n_faces, hdr.n_b, hdr.pad);
  dmcg_sections s{};
  rc = dmcg_parse(data, size, &b.e, &s);
  if (rc) detail::raise(rc, dmcg_parse_error());
  if (sizes) *sizes = detail::from_c(s);
  return b.store();
}
inline CompressedAnimation parse(const std::vector<uint8_t>& bytes, SectionSizes* sizes = nullptr) {
  return parse(bytes.data(), bytes.size(), sizes);
}

}  // namespace dmc
