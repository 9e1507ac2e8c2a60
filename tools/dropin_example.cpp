// A reference-style caller of the C++ drop-in (include/dmc/codec.hpp): it
// uses only names and members of the reference API (include/dmc/mesh.hpp,
// stream.hpp, codec.hpp, metrics.hpp, errors.hpp) on a rotating icosahedron,
// so it is the compile test of source compatibility as well as a GPU run.
// Prints one line per check; exits 0 on success.
#include <cmath>
#include <cstdio>

#include "dmc/codec.hpp"

static double rms_of(const dmc::MeshSequence& a, const dmc::MeshSequence& b) {
  const std::vector<double> r = dmc::frame_rms(a, b);
  double s = 0.0;
  for (double v : r) s += v * v;
  return std::sqrt(s / r.size());
}

int main(int argc, char** argv) {
  const bool compile_only = argc > 1;
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  const double v[12][3] = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                           {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  std::vector<dmc::Face> faces = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},  {0, 7, 10}, {0, 10, 11},
                                  {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                  {3, 9, 4},  {3, 4, 2},  {3, 2, 6},  {3, 6, 8},  {3, 8, 9},
                                  {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},  {9, 8, 1}};
  const int F = 8, n = 12;
  std::vector<dmc::Matrix> frames;
  for (int f = 0; f < F; ++f) {
    dmc::Matrix fr(n, 3);
    const double c = std::cos(0.1 * f), s = std::sin(0.1 * f);
    for (int i = 0; i < n; ++i) {
      fr(i, 0) = c * v[i][0] - s * v[i][1];
      fr(i, 1) = s * v[i][0] + c * v[i][1];
      fr(i, 2) = v[i][2] * (1.0 + 0.05 * f);
    }
    frames.push_back(fr);
  }
  dmc::MeshSequence seq = dmc::MeshSequence::from_frames(faces, frames);
  // host-side entry points of mesh.hpp (no GPU needed)
  const dmc::Connectivity conn = dmc::build_connectivity(seq.faces(), seq.n());
  std::printf("mesh n=%d k=%d degree0=%d connected=%d valid=%d x00=%.3f\n", seq.n(), seq.k(),
              conn.degree(0), (int)dmc::is_connected(conn), (int)dmc::validate_sequence(seq).ok(),
              seq.axis(dmc::Axis::X)(0, 0));
  try {
    dmc::build_connectivity({{0, 1, 1}}, 3);
    return 3;
  } catch (const dmc::DegenerateFace& e) {
    std::printf("host error %d %s\n", e.code(), e.kind().c_str());
  }
  if (compile_only) return 0;

  dmc::EncoderConfig cfg;  // reference defaults: pca_qp, 1% Stride anchors, 16-bit
  cfg.k_l = 8;
  try {
    dmc::CompressedAnimation c = dmc::encode(seq, cfg);
    // reference member layout (stream.hpp:130-155)
    const dmc::QuantRow& r0 = c.axes[0].coeffs[0].rows[0];
    std::printf("stream v%u %s n=%u k=%u k_l=%u n_c=%u dict=%zu rows=%zu q0=%zu anchors=%zu a0=[%g,%g]\n",
                (unsigned)c.version, dmc::variant_name(c.variant), c.n, c.k, c.k_l, c.n_c,
                c.axes[0].dict_first.size(), c.axes[0].coeffs[0].rows.size(), r0.q.size(),
                c.anchor_indices.size(), c.anchors[0].min, c.anchors[0].max);
    dmc::SectionSizes sizes;
    std::vector<uint8_t> bytes = dmc::serialize(c, &sizes);
    dmc::CompressedAnimation back = dmc::parse(bytes);
    const dmc::RateReport rate = dmc::rate_exact(c);
    std::printf("bytes %zu total %zu parse_equal %d q_s %.6f check %.6f\n", bytes.size(), sizes.total(),
                (int)(back == c), rate.q_s, 8.0 * bytes.size() / (double)(c.n * c.k));
    dmc::MeshSequence out = dmc::decode(back);
    std::printf("rms %.3e\n", rms_of(seq, out));
    // blocks variant: 3 blocks of k_f = 3 frames (one padded frame)
    dmc::EncoderConfig bc;
    bc.variant = dmc::Variant::Blocks;
    bc.n_b = 3;
    bc.k_l = 3;
    bc.diff_bits = 16;
    dmc::CompressedAnimation cb = dmc::encode(seq, bc);
    dmc::MeshSequence ob = dmc::decode(cb);
    std::printf("blocks %u %u %zu rms %.3e\n", (unsigned)cb.n_b, (unsigned)cb.pad,
                cb.axes[0].dict_diffs.size(), rms_of(seq, ob));
    dmc::EncoderConfig bad = cfg;
    bad.k_l = F + 1;
    try {
      dmc::encode(seq, bad);
      return 2;
    } catch (const dmc::ConfigError& e) {
      std::printf("error %d %s\n", e.code(), e.kind().c_str());
    }
    dmc::CompressedAnimation corrupt = c;
    corrupt.axes[1].dict_first[0] = 1u << 16;  // level beyond dict_bits
    try {
      dmc::decode(corrupt);
      return 4;
    } catch (const dmc::CorruptPayload& e) {
      std::printf("corrupt %d %s\n", e.code(), e.kind().c_str());
    }
  } catch (const dmc::Error& e) {
    std::printf("failed %d %s\n", e.code(), e.what());
    return 1;
  }
  return 0;
}
