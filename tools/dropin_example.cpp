// Minimal caller of the C++ drop-in (include/dmc/codec.hpp): the same calls
// a reference user makes (dmc::encode / dmc::decode), on a rotating
// icosahedron.  Prints "rms <value>" and exits 0 on success.
#include <cmath>
#include <cstdio>

#include "dmc/codec.hpp"

int main() {
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  const double v[12][3] = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                           {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  std::vector<dmc::Face> faces = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},  {0, 7, 10}, {0, 10, 11},
                                  {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                  {3, 9, 4},  {3, 4, 2},  {3, 2, 6},  {3, 6, 8},  {3, 8, 9},
                                  {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},  {9, 8, 1}};
  const int F = 8, n = 12;
  std::array<dmc::Matrix, 3> axes{dmc::Matrix(F, n), dmc::Matrix(F, n), dmc::Matrix(F, n)};
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < n; ++i) {
      const double c = std::cos(0.1 * f), s = std::sin(0.1 * f);
      axes[0](f, i) = c * v[i][0] - s * v[i][1];
      axes[1](f, i) = s * v[i][0] + c * v[i][1];
      axes[2](f, i) = v[i][2] * (1.0 + 0.05 * f);
    }
  dmc::MeshSequence seq(faces, axes);
  dmc::EncoderConfig cfg;
  cfg.k_l = 8;
  try {
    dmc::CompressedAnimation c = dmc::encode(seq, cfg);
    dmc::MeshSequence out = dmc::decode(c);
    double err = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int f = 0; f < F; ++f)
        for (int i = 0; i < n; ++i) {
          const double d = out.axis(a)(f, i) - seq.axis(a)(f, i);
          err += d * d;
        }
    std::printf("rms %.3e\n", std::sqrt(err / (3.0 * n * F)));
    // blocks variant: 3 blocks of k_f = 3 frames (one padded frame)
    dmc::EncoderConfig bc;
    bc.variant = dmc::Variant::Blocks;
    bc.n_b = 3;
    bc.k_l = 3;
    bc.diff_bits = 16;
    dmc::CompressedAnimation cb = dmc::encode(seq, bc);
    dmc::MeshSequence ob = dmc::decode(cb);
    double eb = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int f = 0; f < F; ++f)
        for (int i = 0; i < n; ++i) {
          const double d = ob.axis(a)(f, i) - seq.axis(a)(f, i);
          eb += d * d;
        }
    std::printf("blocks %u %u %zu rms %.3e\n", (unsigned)cb.n_b, (unsigned)cb.pad,
                cb.dict_diffs[0].size(), std::sqrt(eb / (3.0 * n * F)));
    dmc::EncoderConfig bad = cfg;
    bad.k_l = F + 1;
    try {
      dmc::encode(seq, bad);
      return 2;
    } catch (const dmc::Error& e) {
      std::printf("error %d %s\n", e.code(), e.kind().c_str());
    }
  } catch (const dmc::Error& e) {
    std::printf("failed %d %s\n", e.code(), e.what());
    return 1;
  }
  return 0;
}
