// dmc/metrics.hpp — the rate / distortion entry points of the reference
// include/dmc/metrics.hpp:25-71 that the parity harness uses: RateReport,
// rate_paper_formula (src/metrics.cpp:31-44), rate_exact (:46-65) and
// frame_rms (:67-79).  rate_exact frames the stream through libdmcg's
// serializer, so its byte accounting is the DMC1 format's.
#pragma once

#include <cmath>
#include <vector>

#include "stream.hpp"

namespace dmc {

enum class RateMode { PaperFormula, ExactBits };

struct RateReport {
  double q = 0.0;
  double q_a = 0.0;
  double q_d = 0.0;
  double auxiliary = 0.0;
  double q_s = 0.0;
  RateMode mode = RateMode::ExactBits;
};

inline RateReport rate_paper_formula(double n, double k, double n_b, double k_f, double n_c,
                                     double bits, double bits_a, double bits_d) {
  if (n <= 0 || k <= 0 || n_b <= 0 || k_f <= 0) throw ConfigError("rate formula needs positive dimensions");
  RateReport r;
  r.mode = RateMode::PaperFormula;
  r.q = bits * n * k / (n * k);
  r.q_a = bits_a * n_c * k / (n * k);
  r.q_d = bits_d * n_b * n_b * k_f * k_f / (n * k);
  r.auxiliary = 0.0;
  r.q_s = r.q + r.q_a + r.q_d;
  return r;
}

inline RateReport rate_exact(const SectionSizes& sizes, uint32_t n, uint32_t k) {
  dmcg_sections s{sizes.header,        sizes.connectivity,  sizes.dict_payload, sizes.dict_ranges,
                  sizes.coeff_headers, sizes.coeff_payload, sizes.means,        sizes.anchor_indices,
                  sizes.anchor_ranges, sizes.anchor_payload};
  double v[5];
  dmcg_rate_exact(&s, n, k, v);
  RateReport r;
  r.mode = RateMode::ExactBits;
  r.q = v[0];
  r.q_a = v[1];
  r.q_d = v[2];
  r.auxiliary = v[3];
  r.q_s = v[4];
  return r;
}

inline RateReport rate_exact(const CompressedAnimation& c) {
  SectionSizes sizes;
  serialize(c, &sizes);
  return rate_exact(sizes, c.n, c.k);
}

// Per-frame root-mean-square vertex distance (metrics.cpp:67-79).
inline std::vector<double> frame_rms(const MeshSequence& orig, const MeshSequence& recon) {
  if (orig.n() != recon.n() || orig.k() != recon.k())
    throw DimensionMismatch("sequences differ in vertex or frame count");
  std::vector<double> out((size_t)orig.k());
  for (int f = 0; f < orig.k(); ++f) {
    double sum = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int i = 0; i < orig.n(); ++i) {
        const double d = orig.axis(a)(f, i) - recon.axis(a)(f, i);
        sum += d * d;
      }
    out[(size_t)f] = std::sqrt(sum / orig.n());
  }
  return out;
}

}  // namespace dmc
