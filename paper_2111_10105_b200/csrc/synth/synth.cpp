// Seeded synthetic mesh sequences for the five BASELINE.json configs.
//
// The paper's datasets (Handstand, Samba, ...) are third-party and absent;
// BASELINE.json names synthetic stand-ins and these generators build them
// (choices for the under-specified parts are recorded in DESIGN.md §2).
// Host-only C++; the RNG is SplitMix64 with Box-Muller normals so inputs are
// reproducible across machines (std::*_distribution is implementation
// defined, which is why the reference's own src/synth.cpp is not reused).
//
// Output layout = the reference MeshSequence axis layout (include/dmc/mesh.hpp:
// 33-35,56): per axis a k x n column-major matrix, i.e. n vertex rows of F
// contiguous frames, x[i*F + f].
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

#include "../../../include/dmcg_synth.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }  // [0,1)
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  int uniform_int(int lo, int hi) { return lo + (int)(next() % (uint64_t)(hi - lo + 1)); }
  double normal() {
    const double u1 = ((double)(next() >> 11) + 1.0) * 0x1.0p-53;  // (0,1]
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
  }
  void unit3(double v[3]) {
    double n2;
    do {
      v[0] = normal();
      v[1] = normal();
      v[2] = normal();
      n2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    } while (n2 < 1e-12);
    const double inv = 1.0 / std::sqrt(n2);
    v[0] *= inv;
    v[1] *= inv;
    v[2] *= inv;
  }
};

struct Mesh {
  std::vector<double> v;  // 3 per vertex
  std::vector<uint32_t> f;
  uint32_t n() const { return (uint32_t)(v.size() / 3); }
};

// Icosahedron subdivided `level` times; vertex numbering is subdivision order
// (spatially coherent: new edge midpoints follow the faces that create them).
Mesh icosphere(int level) {
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  Mesh m;
  const double base[12][3] = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0},
                              {0, -1, t}, {0, 1, t}, {0, -1, -t}, {0, 1, -t},
                              {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  for (auto& p : base) {
    const double r = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    m.v.insert(m.v.end(), {p[0] / r, p[1] / r, p[2] / r});
  }
  m.f = {0, 11, 5, 0, 5,  1,  0,  1, 7, 0, 7, 10, 0, 10, 11, 1, 5, 9, 5, 11,
         4, 11, 10, 2, 10, 7,  6, 7, 1, 8, 3, 9,  4, 3,  4,  2, 3, 2, 6, 3,
         6, 8,  3,  8, 9,  4,  9, 5, 2, 4, 11, 6, 2, 10, 8,  6, 7, 9, 8, 1};
  for (int l = 0; l < level; ++l) {
    std::map<std::pair<uint32_t, uint32_t>, uint32_t> mid;
    auto midpoint = [&](uint32_t a, uint32_t b) {
      auto key = std::make_pair(std::min(a, b), std::max(a, b));
      auto it = mid.find(key);
      if (it != mid.end()) return it->second;
      double p[3];
      for (int c = 0; c < 3; ++c) p[c] = 0.5 * (m.v[3 * a + c] + m.v[3 * b + c]);
      const double r = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
      const uint32_t idx = m.n();
      m.v.insert(m.v.end(), {p[0] / r, p[1] / r, p[2] / r});
      mid.emplace(key, idx);
      return idx;
    };
    std::vector<uint32_t> nf;
    nf.reserve(m.f.size() * 4);
    for (size_t i = 0; i < m.f.size(); i += 3) {
      const uint32_t a = m.f[i], b = m.f[i + 1], c = m.f[i + 2];
      const uint32_t ab = midpoint(a, b), bc = midpoint(b, c), ca = midpoint(c, a);
      nf.insert(nf.end(), {a, ab, ca, b, bc, ab, c, ca, bc, ab, bc, ca});
    }
    m.f.swap(nf);
  }
  return m;
}

// Real orthonormal spherical harmonics Y_lm, l <= lmax, m = -l..l, evaluated
// at unit vector p; out has (lmax+1)^2 entries indexed l*l + l + m.
void real_sh(int lmax, const double p[3], double* out) {
  const double ct = std::max(-1.0, std::min(1.0, p[2]));
  const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
  const double phi = std::atan2(p[1], p[0]);
  // associated Legendre P_l^m(ct) without Condon-Shortley phase
  std::vector<double> P((lmax + 1) * (lmax + 1), 0.0);
  auto at = [&](int l, int m) -> double& { return P[l * (lmax + 1) + m]; };
  at(0, 0) = 1.0;
  for (int m = 1; m <= lmax; ++m) at(m, m) = at(m - 1, m - 1) * (2 * m - 1) * st;
  for (int m = 0; m < lmax; ++m) at(m + 1, m) = (2 * m + 1) * ct * at(m, m);
  for (int m = 0; m <= lmax; ++m)
    for (int l = m + 2; l <= lmax; ++l)
      at(l, m) = ((2 * l - 1) * ct * at(l - 1, m) - (l + m - 1) * at(l - 2, m)) / (l - m);
  for (int l = 0; l <= lmax; ++l) {
    for (int m = 0; m <= l; ++m) {
      double fact = 1.0;  // (l-m)!/(l+m)!
      for (int q = l - m + 1; q <= l + m; ++q) fact /= q;
      const double K = std::sqrt((2 * l + 1) / (4 * kPi) * fact);
      if (m == 0) {
        out[l * l + l] = K * at(l, 0);
      } else {
        out[l * l + l + m] = std::sqrt(2.0) * K * at(l, m) * std::cos(m * phi);
        out[l * l + l - m] = std::sqrt(2.0) * K * at(l, m) * std::sin(m * phi);
      }
    }
  }
}

void rotate(const double axis[3], double ang, const double p[3], double o[3]) {
  const double c = std::cos(ang), s = std::sin(ang);
  const double d = axis[0] * p[0] + axis[1] * p[1] + axis[2] * p[2];
  const double cx = axis[1] * p[2] - axis[2] * p[1];
  const double cy = axis[2] * p[0] - axis[0] * p[2];
  const double cz = axis[0] * p[1] - axis[1] * p[0];
  o[0] = p[0] * c + cx * s + axis[0] * d * (1 - c);
  o[1] = p[1] * c + cy * s + axis[1] * d * (1 - c);
  o[2] = p[2] * c + cz * s + axis[2] * d * (1 - c);
}

template <typename T>
void store(T* const axes[3], uint32_t n, uint32_t F, uint32_t i, uint32_t f, const double p[3]) {
  for (int a = 0; a < 3; ++a) axes[a][(size_t)i * F + f] = (T)p[a];
}

// Configs 0, 2, 4: rigid rotation 0.05*t rad about a seeded unit axis of the
// radially displaced sphere; optional 4-bone piecewise-linear bend (config 2).
template <typename T>
void sphere_sequence(const Mesh& m, uint32_t F, int lmax, int bones, uint64_t seed,
                     T* const axes[3]) {
  Rng rng(seed);
  double axis[3];
  rng.unit3(axis);
  const int nh = (lmax + 1) * (lmax + 1);
  std::vector<double> a(nh), fr(nh), ph(nh);
  for (int h = 0; h < nh; ++h) {
    a[h] = 0.05 * rng.normal();  // a_lm ~ N(0, 0.05) read as std 0.05
    fr[h] = rng.uniform_int(1, 4);
    ph[h] = rng.uniform(0.0, 2.0 * kPi);
  }
  struct Bone {
    double dir[3], axis[3], key[5], sigma;
  };
  std::vector<Bone> bs(bones);
  for (auto& b : bs) {
    rng.unit3(b.dir);
    rng.unit3(b.axis);
    for (double& k : b.key) k = rng.uniform(-0.4, 0.4);
    b.sigma = rng.uniform(0.4, 0.8);
  }
  const uint32_t n = m.n();
  std::vector<double> tf((size_t)nh * F);
  for (int h = 0; h < nh; ++h)
    for (uint32_t t = 0; t < F; ++t)
      tf[(size_t)h * F + t] = std::sin(2.0 * kPi * fr[h] * t / F + ph[h]);
#pragma omp parallel
  {
    std::vector<double> Y(nh), w(bones);
#pragma omp for schedule(static)
    for (uint32_t i = 0; i < n; ++i) {
      const double* v = &m.v[3 * i];
      real_sh(lmax, v, Y.data());
      for (int b = 0; b < bones; ++b) {
        const Bone& B = bs[b];
        const double c = std::max(-1.0, std::min(1.0, v[0] * B.dir[0] + v[1] * B.dir[1] +
                                                          v[2] * B.dir[2]));
        const double g = std::acos(c) / B.sigma;  // geodesic distance / falloff
        w[b] = std::exp(-g * g);
      }
      for (uint32_t t = 0; t < F; ++t) {
        double d = 0.0;
        for (int h = 0; h < nh; ++h) d += a[h] * Y[h] * tf[(size_t)h * F + t];
        double p[3] = {v[0] * (1.0 + d), v[1] * (1.0 + d), v[2] * (1.0 + d)};
        for (int b = 0; b < bones; ++b) {
          const Bone& B = bs[b];
          // piecewise-linear bend angle over 4 equal time segments
          const double x = 4.0 * t / (F > 1 ? F - 1 : 1);
          const int sgi = std::min(3, (int)x);
          const double fr2 = x - sgi;
          const double ang = B.key[sgi] * (1 - fr2) + B.key[sgi + 1] * fr2;
          const double j[3] = {0.5 * B.dir[0], 0.5 * B.dir[1], 0.5 * B.dir[2]};
          double q[3] = {p[0] - j[0], p[1] - j[1], p[2] - j[2]}, r[3];
          rotate(B.axis, ang, q, r);
          for (int c = 0; c < 3; ++c) p[c] += w[b] * (r[c] + j[c] - p[c]);
        }
        double o[3];
        rotate(axis, 0.05 * t, p, o);
        store(axes, n, F, i, t, o);
      }
    }
  }
}

}  // namespace

extern "C" {

int dmcg_synth_icosphere_size(int level, uint32_t* n, uint32_t* n_faces) {
  if (level < 0 || level > 9) return 5;
  *n = 10u * (1u << (2 * level)) + 2u;
  *n_faces = 20u * (1u << (2 * level));
  return 0;
}

int dmcg_synth_sphere(int level, uint32_t F, int lmax, int bones, uint64_t seed, int f32,
                      uint32_t* faces, void* const axes[3]) {
  if (level < 0 || level > 9 || F < 1 || lmax < 0 || lmax > 16 || bones < 0) return 5;
  const Mesh m = icosphere(level);
  std::memcpy(faces, m.f.data(), m.f.size() * sizeof(uint32_t));
  if (f32) {
    float* const ax[3] = {(float*)axes[0], (float*)axes[1], (float*)axes[2]};
    sphere_sequence<float>(m, F, lmax, bones, seed, ax);
  } else {
    double* const ax[3] = {(double*)axes[0], (double*)axes[1], (double*)axes[2]};
    sphere_sequence<double>(m, F, lmax, bones, seed, ax);
  }
  return 0;
}

// Config 1: torus nu x nv (R, r); `waves` travelling sine waves along the
// major angle displace vertices along the tube normal, amplitude U[0.01,0.05],
// wavenumber U{1..6}, temporal speed U{1..4} cycles per sequence, phase
// U[0,2pi); plus i.i.d. Gaussian jitter (std `jitter`) per coordinate/frame.
int dmcg_synth_torus(uint32_t nu, uint32_t nv, double R, double r, uint32_t F, int waves,
                     double jitter, uint64_t seed, int f32, uint32_t* faces,
                     void* const axes[3]) {
  if (nu < 3 || nv < 3 || F < 1) return 5;
  Rng rng(seed);
  std::vector<double> amp(waves), kw(waves), sp(waves), ph(waves);
  for (int w = 0; w < waves; ++w) {
    amp[w] = rng.uniform(0.01, 0.05);
    kw[w] = rng.uniform_int(1, 6);
    sp[w] = rng.uniform_int(1, 4);
    ph[w] = rng.uniform(0.0, 2.0 * kPi);
  }
  const uint32_t n = nu * nv;
  size_t fi = 0;
  for (uint32_t i = 0; i < nu; ++i)
    for (uint32_t j = 0; j < nv; ++j) {
      const uint32_t a = i * nv + j, b = ((i + 1) % nu) * nv + j;
      const uint32_t c = i * nv + (j + 1) % nv, d = ((i + 1) % nu) * nv + (j + 1) % nv;
      const uint32_t tri[6] = {a, b, c, b, d, c};
      std::memcpy(faces + fi, tri, sizeof(tri));
      fi += 6;
    }
  // jitter drawn in a fixed (vertex, frame, axis) order from a second stream
  Rng jr(seed ^ 0x5DEECE66Dull);
  for (uint32_t i = 0; i < nu; ++i)
    for (uint32_t j = 0; j < nv; ++j) {
      const double u = 2.0 * kPi * i / nu, v = 2.0 * kPi * j / nv;
      const double nrm[3] = {std::cos(u) * std::cos(v), std::sin(u) * std::cos(v), std::sin(v)};
      const double base[3] = {(R + r * std::cos(v)) * std::cos(u),
                              (R + r * std::cos(v)) * std::sin(u), r * std::sin(v)};
      const uint32_t idx = i * nv + j;
      for (uint32_t t = 0; t < F; ++t) {
        double d = 0.0;
        for (int w = 0; w < waves; ++w)
          d += amp[w] * std::sin(kw[w] * u - 2.0 * kPi * sp[w] * t / F + ph[w]);
        double p[3];
        for (int c = 0; c < 3; ++c) p[c] = base[c] + d * nrm[c] + jitter * jr.normal();
        if (f32)
          store((float* const*)axes, n, F, idx, t, p);
        else
          store((double* const*)axes, n, F, idx, t, p);
      }
    }
  return 0;
}

// Config 3: nx x ny grid on [0,1]^2 (spacing h), in-plane jitter U[-0.2,0.2]*h,
// two triangles per cell; z = sum of `bumps` Gaussian bumps, amplitude
// U[0.05,0.2], width U[0.03,0.1], centre moving linearly from U[0,1]^2 with
// total displacement U[-0.5,0.5]^2 over the sequence.  x, y are static.
int dmcg_synth_grid(uint32_t nx, uint32_t ny, uint32_t F, int bumps, uint64_t seed, int f32,
                    uint32_t* faces, void* const axes[3]) {
  if (nx < 2 || ny < 2 || F < 1) return 5;
  Rng rng(seed);
  const double h = 1.0 / (double)(nx - 1);
  const uint32_t n = nx * ny;
  std::vector<double> xy(2 * (size_t)n);
  for (uint32_t j = 0; j < ny; ++j)
    for (uint32_t i = 0; i < nx; ++i) {
      const uint32_t v = j * nx + i;
      xy[2 * v] = i * h + rng.uniform(-0.2, 0.2) * h;
      xy[2 * v + 1] = j * h + rng.uniform(-0.2, 0.2) * h;
    }
  size_t fi = 0;
  for (uint32_t j = 0; j + 1 < ny; ++j)
    for (uint32_t i = 0; i + 1 < nx; ++i) {
      const uint32_t a = j * nx + i, b = a + 1, c = a + nx, d = c + 1;
      const uint32_t tri[6] = {a, b, c, b, d, c};
      std::memcpy(faces + fi, tri, sizeof(tri));
      fi += 6;
    }
  std::vector<double> A(bumps), S(bumps), cx(bumps), cy(bumps), vx(bumps), vy(bumps);
  for (int b = 0; b < bumps; ++b) {
    A[b] = rng.uniform(0.05, 0.2);
    S[b] = rng.uniform(0.03, 0.1);
    cx[b] = rng.uniform();
    cy[b] = rng.uniform();
    vx[b] = rng.uniform(-0.5, 0.5);
    vy[b] = rng.uniform(-0.5, 0.5);
  }
#pragma omp parallel for schedule(static)
  for (uint32_t v = 0; v < n; ++v) {
    for (uint32_t t = 0; t < F; ++t) {
      const double s = (double)t / F;
      double z = 0.0;
      for (int b = 0; b < bumps; ++b) {
        const double dx = xy[2 * v] - (cx[b] + vx[b] * s);
        const double dy = xy[2 * v + 1] - (cy[b] + vy[b] * s);
        const double q = (dx * dx + dy * dy) / (2.0 * S[b] * S[b]);
        if (q < 40.0) z += A[b] * std::exp(-q);
      }
      const double p[3] = {xy[2 * v], xy[2 * v + 1], z};
      if (f32)
        store((float* const*)axes, n, F, v, t, p);
      else
        store((double* const*)axes, n, F, v, t, p);
    }
  }
  return 0;
}

}  // extern "C"
