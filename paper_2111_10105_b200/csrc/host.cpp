// Host side of libdmcg: the C ABI (include/dmcg.h), mesh preprocessing,
// configuration checks, plan lifetime and the DMC1 stream.  Reference
// behaviour is cited per function (paths relative to /root/reference/proj).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <limits>
#include <malloc.h>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"
#include "ozaki.h"
#include "kernels.h"
#include "par.h"

namespace dmcg {

constexpr uint32_t kColBlock = 4;  // CG column-block width, = kCB in common.cuh

Status plan_encode(dmcg_plan* p, const void* const x[3],
                   const std::function<void()>* between = nullptr);
Status plan_decode(dmcg_plan* p, const dmcg_decode_options* opt, void* const out[3]);

#define CUDA_OK(expr)                                                                      \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return Status{DMCG_E_CUDA, std::string("CudaError: ") + cudaGetErrorString(_e)};     \
  } while (0)

static double wall_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
PhaseTimer::PhaseTimer(const char* s) : scope(s), on(std::getenv("DMCG_TIMING") != nullptr) {
  t0 = wall_ms();
}
void PhaseTimer::lap(const char* what) {
  if (!on) return;
  const double t = wall_ms();
  std::fprintf(stderr, "  %s %-16s %.2f ms\n", scope, what, t - t0);
  t0 = t;
}

// ---- device pool -----------------------------------------------------------
void* DevicePool::get(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  auto it = free_.find(bytes);
  if (it != free_.end()) {
    void* p = it->second;
    free_.erase(it);
    return p;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    // trim the cache and retry once
    release_all();
    cudaGetLastError();
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  }
  return p;
}
void DevicePool::put(void* p, size_t bytes) {
  if (!p) return;
  bytes = (bytes + 255) & ~size_t(255);
  free_.emplace(bytes, p);
}
void DevicePool::release_all() {
  for (auto& kv : free_) cudaFree(kv.second);
  free_.clear();
}

// ---- mesh --------------------------------------------------------------------
// build_connectivity (src/mesh.cpp:60-86) with the errors of mesh.cpp:66-75.
Status build_mesh(const uint32_t* faces, uint32_t n_faces, uint32_t n, MeshHost* out) {
  if (n_faces == 0) return {DMCG_E_INDEX, "ValidationError: face list is empty"};
  for (uint32_t t = 0; t < n_faces; ++t) {
    const uint32_t* f = faces + 3 * (size_t)t;
    for (int j = 0; j < 3; ++j)
      if (f[j] >= n)
        return {DMCG_E_INDEX, "IndexOutOfRange: face " + std::to_string(t) + " refers to vertex " +
                                  std::to_string(f[j]) + " >= " + std::to_string(n)};
    if (f[0] == f[1] || f[1] == f[2] || f[0] == f[2])
      return {DMCG_E_INDEX, "DegenerateFace: face " + std::to_string(t) + " repeats a vertex index"};
  }
  out->n = n;
  std::vector<uint32_t> cnt((size_t)n + 1, 0);
  for (size_t t = 0; t < 3 * (size_t)n_faces; ++t) cnt[faces[t] + 1] += 2;
  for (uint32_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<uint32_t> col(cnt[n]);
  std::vector<uint32_t> fill(cnt.begin(), cnt.end() - 1);
  for (uint32_t t = 0; t < n_faces; ++t) {
    const uint32_t* f = faces + 3 * (size_t)t;
    for (int j = 0; j < 3; ++j) {
      col[fill[f[j]]++] = f[(j + 1) % 3];
      col[fill[f[j]]++] = f[(j + 2) % 3];
    }
  }
  // per vertex: sort + deduplicate its neighbour list in place (parallel),
  // then the CSR of the one-ring and of the Laplacian (diagonal in sorted
  // position) by prefix sums
  std::vector<uint32_t> deg(n, 0);
  parallel_for(n, 1024, [&](uint32_t v0, uint32_t v1, uint32_t) {
    for (uint32_t i = v0; i < v1; ++i) {
      auto b = col.begin() + cnt[i], e = col.begin() + cnt[i + 1];
      std::sort(b, e);
      deg[i] = (uint32_t)(std::unique(b, e) - b);
    }
  });
  out->adj_rp.assign((size_t)n + 1, 0);
  out->lap_rp.assign((size_t)n + 1, 0);
  for (uint32_t i = 0; i < n; ++i) {
    out->adj_rp[i + 1] = out->adj_rp[i] + deg[i];
    out->lap_rp[i + 1] = out->lap_rp[i] + deg[i] + 1;
  }
  out->adj_ci.resize(out->adj_rp[n]);
  out->lap_ci.resize(out->lap_rp[n]);
  parallel_for(n, 1024, [&](uint32_t v0, uint32_t v1, uint32_t) {
    for (uint32_t i = v0; i < v1; ++i) {
      const uint32_t* src = col.data() + cnt[i];
      std::copy(src, src + deg[i], out->adj_ci.begin() + out->adj_rp[i]);
      // Laplacian structure (laplacian.cpp:21-37): diagonal in sorted position
      uint32_t o = out->lap_rp[i];
      bool placed = false;
      for (uint32_t t = 0; t < deg[i]; ++t) {
        if (!placed && src[t] > i) {
          out->lap_ci[o++] = i;
          placed = true;
        }
        out->lap_ci[o++] = src[t];
      }
      if (!placed) out->lap_ci[o++] = i;
    }
  });
  return Status::ok();
}

// validate_sequence's graph checks (src/mesh.cpp:108-136): isolated vertex,
// connectivity by BFS (mesh.cpp:88-106).
Status validate_mesh(const MeshHost& m) {
  std::string issues;
  for (uint32_t i = 0; i < m.n; ++i)
    if (m.adj_rp[i] == m.adj_rp[i + 1]) {
      issues = "vertex " + std::to_string(i) + " is isolated";
      break;
    }
  std::vector<char> seen(m.n, 0);
  std::deque<uint32_t> queue{0};
  seen[0] = 1;
  uint32_t visited = 1;
  while (!queue.empty()) {
    const uint32_t v = queue.front();
    queue.pop_front();
    for (uint32_t p = m.adj_rp[v]; p < m.adj_rp[v + 1]; ++p) {
      const uint32_t w = m.adj_ci[p];
      if (!seen[w]) {
        seen[w] = 1;
        ++visited;
        queue.push_back(w);
      }
    }
  }
  if (visited != m.n) issues += std::string(issues.empty() ? "" : "; ") + "graph not connected";
  if (!issues.empty()) return {DMCG_E_INDEX, "ValidationError: " + issues};
  return Status::ok();
}

// anchored_normal_matrix (src/solver.cpp:25-39): M = L^T L + S^T S.  L is
// symmetric and integer valued, so M's entries are small integers held
// exactly in float.
void build_normal_matrix(MeshHost* m) {
  // Rows of M are independent: each chunk of rows is built into its own
  // arrays by one host thread, then the chunks are concatenated.
  const uint32_t n = m->n;
  const uint32_t grain = 2048;
  const uint32_t nch = parallel_chunks(n, grain);
  std::vector<std::vector<uint32_t>> cci(nch), crl(nch);
  std::vector<std::vector<float>> cval(nch);
  auto lval = [&](uint32_t row, uint32_t p) -> double {
    return m->lap_ci[p] == row ? (double)(m->lap_rp[row + 1] - m->lap_rp[row] - 1) : -1.0;
  };
  parallel_for(n, grain, [&](uint32_t r0, uint32_t r1, uint32_t c) {
    std::unique_ptr<double[]> acc(new double[n]);  // valid where mark[j] == row
    std::vector<int32_t> mark(n, -1);
    std::vector<uint32_t> list, ci, rl;  // thread-local: no shared vector headers
    std::vector<float> va;
    ci.reserve((size_t)(r1 - r0) * 20);
    va.reserve((size_t)(r1 - r0) * 20);
    rl.reserve(r1 - r0);
    for (uint32_t i = r0; i < r1; ++i) {
      list.clear();
      for (uint32_t p = m->lap_rp[i]; p < m->lap_rp[i + 1]; ++p) {
        const uint32_t k = m->lap_ci[p];
        const double a = lval(i, p);  // L^T(i,k) = L(k,i) = L(i,k)
        for (uint32_t q = m->lap_rp[k]; q < m->lap_rp[k + 1]; ++q) {
          const uint32_t j = m->lap_ci[q];
          if (mark[j] != (int32_t)i) {
            mark[j] = (int32_t)i;
            acc[j] = 0.0;
            list.push_back(j);
          }
          acc[j] += a * lval(k, q);
        }
      }
      if (m->anchor_pos[i] >= 0) acc[i] += 1.0;
      std::sort(list.begin(), list.end());
      for (uint32_t j : list) {
        ci.push_back(j);
        va.push_back((float)acc[j]);
      }
      rl.push_back((uint32_t)list.size());
    }
    cci[c] = std::move(ci);
    cval[c] = std::move(va);
    crl[c] = std::move(rl);
  });
  // concatenate: every chunk copies its rows to its offset (parallel)
  std::vector<size_t> off(nch + 1, 0);
  std::vector<uint32_t> row0(nch + 1, 0);
  for (uint32_t c = 0; c < nch; ++c) {
    off[c + 1] = off[c] + cci[c].size();
    row0[c + 1] = row0[c] + (uint32_t)crl[c].size();
  }
  m->m_rp.resize((size_t)n + 1);
  m->m_ci.resize(off[nch]);
  m->m_val.resize(off[nch]);
  m->m_rp[0] = 0;
  parallel_for(nch, 1, [&](uint32_t c0, uint32_t c1, uint32_t) {
    for (uint32_t c = c0; c < c1; ++c) {
      std::copy(cci[c].begin(), cci[c].end(), m->m_ci.begin() + off[c]);
      std::copy(cval[c].begin(), cval[c].end(), m->m_val.begin() + off[c]);
      uint32_t at = (uint32_t)off[c], row = row0[c];
      for (uint32_t len : crl[c]) {
        at += len;
        m->m_rp[++row] = at;
      }
    }
  });
}

void build_reduced_normal(MeshHost* m) {
  build_normal_matrix(m);  // L^T L: no anchors on the anchor-free variants
  const uint32_t n = m->n;
  std::vector<uint32_t> rp(n, 0), ci;
  std::vector<float> va;
  ci.reserve(m->m_ci.size());
  va.reserve(m->m_ci.size());
  for (uint32_t i = 1; i < n; ++i) {
    for (uint32_t p = m->m_rp[i]; p < m->m_rp[i + 1]; ++p)
      if (m->m_ci[p] > 0) {
        ci.push_back(m->m_ci[p] - 1);
        va.push_back(m->m_val[p]);
      }
    rp[i] = (uint32_t)ci.size();
  }
  m->m_rp = std::move(rp);
  m->m_ci = std::move(ci);
  m->m_val = std::move(va);
}

uint64_t hash_faces(const uint32_t* faces, uint32_t n_faces) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a over the index words
  for (size_t t = 0; t < 3 * (size_t)n_faces; ++t) {
    h ^= faces[t];
    h *= 1099511628211ull;
  }
  return h;
}

// ---- anchors (src/codec.cpp:199-242) ----------------------------------------
namespace {
struct Mt64 {  // MT19937-64, the engine std::mt19937_64 specifies
  uint64_t mt[312];
  int mti = 313;
  explicit Mt64(uint64_t seed) {
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    mti = 312;
  }
  uint64_t next() {
    static const uint64_t mag01[2] = {0ull, 0xB5026F5AA96619E9ull};
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    if (mti >= 312) {
      int i;
      uint64_t x;
      for (i = 0; i < 156; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + 156] ^ (x >> 1) ^ mag01[x & 1ull];
      }
      for (; i < 311; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i - 156] ^ (x >> 1) ^ mag01[x & 1ull];
      }
      x = (mt[311] & UM) | (mt[0] & LM);
      mt[311] = mt[155] ^ (x >> 1) ^ mag01[x & 1ull];
      mti = 0;
    }
    uint64_t x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
  }
};

uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

Status check_config(const dmcg_config& cfg, uint32_t n, uint32_t k, std::vector<int>* row_bits) {
  // src/codec.cpp:69-120, in the reference's order.
  if (cfg.n_b < 1) return {DMCG_E_CONFIG, "ConfigError: block count must be >= 1"};
  if (cfg.variant != DMCG_BLOCKS && cfg.n_b != 1)
    return {DMCG_E_CONFIG, "ConfigError: block count > 1 requires the blocks variant"};
  if (cfg.n_b > k)
    return {DMCG_E_CONFIG, "BlockSizeError: cannot split " + std::to_string(k) + " frames into " +
                               std::to_string(cfg.n_b) + " blocks"};
  if (cfg.t_max < 1) return {DMCG_E_CONFIG, "ConfigError: t_max must be >= 1"};
  if (!(cfg.anchor_fraction >= 0.0 && cfg.anchor_fraction <= 1.0))
    return {DMCG_E_CONFIG, "ConfigError: anchor fraction outside [0, 1]"};
  for (int bits : {cfg.anchor_bits, cfg.dict_bits, cfg.diff_bits})
    if (bits < 1 || bits > 16)
      return {DMCG_E_CONFIG, "InvalidBits: bit depth " + std::to_string(bits) + " outside 1..16"};
  const uint32_t pad = (cfg.n_b - k % cfg.n_b) % cfg.n_b;
  const uint32_t k_f = (k + pad) / cfg.n_b;
  if (cfg.variant == DMCG_PER_MESH_GFT) {
    if (n > 5000) return {DMCG_E_CONFIG, "ConfigError: per_mesh_gft limited to n <= 5000"};
  } else if (cfg.k_l > k_f) {
    return {DMCG_E_CONFIG, "ConfigError: k_l = " + std::to_string(cfg.k_l) +
                               " exceeds dictionary dimension " + std::to_string(k_f)};
  }
  row_bits->clear();
  if (!cfg.row_bits || cfg.n_row_bits == 0) {
    if (cfg.row_bits && cfg.n_row_bits == 0 && cfg.k_l != 0)
      return {DMCG_E_CONFIG, "ConfigError: row_bits must have one entry per retained row"};
    row_bits->assign(cfg.k_l, 16);
  } else {
    if (cfg.n_row_bits != cfg.k_l)
      return {DMCG_E_CONFIG, "ConfigError: row_bits must have one entry per retained row"};
    row_bits->assign(cfg.row_bits, cfg.row_bits + cfg.k_l);
  }
  for (int bits : *row_bits)
    if (bits < 1 || bits > 16)
      return {DMCG_E_CONFIG,
              "InvalidBits: row bit depth " + std::to_string(bits) + " outside 1..16"};
  // Scope of the B200 path.
  if (cfg.variant < DMCG_PCA || cfg.variant > DMCG_BLOCKS)
    return {DMCG_E_UNSUPPORTED,
            "Unsupported: only the variants pca, pca_q, v2v, pca_qs, pca_qp, blocks are on the "
            "B200 path"};
  if (cfg.raw_payload) return {DMCG_E_UNSUPPORTED, "Unsupported: raw_payload debug mode"};
  if (cfg.laplacian != 0)
    return {DMCG_E_UNSUPPORTED, "Unsupported: only the combinatorial Laplacian"};
  if (cfg.oi_rounds < 0) return {DMCG_E_CONFIG, "ConfigError: oi_rounds must be >= 0"};
  if (k > 512) return {DMCG_E_UNSUPPORTED, "Unsupported: more than 512 frames"};
  return Status::ok();
}
}  // namespace

}  // namespace dmcg

using namespace dmcg;

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int dmcg_abi_version(void) { return DMCG_ABI_VERSION; }

// The decoder's host analysis (mesh CSR, normal matrix, symbolic Cholesky)
// allocates and frees ~200 MB of index arrays per call.  With glibc's default
// thresholds every such array is a fresh mmap whose first touch page-faults
// (from 16 pool threads at once: they serialise on the mm lock); on the B200
// host that is half of the analysis time (115 -> 65 ms for 262 144 vertices,
// tools/analysis_bench.py).  Keep freed blocks on the heap instead: process-
// wide, set once, DMCG_NO_MALLOPT=1 leaves the allocator alone.
static void tune_host_allocator() {
  static std::once_flag once;
  std::call_once(once, [] {
    if (std::getenv("DMCG_NO_MALLOPT")) return;
    mallopt(M_MMAP_THRESHOLD, 32 << 20);  // glibc's upper limit
    mallopt(M_TRIM_THRESHOLD, std::numeric_limits<int>::max());
    mallopt(M_TOP_PAD, 256 << 20);
  });
}

int dmcg_create(dmcg_ctx** out, int device) {
  tune_host_allocator();
  if (!out) return DMCG_E_CONFIG;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return DMCG_E_CUDA;
  }
  if (device < 0 || device >= count) return DMCG_E_CONFIG;
  if (cudaSetDevice(device) != cudaSuccess) return DMCG_E_CUDA;
  auto* c = new dmcg_ctx();
  c->device = device;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->aux2, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in[2], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_q[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_q[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_q[2], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_cp, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return DMCG_E_CUDA;
  }
  *out = c;
  return DMCG_OK;
}

static void drop_pending_decode(dmcg_ctx* ctx);

void dmcg_destroy(dmcg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  c->pending.reset();
  drop_pending_decode(c);
  cudaStreamSynchronize(c->stream);
  c->pool.release_all();
  cudaStreamSynchronize(c->aux);
  cudaStreamSynchronize(c->aux2);
  cudaStreamSynchronize(c->copy);
  for (auto e : c->ev_in)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_q)
    if (e) cudaEventDestroy(e);
  if (c->ev_cp) cudaEventDestroy(c->ev_cp);
  cudaStreamDestroy(c->copy);
  for (auto e : c->ev_timing) cudaEventDestroy(e);
  for (auto e : c->ev_plain) cudaEventDestroy(e);
  cudaStreamDestroy(c->aux2);
  cudaStreamDestroy(c->aux);
  cudaStreamDestroy(c->stream);
  delete c;
}

const char* dmcg_last_error(const dmcg_ctx* c) { return c ? c->err.c_str() : "no context"; }

void dmcg_config_default(dmcg_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->variant = DMCG_PCA_QP;  // include/dmc/codec.hpp:31-48
  cfg->k_l = 20;
  cfg->n_b = 1;
  cfg->t_max = 4;
  cfg->anchor_fraction = 0.01;
  cfg->anchor_bits = 16;
  cfg->dict_bits = 16;
  cfg->diff_bits = 8;
  cfg->anchor_strategy = 0;
  cfg->seed = 0;
  cfg->laplacian = 0;
  cfg->raw_payload = 0;
  cfg->oi_rounds = 0;
  cfg->oi_seed = 0;
  cfg->oi_implicit = 0;
  cfg->oi_tolerance = -1.0;
}

void dmcg_decode_options_default(dmcg_decode_options* o) {
  o->cg_rtol = 1e-10;
  o->cg_max_iter = 20000;
  o->solver = 0;
  o->refine = 1;
  o->reuse_factor = 0;
  o->frame_begin = 0;
  o->frame_count = 0;
}

uint32_t dmcg_anchor_count(uint32_t n, double fraction) {
  const auto rounded = (int64_t)std::llround(fraction * n);
  return (uint32_t)std::clamp<int64_t>(rounded, 1, n);
}

int dmcg_select_anchors(uint32_t n, uint32_t n_c, int strategy, uint64_t seed, uint32_t* out) {
  if (n_c < 1 || n_c > n) return DMCG_E_CONFIG;  // InvalidCount
  std::vector<uint32_t> idx;
  idx.reserve(n_c);
  if (strategy == 0) {
    for (uint64_t j = 0; j < n_c; ++j) idx.push_back((uint32_t)(j * n / n_c));
    std::sort(idx.begin(), idx.end());
    idx.erase(std::unique(idx.begin(), idx.end()), idx.end());
    std::vector<char> used(n, 0);
    for (uint32_t v : idx) used[v] = 1;
    for (uint32_t i = 0; idx.size() < n_c && i < n; ++i)
      if (!used[i]) {
        idx.push_back(i);
        used[i] = 1;
      }
    std::sort(idx.begin(), idx.end());
  } else {
    std::vector<uint32_t> pool(n);
    for (uint32_t i = 0; i < n; ++i) pool[i] = i;
    Mt64 rng(seed);
    for (uint32_t i = n - 1; i > 0; --i) {
      const uint64_t j = rng.next() % ((uint64_t)i + 1);
      std::swap(pool[i], pool[j]);
    }
    idx.assign(pool.begin(), pool.begin() + n_c);
    std::sort(idx.begin(), idx.end());
  }
  std::memcpy(out, idx.data(), idx.size() * sizeof(uint32_t));
  return DMCG_OK;
}

int dmcg_encoded_sizes(uint32_t n, uint32_t F, const dmcg_config* cfg, dmcg_sizes* out) {
  if (!cfg || !out) return DMCG_E_CONFIG;
  out->dict_q = (size_t)F * F;
  out->rows = cfg->k_l;
  out->coeff_q = (size_t)cfg->k_l * n;
  out->anchor_idx =
      variant_uses_anchors(cfg->variant) ? dmcg_anchor_count(n, cfg->anchor_fraction) : 0;
  out->anchor_q = out->anchor_idx * (size_t)F;
  out->means = variant_uses_means(cfg->variant) ? F : 0;
  const uint32_t nb = cfg->n_b ? cfg->n_b : 1;
  out->n_b = (uint16_t)nb;
  out->pad = 0;
  out->dict_ranges = 0;
  if (nb > 1) {  // blocks: padded frames, n_b dictionaries and coefficient blocks
    if (nb > F) return DMCG_E_CONFIG;
    const uint32_t pad = (nb - F % nb) % nb, kf = (F + pad) / nb;
    out->pad = (uint16_t)pad;
    out->dict_q = (size_t)nb * kf * kf;
    out->dict_ranges = nb - 1;
    out->rows = (size_t)nb * cfg->k_l;
    out->coeff_q = out->rows * n;
  }
  return DMCG_OK;
}

// ---- plan ---------------------------------------------------------------------
}  // extern "C"

void* dmcg::plan_alloc(dmcg_plan* p, size_t bytes) {
  if (bytes == 0) bytes = 256;
  void* d = p->ctx->pool.get(bytes);
  if (d) p->owned.emplace_back(d, bytes);
  return d;
}

extern "C" {

static void* plan_get(dmcg_plan* p, size_t bytes) {
  if (bytes == 0) bytes = 256;
  void* d = p->ctx->pool.get(bytes);
  if (d) p->owned.emplace_back(d, bytes);
  return d;
}

void dmcg_plan_destroy(dmcg_plan* p) {
  if (!p) return;
  cudaSetDevice(p->ctx->device);
  cudaStreamSynchronize(p->ctx->stream);
  for (auto* g : {&p->g_encode, &p->g_decode})
    if (g->exec) cudaGraphExecDestroy(g->exec);
  for (auto& kv : p->owned) p->ctx->pool.put(kv.first, kv.second);
  for (auto& e : p->ev) p->ctx->give_event(e, true);
  for (auto e : {p->ev_fork, p->ev_join, p->ev_pf_fork, p->ev_pf_join}) p->ctx->give_event(e, false);
  for (auto e : {p->ev_pf0, p->ev_pf1}) p->ctx->give_event(e, true);
  for (auto e : p->solve_ev) cudaEventDestroy(e);
  delete p;
}

// mesh_given: Laplacian structure of these faces already built (the decoder
// reuses the encoder's, see dmcg_decode); encode_side = false skips the
// encode-only set-up (OI start matrices).
static Status plan_create_impl(dmcg_ctx* ctx, uint32_t n, uint32_t F, int dtype,
                               const uint32_t* faces, uint32_t n_faces, const dmcg_config* cfg,
                               const uint32_t* anchors_given, uint32_t n_c_given,
                               dmcg_plan** out, MeshHost* mesh_given = nullptr,
                               bool encode_side = true, cudaStream_t up_stream = nullptr) {
  *out = nullptr;
  if (n == 0 || F == 0) return {DMCG_E_INDEX, "ValidationError: sequence is empty"};
  if (dtype != DMCG_F64 && dtype != DMCG_F32) return {DMCG_E_CONFIG, "ConfigError: bad dtype"};
  auto* p = new dmcg_plan();
  p->ctx = ctx;
  p->n = n;
  p->F = F;
  p->dtype = dtype;
  p->n_faces = n_faces;
  PhaseTimer tm("plan");
  p->faces.assign(faces, faces + 3 * (size_t)n_faces);
  Status st;
  if (mesh_given) {
    p->mesh.n = n;
    p->mesh.lap_rp = std::move(mesh_given->lap_rp);
    p->mesh.lap_ci = std::move(mesh_given->lap_ci);
    p->mesh.adj_rp = std::move(mesh_given->adj_rp);  // present when the caller built the mesh
    p->mesh.adj_ci = std::move(mesh_given->adj_ci);
  } else {
    st = build_mesh(faces, n_faces, n, &p->mesh);
  }
  tm.lap("mesh");
  if (st.good() && !anchors_given) st = validate_mesh(p->mesh);
  tm.lap("validate");
  if (st.good()) st = check_config(*cfg, n, F, &p->row_bits);
  if (!st.good()) {
    delete p;
    return st;
  }
  p->k = cfg->k_l;
  p->k_l = cfg->k_l;
  p->F_in = F;
  if (cfg->variant == DMCG_BLOCKS) {
    // pad_frames (codec.cpp:43-49): the plan works on F + pad frames
    p->nb = cfg->n_b;
    p->pad = (p->nb - F % p->nb) % p->nb;
    F += p->pad;
    p->F = F;
    p->kf = F / p->nb;
    p->k = p->nb * p->k_l;
    if (p->kf > 512) {
      delete p;
      return {DMCG_E_UNSUPPORTED, "Unsupported: blocks of more than 512 frames"};
    }
    std::vector<int> tiled;
    for (uint32_t b = 0; b < p->nb; ++b) tiled.insert(tiled.end(), p->row_bits.begin(), p->row_bits.end());
    p->row_bits.swap(tiled);
  }
  p->t_max = cfg->t_max;
  p->oi_tol = cfg->oi_tolerance;
  p->variant = cfg->variant;
  // blocks: block 0 is always the full eigenbasis (codec.cpp:159); oi_rounds
  // only applies to the n_b = 1 rank-k path
  p->rounds = cfg->variant == DMCG_BLOCKS ? 0 : cfg->oi_rounds;
  p->oi_seed = cfg->oi_seed;
  p->implicit = cfg->oi_implicit != 0;
  p->anchor_bits = cfg->anchor_bits;
  p->dict_bits = cfg->dict_bits;
  p->diff_bits = cfg->diff_bits;
  // anchors (codec.cpp:374, 445)
  if (!variant_uses_anchors(p->variant)) {
    p->n_c = 0;  // anchor-free variants (codec.cpp:374)
  } else if (anchors_given) {
    p->n_c = n_c_given;
    p->mesh.anchors.assign(anchors_given, anchors_given + n_c_given);
  } else {
    p->n_c = dmcg_anchor_count(n, cfg->anchor_fraction);
    p->mesh.anchors.resize(p->n_c);
    if (dmcg_select_anchors(n, p->n_c, cfg->anchor_strategy, cfg->seed, p->mesh.anchors.data())) {
      delete p;
      return {DMCG_E_CONFIG, "InvalidCount: anchor count outside 1..n"};
    }
  }
  p->mesh.anchor_pos.assign(n, -1);
  for (uint32_t t = 0; t < p->n_c; ++t) p->mesh.anchor_pos[p->mesh.anchors[t]] = (int32_t)t;
  p->stats.nnz_laplacian = (long long)p->mesh.lap_ci.size();

  const uint32_t k = p->k;
  p->W = 3 * F;
  p->W_pad = (p->W + kColBlock - 1) / kColBlock * kColBlock;
  p->nblk = p->W_pad / kColBlock;
  const size_t nF = (size_t)n * F, FF = (size_t)F * F;
  const uint32_t F2 = F + (F & 1);
  const size_t kk = (size_t)std::max<uint32_t>(k, 1);
  bool ok = true;
  auto get = [&](size_t bytes) {
    void* d = plan_get(p, bytes);
    ok = ok && d;
    return d;
  };
  const MeshHost& m = p->mesh;
  p->d_lap_rp = (uint32_t*)get(m.lap_rp.size() * 4);
  p->d_lap_ci = (uint32_t*)get(m.lap_ci.size() * 4);
  p->d_anchor_idx = (uint32_t*)get((size_t)p->n_c * 4);
  p->d_anchor_pos = (int32_t*)get((size_t)n * 4);
  p->d_delta = (double*)get(3 * nF * 8);
  p->d_R = (double*)get(3 * FF * 8);
  const int tiles = ((F + 63) / 64) * ((F + 63) / 64);
  size_t splits = std::max<size_t>(1, (2 * 148 + tiles * 3 - 1) / (tiles * 3));
  // Ozaki INT8 tensor-core Gram for fp32 storage: its split-K
  // partials need the larger of the two partial counts
  p->oz_slices = 0;
  if (dtype == DMCG_F32 && p->nb == 1 && !getenv("DMCG_NO_OZAKI")) {
    const char* e = getenv("DMCG_OZ_SLICES");
    p->oz_slices = e ? std::max(3, std::min(7, atoi(e))) : 5;
    const size_t ozs = (size_t)dmcg::oz_gram_splits((int)F, (int)n, p->oz_slices);
    splits = std::max(splits, ozs);
  }
  p->part_elems = splits * 3 * FF;
  p->d_part = (double*)get(p->part_elems * 8);
  if (p->oz_slices) {
    // one slice buffer for the three Ozaki contractions of the plan (they
    // run one after another on the plan stream): the Gram (X^T X), the
    // projection (U_k^T, delta rows) and the decode's reconstruction (c~
    // rows, U~ rows); projection and reconstruction need K <= kOzKChunk
    using dmcg::oz_slice_bytes;
    using dmcg::oz_rows_pad;
    auto env_s = [](const char* name, int dflt) {
      const char* e = getenv(name);
      return e ? std::max(3, std::min(7, atoi(e))) : dflt;
    };
    const bool kfit = k > 0 && dmcg::oz_k_pad((int)F) <= dmcg::kOzKChunk &&
                      dmcg::oz_k_pad((int)k) <= dmcg::kOzKChunk;
    // the projection stays on DMMA unless asked for: its K = F is short, so
    // the slicing passes outweigh the tensor-core gain
    p->oz_proj_slices = (kfit && variant_uses_delta(p->variant) && getenv("DMCG_OZ_PROJ"))
                            ? env_s("DMCG_OZ_PROJ_SLICES", 6) : 0;
    p->oz_rec_slices = kfit ? env_s("DMCG_OZ_REC_SLICES", 4) : 0;
    if (getenv("DMCG_NO_OZAKI_GEMMS")) p->oz_proj_slices = p->oz_rec_slices = 0;
    size_t qb = oz_slice_bytes((int)F, (int)n, p->oz_slices, 3);
    size_t mx = 3 * (size_t)oz_rows_pad((int)F);
    if (p->oz_proj_slices) {
      const int sp = p->oz_proj_slices;
      qb = std::max(qb, oz_slice_bytes((int)k, (int)F, sp, 3) + oz_slice_bytes((int)n, (int)F, sp, 3));
      mx = std::max(mx, 3 * (size_t)(oz_rows_pad((int)k) + oz_rows_pad((int)n)));
    }
    if (p->oz_rec_slices) {
      const int sr = p->oz_rec_slices;
      qb = std::max(qb, oz_slice_bytes((int)n, (int)k, sr, 3) + oz_slice_bytes((int)F, (int)k, sr, 3));
      mx = std::max(mx, 3 * (size_t)(oz_rows_pad((int)n) + oz_rows_pad((int)F)));
    }
    p->oz_q_bytes = qb;
    p->oz_max_elems = mx;
    p->d_oz_q = (int8_t*)get(qb);
    p->d_oz_max = (unsigned long long*)get(mx * 8);
  }
  p->d_U = (double*)get(3 * FF * 8);
  p->d_evals = (double*)get(3 * (size_t)F * 8);
  p->d_Q = (double*)get(3 * (size_t)F * kk * 8);
  p->d_Z = (double*)get(3 * (size_t)F * kk * 8);
  p->d_tau = (double*)get(3 * (size_t)F * 8);
  size_t jac = 3 * 2 * (size_t)F2 * (F2 + 1);  // jacobi: A (m2 x m2+1) + V per axis
  if (p->nb > 1) {  // the blocks' eigenbases: 3 nb batches of kf
    const size_t kf2 = p->kf + (p->kf & 1);
    jac = std::max(jac, 3 * (size_t)p->nb * 2 * kf2 * (kf2 + 1));
  }
  // k_jacobi_blk keeps the eigenvectors of each (zero padded) 256 x 256
  // problem in this scratch
  jac = std::max(jac, 3 * (size_t)std::max<uint32_t>(p->nb, 1) * dmcg::kJacobiBlkWork);
  p->d_H = (double*)get(jac * 8);
  p->d_V = (double*)get(3 * FF * 8);
  p->d_qr_scr = (double*)get(3 * dmcg::qr_scratch_doubles((int)F, (int)kk) * 8);
  p->d_oi_mirror = (double*)get(dmcg::oi_mirror_doubles((int)F, 3) * 8);
  p->d_w = (double*)get(3 * (size_t)F * 8);
  p->d_start = (double*)get(3 * (size_t)F * kk * 8);
  p->d_C = (double*)get(3 * kk * std::max<size_t>(n, kk) * 8);
  // row (min, max) keys of the projection, then the 3 anchor-range pairs
  p->d_keys = (unsigned long long*)get((3 * kk + 3) * 2 * 8);
  p->d_flags = (int*)get(8 * sizeof(int));
  p->d_pf_flag = (int*)get(sizeof(int));
  p->d_dict_q = (uint16_t*)get(3 * FF * 2);
  p->d_row_min = (float*)get(3 * kk * 4);
  p->d_row_max = (float*)get(3 * kk * 4);
  p->d_row_bits = (uint8_t*)get(4 * kk);
  p->d_coeff_q = (uint16_t*)get(3 * kk * n * 2);
  p->d_anchor_rng = (float*)get(6 * 4);
  p->d_means = (float*)get(3 * (size_t)F * 4);
  p->d_colsum = (double*)get(3 * 64 * 3 * (size_t)F * 8);
  p->d_anchor_q = (uint16_t*)get(3 * (size_t)p->n_c * F * 2);
  p->d_rowp = (double*)get(3 * kk * 2 * 8);
  p->d_cg_iters = (int*)get(p->W_pad * 4);
  p->d_cg_res = (double*)get(p->W_pad * 8);
  if (p->nb > 1) {
    const size_t bk = (size_t)p->nb * p->kf * p->kf;
    p->d_bUeig = (double*)get(3 * bk * 8);
    p->d_bUd = (double*)get(3 * bk * 8);
    p->d_bwork = (double*)get(3 * dmcg::block_work_doubles((int)p->kf) * 8);
    p->d_diff_rng = (float*)get(3 * (size_t)(p->nb - 1) * 2 * 4);
    if (p->pad) p->d_xpad = get(3 * nF * (dtype == DMCG_F32 ? 4 : 8));
  }
  if (!ok) {
    dmcg_plan_destroy(p);
    return {DMCG_E_CUDA, "CudaError: device allocation failed"};
  }
  tm.lap("alloc");
  for (auto& e : p->ev) e = ctx->take_event(true);
  p->ev_fork = ctx->take_event(false);
  p->ev_join = ctx->take_event(false);
  p->ev_pf_fork = ctx->take_event(false);
  p->ev_pf_join = ctx->take_event(false);
  p->ev_pf0 = ctx->take_event(true);
  p->ev_pf1 = ctx->take_event(true);
  // the plan's (pageable) uploads go on the side stream and are waited for
  // here: a drop-in encode has already queued its input H2D on ctx->stream,
  // which keeps running under the host-side plan work
  cudaStream_t s = up_stream ? up_stream : ctx->aux;
  p->up_stream = up_stream;
  auto h2d = [&](void* d, const void* h, size_t bytes) {
    if (bytes) ok = ok && cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s) == cudaSuccess;
  };
  h2d(p->d_lap_rp, m.lap_rp.data(), m.lap_rp.size() * 4);
  h2d(p->d_lap_ci, m.lap_ci.data(), m.lap_ci.size() * 4);
  h2d(p->d_anchor_idx, m.anchors.data(), (size_t)p->n_c * 4);
  h2d(p->d_anchor_pos, m.anchor_pos.data(), (size_t)n * 4);
  std::vector<uint8_t> rb(4 * kk, 0);
  for (uint32_t r = 0; r < k; ++r) rb[3 * kk + r] = (uint8_t)p->row_bits[r];
  h2d(p->d_row_bits, rb.data(), rb.size());
  // OI start matrices: SplitMix64 uniform in [-1, 1), column-major F x k,
  // axis a seeded with oi_seed + a (same stream as oracle orc_start_matrix).
  std::vector<double> start(3 * (size_t)F * kk, 0.0);
  if (k > 0 && encode_side)
    for (int a = 0; a < 3; ++a) {
      uint64_t st64 = p->oi_seed + (uint64_t)a;
      for (size_t t = 0; t < (size_t)F * k; ++t)
        start[a * (size_t)F * k + t] = (double)(splitmix64(&st64) >> 11) * 0x1.0p-52 - 1.0;
    }
  tm.lap("events+start");
  if (encode_side) h2d(p->d_start, start.data(), start.size() * 8);
  if (ctx->after_plan_uploads) {
    ctx->after_plan_uploads();
    ctx->after_plan_uploads = nullptr;
  }
  if (ok) ok = cudaStreamSynchronize(s) == cudaSuccess;
  tm.lap("upload+sync");
  if (!ok) {
    dmcg_plan_destroy(p);
    return {DMCG_E_CUDA, "CudaError: plan upload failed"};
  }
  *out = p;
  return Status::ok();
}

}  // extern "C"

// Decode-side state (symbolic Cholesky analysis of M, factor / RHS buffers)
// is built on the first decode of a plan only: encode-only plans never pay
// for it.  Reference: the normal matrix and its factorisation are per
// decode call (solver.cpp:62-90).
// M = L^T L + S^T S on the host and in HBM, built on first use (only the
// decoder needs it; solver.cpp:25-39).
dmcg::Status dmcg::plan_prepare_normal(dmcg_plan* p) {
  if (p->d_m_rp) return Status::ok();
  PhaseTimer tm("normal");
  if (!p->chol_given) {
    if (variant_uses_means(p->variant))
      build_reduced_normal(&p->mesh);
    else
      build_normal_matrix(&p->mesh);
  }
  tm.lap("build");
  const MeshHost& m = p->mesh;
  p->stats.nnz_normal = (long long)m.m_ci.size();
  p->d_m_rp = (uint32_t*)plan_alloc(p, m.m_rp.size() * 4);
  p->d_m_ci = (uint32_t*)plan_alloc(p, m.m_ci.size() * 4);
  p->d_m_val = (float*)plan_alloc(p, m.m_val.size() * 4);
  if (!p->d_m_rp || !p->d_m_ci || !p->d_m_val)
    return {DMCG_E_CUDA, "CudaError: device allocation failed"};
  cudaStream_t s = p->up_stream ? p->up_stream : p->ctx->stream;
  bool ok = cudaMemcpyAsync(p->d_m_rp, m.m_rp.data(), m.m_rp.size() * 4, cudaMemcpyHostToDevice,
                            s) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(p->d_m_ci, m.m_ci.data(), m.m_ci.size() * 4,
                             cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(p->d_m_val, m.m_val.data(), m.m_val.size() * 4,
                             cudaMemcpyHostToDevice, s) == cudaSuccess;
  if (!ok) return {DMCG_E_CUDA, "CudaError: normal matrix upload failed"};
  tm.lap("upload");
  return Status::ok();
}

dmcg::Status dmcg::plan_prepare_decode(dmcg_plan* p) {
  if (p->decode_ready) return Status::ok();
  PhaseTimer tm("prepare");
  if (p->variant == DMCG_V2V) {  // no solve: the reconstruction buffers only
    const size_t nW = (size_t)p->n * p->W;
    p->d_rm_delta = (double*)plan_alloc(p, nW * 8);
    p->d_Ud = (double*)plan_alloc(p, 3 * (size_t)std::max<uint32_t>(p->k, 1) * p->F * 8);
    if (!p->d_rm_delta || !p->d_Ud) return {DMCG_E_CUDA, "CudaError: device allocation failed"};
    p->decode_ready = true;
    return Status::ok();
  }
  {
    Status sn = plan_prepare_normal(p);
    if (!sn.good()) return sn;
  }
  tm.lap("normal matrix");
  const uint32_t n = p->n;
  // the anchor-free variants solve with vertex 0 pinned: n - 1 unknowns
  const uint32_t nm = variant_uses_means(p->variant) ? n - 1 : n;
  const MeshHost& m = p->mesh;
  bool ok = true;
  auto get = [&](size_t bytes) {
    void* d = plan_alloc(p, bytes);
    ok = ok && d;
    return d;
  };
  // direct solver: symbolic analysis of M (host) + device structures
  {
    const auto t0 = std::chrono::steady_clock::now();
    if (!p->chol_given)
      chol_analyze(nm, m.m_rp, m.m_ci, m.m_val, &p->chol, nm == n ? &m.lap_rp : nullptr,
                   nm == n ? &m.lap_ci : nullptr);
    p->analyze_seconds = p->chol_given
                             ? p->analyze_seconds
                             : std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
                                   .count();
  }
  tm.lap("analyze");
  const CholPlan& cp = p->chol;
  const size_t nW = (size_t)n * p->W;
  p->d_rm_delta = (double*)get(nW * 8);
  p->d_rm_b = (double*)get(nW * 8);
  p->d_rm_x = (double*)get(nW * 8);
  p->d_rm_y = (double*)get(nW * 8);
  p->d_rm_xp = (double*)get(nW * 8);
  p->d_rm_r = (double*)get(nW * 8);
  p->d_Ud = (double*)get(3 * (size_t)std::max<uint32_t>(p->k, 1) * p->F * 8);
  CholDev& cd = p->cdev;
  cd.n = nm;
  cd.nsup = cp.nsup;
  cd.W = p->W;
  cd.first = (const uint32_t*)get(cp.first.size() * 4);
  cd.str_ptr = (const unsigned long long*)get(cp.str_ptr.size() * 8);
  cd.str_idx = (const uint32_t*)get(cp.str_idx.size() * 4);
  cd.child_ptr = (const uint32_t*)get(cp.child_ptr.size() * 4);
  cd.child_idx = (const uint32_t*)get(cp.child_idx.size() * 4 + 4);
  cd.rel_ptr = (const unsigned long long*)get(cp.rel_ptr.size() * 8);
  cd.rel_idx = (const uint32_t*)get(cp.rel_idx.size() * 4 + 4);
  cd.a_ptr = (const unsigned long long*)get(cp.a_ptr.size() * 8);
  cd.a_pos = (const uint32_t*)get(cp.a_pos.size() * 4);
  cd.a_val = (const float*)get(cp.a_val.size() * 4);
  cd.front_off = (const unsigned long long*)get(cp.front_off.size() * 8);
  cd.inv_off = (const unsigned long long*)get(cp.inv_off.size() * 8);
  cd.rhs_off = (const unsigned long long*)get(cp.rhs_off.size() * 8);
  cd.op_off = (const unsigned long long*)get(cp.op_off.size() * 8);
  cd.perm = (const uint32_t*)get(cp.perm.size() * 4);
  cd.level_sup = (const uint32_t*)get(cp.level_sup.size() * 4 + 4);
  cd.level_ptr = (const uint32_t*)get(cp.level_ptr.size() * 4 + 4);
  cd.pull_ptr = (const uint32_t*)get(cp.pull_ptr.size() * 4 + 4);
  cd.pull_src = (const uint32_t*)get(cp.pull_src.size() * 4 + 4);
  cd.nlevels = cp.nlevels;
  cd.F = (double*)get(cp.front_off[cp.nsup] * 8);
  cd.Linv = (double*)get(cp.inv_off[cp.nsup] * 8 + 8);
  cd.P = (double*)get(cp.op_off[cp.nsup] * 8 + 8);
  cd.R = (double*)get(cp.rhs_off[cp.nsup] * p->W * 8);
  cd.flags = p->d_flags + 4;
  CholLevels& lv = p->levels;
  lv.nlevels = cp.nlevels;
  lv.offset.assign(cp.nlevels, 0);
  lv.count.assign(cp.nlevels, 0);
  lv.maxw.assign(cp.nlevels, 0);
  lv.maxm.assign(cp.nlevels, 0);
  lv.maxu.assign(cp.nlevels, 0);
  for (uint32_t l = 0; l < cp.nlevels; ++l) {
    lv.offset[l] = cp.level_ptr[l];
    lv.count[l] = cp.level_ptr[l + 1] - cp.level_ptr[l];
    for (uint32_t q = cp.level_ptr[l]; q < cp.level_ptr[l + 1]; ++q) {
      const uint32_t s = cp.level_sup[q];
      lv.maxw[l] = std::max(lv.maxw[l], cp.w(s));
      lv.maxm[l] = std::max(lv.maxm[l], cp.m(s));
      lv.maxu[l] = std::max(lv.maxu[l], cp.m(s) - cp.w(s));
    }
  }
  cd.linv_doubles = cp.inv_off[cp.nsup];
  cd.scratch = (double*)get(chol_scratch_doubles(lv) * 8 + 8);
  p->stats.supernodes = (int)cp.nsup;
  p->stats.levels = (int)cp.nlevels;
  p->stats.nnz_factor = (long long)cp.nnz_l;
  p->stats.flops_factor = cp.flops_factor;
  p->stats.analyze_seconds = p->analyze_seconds;
  if (!ok) return {DMCG_E_CUDA, "CudaError: device allocation failed"};
  tm.lap("alloc");
  cudaStream_t s = p->up_stream ? p->up_stream : p->ctx->stream;
  auto h2d = [&](void* d, const void* h, size_t bytes) {
    if (bytes) ok = ok && cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s) == cudaSuccess;
  };
  h2d((void*)cd.first, cp.first.data(), cp.first.size() * 4);
  h2d((void*)cd.str_ptr, cp.str_ptr.data(), cp.str_ptr.size() * 8);
  h2d((void*)cd.str_idx, cp.str_idx.data(), cp.str_idx.size() * 4);
  h2d((void*)cd.child_ptr, cp.child_ptr.data(), cp.child_ptr.size() * 4);
  h2d((void*)cd.child_idx, cp.child_idx.data(), cp.child_idx.size() * 4);
  h2d((void*)cd.rel_ptr, cp.rel_ptr.data(), cp.rel_ptr.size() * 8);
  h2d((void*)cd.rel_idx, cp.rel_idx.data(), cp.rel_idx.size() * 4);
  h2d((void*)cd.a_ptr, cp.a_ptr.data(), cp.a_ptr.size() * 8);
  h2d((void*)cd.a_pos, cp.a_pos.data(), cp.a_pos.size() * 4);
  h2d((void*)cd.a_val, cp.a_val.data(), cp.a_val.size() * 4);
  h2d((void*)cd.front_off, cp.front_off.data(), cp.front_off.size() * 8);
  h2d((void*)cd.inv_off, cp.inv_off.data(), cp.inv_off.size() * 8);
  h2d((void*)cd.rhs_off, cp.rhs_off.data(), cp.rhs_off.size() * 8);
  h2d((void*)cd.op_off, cp.op_off.data(), cp.op_off.size() * 8);
  h2d((void*)cd.perm, cp.perm.data(), cp.perm.size() * 4);
  h2d((void*)cd.level_sup, cp.level_sup.data(), cp.level_sup.size() * 4);
  h2d((void*)cd.level_ptr, cp.level_ptr.data(), cp.level_ptr.size() * 4);
  h2d((void*)cd.pull_ptr, cp.pull_ptr.data(), cp.pull_ptr.size() * 4);
  h2d((void*)cd.pull_src, cp.pull_src.data(), cp.pull_src.size() * 4);
  if (ok) ok = cudaStreamSynchronize(s) == cudaSuccess;
  if (!ok) return {DMCG_E_CUDA, "CudaError: decode plan upload failed"};
  tm.lap("upload+sync");
  p->decode_ready = true;
  return Status::ok();
}

extern "C" {

static Status plan_serialize_impl(dmcg_plan* p, uint8_t* out, size_t cap, dmcg_sections* sec,
                                  size_t* size);

int dmcg_plan_distortion(dmcg_plan* p, const void* const d_orig[3], const void* const d_recon[3],
                         double* frame_rms, double* nmsve, double* vertex_mean_error) {
  if (!p || !d_orig || !d_recon || !frame_rms || !nmsve) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  const size_t n = p->n, F = p->F_in;  // the caller's (unpadded) frames
  if (!p->d_metric) p->d_metric = (double*)plan_alloc(p, (3 * n * F + 2 * F + n) * 8);
  if (!p->d_metric) return p->ctx->set_error({DMCG_E_CUDA, "CudaError: device allocation failed"});
  cudaStream_t s = p->ctx->stream;
  double* rms = p->d_metric + 3 * n * F;
  double* nm = rms + F;
  double* vme = nm + F;
  cudaError_t e = launch_distortion(s, (int)n, (int)F, p->d_lap_rp, p->d_lap_ci, d_orig, d_recon,
                                    p->dtype == DMCG_F32, p->d_metric, rms, nm,
                                    vertex_mean_error ? vme : nullptr);
  if (e == cudaSuccess) e = cudaMemcpyAsync(frame_rms, rms, F * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(nmsve, nm, F * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && vertex_mean_error)
    e = cudaMemcpyAsync(vertex_mean_error, vme, n * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess)
    return p->ctx->set_error({DMCG_E_CUDA, std::string("CudaError: ") + cudaGetErrorString(e)});
  return DMCG_OK;
}

size_t dmcg_plan_serialize(dmcg_plan* p, uint8_t* out, size_t cap, dmcg_sections* sec) {
  if (!p) return 0;
  cudaSetDevice(p->ctx->device);
  size_t size = 0;
  Status st = plan_serialize_impl(p, out, cap, sec, &size);
  p->ctx->set_error(st);
  return st.good() ? size : 0;
}

int dmcg_plan_create(dmcg_ctx* ctx, uint32_t n, uint32_t F, int dtype, const uint32_t* faces,
                     uint32_t n_faces, const dmcg_config* cfg, dmcg_plan** plan) {
  if (!ctx || !plan || !cfg) return DMCG_E_CONFIG;
  cudaSetDevice(ctx->device);
  Status st = plan_create_impl(ctx, n, F, dtype, faces, n_faces, cfg, nullptr, 0, plan);
  if (st.good()) (*plan)->use_graphs = true;  // reused across calls: replay CUDA graphs
  return ctx->set_error(st);
}

int dmcg_plan_create_shard(dmcg_ctx* ctx, uint32_t n, uint32_t F, int dtype, const uint32_t* faces,
                           uint32_t n_faces, const dmcg_config* cfg, int nranks, int rank,
                           dmcg_comm* comm, dmcg_plan** plan) {
  if (!ctx || !plan || !cfg || nranks < 1 || rank < 0 || rank >= nranks) return DMCG_E_CONFIG;
  if (n < (uint32_t)nranks)
    return ctx->set_error({DMCG_E_CONFIG, "ConfigError: fewer vertices than ranks"});
  if (variant_uses_means(cfg->variant))
    return ctx->set_error({DMCG_E_UNSUPPORTED,
                           "Unsupported: vertex-row shards of the pca / pca_q variants (their "
                           "frame means need a cross-rank reduction)"});
  if (cfg->variant == DMCG_BLOCKS)
    return ctx->set_error({DMCG_E_UNSUPPORTED,
                           "Unsupported: vertex-row shards of the blocks variant"});
  if (comm && (comm_size(comm) != nranks || comm_rank(comm) != rank))
    return ctx->set_error({DMCG_E_CONFIG, "ConfigError: communicator does not match rank"});
  cudaSetDevice(ctx->device);
  Status st = plan_create_impl(ctx, n, F, dtype, faces, n_faces, cfg, nullptr, 0, plan);
  if (!st.good()) return ctx->set_error(st);
  dmcg_plan* p = *plan;
  p->use_graphs = true;  // decode graphs; the sharded encode launches directly
  p->shard.reset(new ShardState());
  ShardState& sh = *p->shard;
  shard_layout(p->mesh, F, p->k, nranks, rank, &sh);
  sh.comm = comm;
  const uint32_t na = sh.a0[rank + 1] - sh.a0[rank];
  std::vector<uint32_t> loc_anchor(na);
  for (uint32_t t = 0; t < na; ++t) loc_anchor[t] = p->mesh.anchors[sh.a0[rank] + t] - sh.r0[rank];
  sh.d_loc_rp = (uint32_t*)plan_get(p, sh.loc_rp.size() * 4);
  sh.d_loc_ci = (uint32_t*)plan_get(p, sh.loc_ci.size() * 4);
  sh.d_loc_anchor = (uint32_t*)plan_get(p, (size_t)na * 4);
  sh.d_keys = (unsigned long long*)plan_get(p, (3 * (size_t)p->k + 3) * 2 * 8);
  sh.d_gather = (uint16_t*)plan_get(p, sh.stage_off[nranks] * 2);
  bool ok = sh.d_loc_rp && sh.d_loc_ci && sh.d_loc_anchor && sh.d_keys && sh.d_gather;
  cudaStream_t s = ctx->stream;
  auto h2d = [&](void* d, const void* h, size_t bytes) {
    if (bytes && ok) ok = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s) == cudaSuccess;
  };
  h2d(sh.d_loc_rp, sh.loc_rp.data(), sh.loc_rp.size() * 4);
  h2d(sh.d_loc_ci, sh.loc_ci.data(), sh.loc_ci.size() * 4);
  h2d(sh.d_loc_anchor, loc_anchor.data(), (size_t)na * 4);
  if (ok) ok = cudaStreamSynchronize(s) == cudaSuccess;
  if (!ok) {
    dmcg_plan_destroy(p);
    *plan = nullptr;
    return ctx->set_error({DMCG_E_CUDA, "CudaError: shard plan allocation / upload failed"});
  }
  return ctx->set_error(Status::ok());
}

int dmcg_plan_encode_device(dmcg_plan* p, const void* const d_axes[3]) {
  if (!p) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  return p->ctx->set_error(plan_encode(p, d_axes));
}

int dmcg_plan_decode_device(dmcg_plan* p, const dmcg_decode_options* opt, void* const d_out[3]) {
  if (!p) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  dmcg_decode_options o;
  dmcg_decode_options_default(&o);
  if (opt) o = *opt;
  return p->ctx->set_error(plan_decode(p, &o, d_out));
}

// download = issue (header fields + every D2H copy queued on the plan stream,
// asynchronous for page-locked destinations) + a stream synchronise + finish
// (host-side fix-ups).  dmcg_encode queues the copies behind its kernels and
// prepares the next decode before waiting for them.
static Status download_issue(dmcg_plan* p, dmcg_encoded* e) {
  cudaStream_t s = p->ctx->stream;
  // blocks: per axis nb k_f^2 dictionary levels and nb k_l rows; anchors
  // and frames unpadded (F_in) on the host
  const size_t n = p->n, F = p->F, k = p->k, Fo = p->F_in;
  const size_t FF = p->nb > 1 ? (size_t)p->nb * p->kf * p->kf : F * F;
  e->n = p->n;
  e->F = p->F_in;
  e->k_l = p->k_l;
  e->n_b = (uint16_t)p->nb;
  e->pad = (uint16_t)p->pad;
  e->n_c = p->n_c;
  e->n_faces = p->n_faces;
  e->variant = (uint8_t)p->variant;
  e->flags = 0;
  e->anchor_bits = (uint8_t)p->anchor_bits;
  e->dict_bits = (uint8_t)p->dict_bits;
  e->diff_bits = (uint8_t)p->diff_bits;
  if (!e->faces) e->faces = p->faces.data();
  float* rng = p->h_anchor_rng;
  for (int a = 0; a < 3; ++a) {
    CUDA_OK(cudaMemcpyAsync(e->dict_q[a], p->d_dict_q + a * FF, FF * 2, cudaMemcpyDeviceToHost, s));
    if (k) {
      CUDA_OK(cudaMemcpyAsync(e->row_min[a], p->d_row_min + a * k, k * 4, cudaMemcpyDeviceToHost, s));
      CUDA_OK(cudaMemcpyAsync(e->row_max[a], p->d_row_max + a * k, k * 4, cudaMemcpyDeviceToHost, s));
      CUDA_OK(cudaMemcpyAsync(e->row_bits[a], p->d_row_bits + a * k, k, cudaMemcpyDeviceToHost, s));
      if (!p->coeff_streamed)  // else already on its way (enqueue_encode, per axis)
        CUDA_OK(cudaMemcpyAsync(e->coeff_q[a], p->d_coeff_q + a * k * n, k * n * 2,
                                cudaMemcpyDeviceToHost, s));
    }
    if (p->n_c)
      CUDA_OK(cudaMemcpy2DAsync(e->anchor_q[a], Fo * 2, p->d_anchor_q + a * (size_t)p->n_c * F,
                                F * 2, Fo * 2, p->n_c, cudaMemcpyDeviceToHost, s));
    if (p->nb > 1) {
      std::vector<float> rng2(2 * (p->nb - 1));
      // pageable destination: returns once the copy (ordered on the plan stream) is done
      CUDA_OK(cudaMemcpyAsync(rng2.data(), p->d_diff_rng + a * rng2.size(), rng2.size() * 4,
                              cudaMemcpyDeviceToHost, s));
      for (uint32_t b = 0; b + 1 < p->nb; ++b) {
        e->diff_min[a][b] = rng2[2 * b];
        e->diff_max[a][b] = rng2[2 * b + 1];
      }
    }
    if (variant_uses_means(p->variant) && e->means[a])
      CUDA_OK(cudaMemcpyAsync(e->means[a], p->d_means + a * F, F * 4, cudaMemcpyDeviceToHost, s));
  }
  std::memset(rng, 0, 6 * sizeof(float));
  if (p->n_c)
    CUDA_OK(cudaMemcpyAsync(rng, p->d_anchor_rng, 6 * sizeof(float), cudaMemcpyDeviceToHost, s));
  return Status::ok();
}
static void download_finish(dmcg_plan* p, dmcg_encoded* e) {
  const size_t n = p->n, k = p->k;
  const float* rng = p->h_anchor_rng;
  if (p->n_c) std::memcpy(e->anchor_idx, p->mesh.anchors.data(), (size_t)p->n_c * 4);
  for (int a = 0; a < 3; ++a) {
    e->anchor_min[a] = rng[2 * a];
    e->anchor_max[a] = rng[2 * a + 1];
  }
  // Degenerate rows carry no payload (codec.cpp:259-262): zero their levels
  // so the representation is canonical.
  for (int a = 0; a < 3; ++a)
    for (size_t r = 0; r < k; ++r)
      if (e->row_min[a][r] == e->row_max[a][r])
        std::memset(e->coeff_q[a] + r * n, 0, n * 2);
}
static Status download_impl(dmcg_plan* p, dmcg_encoded* e) {
  Status st = download_issue(p, e);
  if (!st.good()) return st;
  CUDA_OK(cudaStreamSynchronize(p->ctx->stream));
  download_finish(p, e);
  return Status::ok();
}

int dmcg_plan_download(dmcg_plan* p, dmcg_encoded* out) {
  if (!p || !out) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  return p->ctx->set_error(download_impl(p, out));
}

// dmcg_plan_serialize: host frame + device payload packing (see dmcg.h).
static Status plan_serialize_impl(dmcg_plan* p, uint8_t* out, size_t cap, dmcg_sections* sec,
                                  size_t* size) {
  cudaStream_t s = p->ctx->stream;
  if (p->nb > 1) {
    // blocks: the per-block sections are framed on the host from the
    // downloaded symbols (the device packer covers the n_b = 1 layout)
    const size_t nb = p->nb, kk = (size_t)p->kf * p->kf, rows = (size_t)p->k;
    std::vector<uint16_t> dq(3 * nb * kk), cq(3 * rows * p->n), aq(3 * (size_t)p->n_c * p->F_in);
    std::vector<float> rmin(3 * rows + 1), rmax(3 * rows + 1), dmin(3 * nb), dmax(3 * nb);
    std::vector<uint8_t> rbits(3 * rows + 1);
    std::vector<uint32_t> aidx(p->n_c + 1);
    dmcg_encoded m;
    std::memset(&m, 0, sizeof(m));
    for (int a = 0; a < 3; ++a) {
      m.dict_q[a] = dq.data() + a * nb * kk;
      m.row_min[a] = rmin.data() + a * rows;
      m.row_max[a] = rmax.data() + a * rows;
      m.row_bits[a] = rbits.data() + a * rows;
      m.coeff_q[a] = cq.data() + a * rows * p->n;
      m.anchor_q[a] = aq.data() + a * (size_t)p->n_c * p->F_in;
      m.diff_min[a] = dmin.data() + a * nb;
      m.diff_max[a] = dmax.data() + a * nb;
    }
    m.anchor_idx = aidx.data();
    m.faces = p->faces.data();
    Status st = download_impl(p, &m);
    if (!st.good()) return st;
    *size = serialize_stream(&m, nullptr, 0, sec, nullptr);
    if (!out) return Status::ok();
    if (cap < *size) return {DMCG_E_CONFIG, "ConfigError: serialize buffer too small"};
    serialize_stream(&m, out, cap, sec, nullptr);
    return Status::ok();
  }
  const size_t n = p->n, F = p->F, k = p->k;
  std::vector<float> rmin(3 * k + 1), rmax(3 * k + 1);
  std::vector<uint8_t> rbits(3 * k + 1);
  float rng[6] = {0, 0, 0, 0, 0, 0};
  std::vector<float> means(3 * F);
  if (k) {
    CUDA_OK(cudaMemcpyAsync(rmin.data(), p->d_row_min, 3 * k * 4, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(rmax.data(), p->d_row_max, 3 * k * 4, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(rbits.data(), p->d_row_bits, 3 * k, cudaMemcpyDeviceToHost, s));
  }
  if (p->n_c) CUDA_OK(cudaMemcpyAsync(rng, p->d_anchor_rng, sizeof(rng), cudaMemcpyDeviceToHost, s));
  if (variant_uses_means(p->variant))
    CUDA_OK(cudaMemcpyAsync(means.data(), p->d_means, 3 * F * 4, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  dmcg_encoded m;
  std::memset(&m, 0, sizeof(m));
  m.n = p->n;
  m.F = p->F;
  m.k_l = p->k;
  m.n_c = p->n_c;
  m.n_faces = p->n_faces;
  m.variant = (uint8_t)p->variant;
  m.anchor_bits = (uint8_t)p->anchor_bits;
  m.dict_bits = (uint8_t)p->dict_bits;
  m.diff_bits = (uint8_t)p->diff_bits;
  m.faces = p->faces.data();
  m.anchor_idx = p->mesh.anchors.data();
  for (int a = 0; a < 3; ++a) {
    m.row_min[a] = rmin.data() + a * k;
    m.row_max[a] = rmax.data() + a * k;
    m.row_bits[a] = rbits.data() + a * k;
    m.anchor_min[a] = rng[2 * a];
    m.anchor_max[a] = rng[2 * a + 1];
    m.means[a] = means.data() + a * F;
  }
  PayloadSpans sp{};
  const size_t total = serialize_stream(&m, nullptr, 0, sec, &sp);
  *size = total;
  if (!out) return Status::ok();
  if (cap < total) return {DMCG_E_CONFIG, "ConfigError: serialize buffer too small"};
  serialize_stream(&m, out, cap, sec, &sp);  // header, faces, row headers, indices, ranges
  // payload bit offsets of the coefficient rows (degenerate rows carry none)
  std::vector<unsigned long long> off(3 * k + 1, ~0ull);
  for (int a = 0; a < 3; ++a) {
    unsigned long long bit = 0;
    for (size_t r = 0; r < k; ++r)
      if (rmin[a * k + r] != rmax[a * k + r]) {
        off[a * k + r] = bit;
        bit += (unsigned long long)n * rbits[a * k + r];
      }
  }
  const size_t words = (total + 3) / 4;
  if (p->stream_cap < words) {
    p->d_stream = (uint32_t*)plan_alloc(p, words * 4);
    p->stream_cap = p->d_stream ? words : 0;
  }
  if (!p->d_row_bitoff) p->d_row_bitoff = (unsigned long long*)plan_alloc(p, (3 * k + 1) * 8);
  if (!p->d_stream || !p->d_row_bitoff)
    return {DMCG_E_CUDA, "CudaError: device allocation failed"};
  CUDA_OK(cudaMemsetAsync(p->d_stream, 0, words * 4, s));
  if (k)
    CUDA_OK(cudaMemcpyAsync(p->d_row_bitoff, off.data(), 3 * k * 8, cudaMemcpyHostToDevice, s));
  const size_t FF = F * F;
  for (int a = 0; a < 3; ++a) {
    CUDA_OK(launch_pack_uniform(s, p->d_dict_q + a * FF, (long)FF, p->dict_bits, sp.dict[a],
                                p->d_stream));
    if (k)
      CUDA_OK(launch_pack_rows(s, p->d_coeff_q + a * k * n, (long)n, (int)k, p->d_row_bits + a * k,
                               p->d_row_bitoff + a * k, sp.coeff[a], p->d_stream));
    if (p->n_c)
      CUDA_OK(launch_pack_uniform(s, p->d_anchor_q + a * (size_t)p->n_c * F, (long)p->n_c * F,
                                  p->anchor_bits, sp.anchor[a], p->d_stream));
  }
  const uint8_t* dev = (const uint8_t*)p->d_stream;
  auto span_copy = [&](size_t off0, size_t bytes) -> cudaError_t {
    return bytes ? cudaMemcpyAsync(out + off0, dev + off0, bytes, cudaMemcpyDeviceToHost, s)
                 : cudaSuccess;
  };
  for (int a = 0; a < 3; ++a) {
    size_t cbits = 0;
    for (size_t r = 0; r < k; ++r)
      if (rmin[a * k + r] != rmax[a * k + r]) cbits += n * rbits[a * k + r];
    CUDA_OK(span_copy(sp.dict[a], (FF * p->dict_bits + 7) / 8));
    CUDA_OK(span_copy(sp.coeff[a], (cbits + 7) / 8));
    CUDA_OK(span_copy(sp.anchor[a], ((size_t)p->n_c * F * p->anchor_bits + 7) / 8));
  }
  CUDA_OK(cudaStreamSynchronize(s));
  return Status::ok();
}

// stream_coeffs (the drop-in decode of a single-block stream held in
// page-locked arrays): the coefficient symbols, the bulk of the stream, go axis
// by axis on the copy stream with an event each, and the reconstruction starts
// on an axis while the next is in flight (pipeline.cu, coeff_events).
static Status upload_impl(dmcg_plan* p, const dmcg_encoded* e, bool stream_coeffs = false) {
  cudaStream_t s = p->ctx->stream;
  p->rec_a_valid = false;  // new coefficient symbols
  if (stream_coeffs && p->k > 0 && p->nb == 1) {
    for (int a = 0; a < 3 && stream_coeffs; ++a) {
      cudaPointerAttributes at;
      stream_coeffs = e->coeff_q[a] &&
                      cudaPointerGetAttributes(&at, e->coeff_q[a]) == cudaSuccess &&
                      at.type == cudaMemoryTypeHost;
    }
    cudaGetLastError();
  } else {
    stream_coeffs = false;
  }
  p->coeff_events = stream_coeffs;
  PhaseTimer tu("upload");
  if (stream_coeffs) tu.lap("streamed symbols: yes");
  const size_t n = p->n, F = p->F, k = p->k, Fo = p->F_in;
  const size_t FF = p->nb > 1 ? (size_t)p->nb * p->kf * p->kf : F * F;
  float rng[6];
  if (p->nb > 1) {
    std::vector<float> rng2(3 * 2 * (p->nb - 1));
    for (int a = 0; a < 3; ++a)
      for (uint32_t b = 0; b + 1 < p->nb; ++b) {
        rng2[(a * (p->nb - 1) + b) * 2] = e->diff_min[a][b];
        rng2[(a * (p->nb - 1) + b) * 2 + 1] = e->diff_max[a][b];
      }
    // pageable source: staged before return, so rng2 may go out of scope
    CUDA_OK(cudaMemcpyAsync(p->d_diff_rng, rng2.data(), rng2.size() * 4, cudaMemcpyHostToDevice, s));
  }
  for (int a = 0; a < 3; ++a) {
    CUDA_OK(cudaMemcpyAsync(p->d_dict_q + a * FF, e->dict_q[a], FF * 2, cudaMemcpyHostToDevice, s));
    if (k) {
      CUDA_OK(cudaMemcpyAsync(p->d_row_min + a * k, e->row_min[a], k * 4, cudaMemcpyHostToDevice, s));
      CUDA_OK(cudaMemcpyAsync(p->d_row_max + a * k, e->row_max[a], k * 4, cudaMemcpyHostToDevice, s));
      CUDA_OK(cudaMemcpyAsync(p->d_row_bits + a * k, e->row_bits[a], k, cudaMemcpyHostToDevice, s));
      if (!stream_coeffs)
        CUDA_OK(cudaMemcpyAsync(p->d_coeff_q + a * k * n, e->coeff_q[a], k * n * 2,
                                cudaMemcpyHostToDevice, s));
    }
    if (p->n_c)
      CUDA_OK(cudaMemcpy2DAsync(p->d_anchor_q + a * (size_t)p->n_c * F, F * 2, e->anchor_q[a],
                                Fo * 2, Fo * 2, p->n_c, cudaMemcpyHostToDevice, s));
    if (variant_uses_means(p->variant)) {
      if (!e->means[a]) return {DMCG_E_CORRUPT, "CorruptPayload: missing frame means"};
      CUDA_OK(cudaMemcpyAsync(p->d_means + a * F, e->means[a], F * 4, cudaMemcpyHostToDevice, s));
    }
    rng[2 * a] = e->anchor_min[a];
    rng[2 * a + 1] = e->anchor_max[a];
  }
  CUDA_OK(cudaMemcpyAsync(p->d_anchor_rng, rng, sizeof(rng), cudaMemcpyHostToDevice, s));
  // the streamed symbols last: the copy engine serves its queue in order, and
  // the small arrays above must not wait behind 400 MB
  if (stream_coeffs)
    for (int a = 0; a < 3; ++a) {
      CUDA_OK(cudaMemcpyAsync(p->d_coeff_q + a * k * n, e->coeff_q[a], k * n * 2,
                              cudaMemcpyHostToDevice, p->ctx->copy));
      CUDA_OK(cudaEventRecord(p->ctx->ev_in[a], p->ctx->copy));
    }
  // the decoder's anchor padding (codec.cpp:483-495): frames F_in.. repeat the last
  if (p->n_c && F > Fo) CUDA_OK(launch_pad_anchor_levels(s, (int)p->n_c, (int)Fo, (int)F, p->d_anchor_q));
  tu.lap("issue");
  // dmcg_plan_upload returns with the copies done (the caller may reuse its
  // arrays); the drop-in decode keeps the caller's arrays until it returns and
  // lets its kernels follow the copies in stream order (the stack / vector
  // sources above are pageable: staged before cudaMemcpyAsync returns)
  if (!stream_coeffs) CUDA_OK(cudaStreamSynchronize(s));
  tu.lap("sync");
  return Status::ok();
}

int dmcg_plan_upload(dmcg_plan* p, const dmcg_encoded* in) {
  if (!p || !in) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  return p->ctx->set_error(upload_impl(p, in));
}

int dmcg_plan_delta(dmcg_plan* p, int axis, double* delta_host) {
  if (!p || !delta_host || axis < 0 || axis > 2 || p->nb > 1 || !p->d_delta) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  const size_t nF = (size_t)p->n * p->F;
  cudaStream_t s = p->ctx->stream;
  cudaMemcpyAsync(delta_host, p->d_delta + axis * nF, nF * 8, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return DMCG_E_CUDA;
  return DMCG_OK;
}

int dmcg_plan_basis(dmcg_plan* p, int axis, double* U_host, double* evals_host) {
  if (!p || axis < 0 || axis > 2) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  // blocks: the nb k_f x k_f dictionaries of the axis (nb k_f^2 doubles);
  // evals = the per-block eigenvalues of the direct decomposition
  const size_t FF = p->nb > 1 ? (size_t)p->nb * p->kf * p->kf : (size_t)p->F * p->F;
  cudaStream_t s = p->ctx->stream;
  if (U_host) cudaMemcpyAsync(U_host, p->d_U + axis * FF, FF * 8, cudaMemcpyDeviceToHost, s);
  if (evals_host)
    cudaMemcpyAsync(evals_host, p->d_evals + (size_t)axis * p->F, p->F * 8, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return DMCG_E_CUDA;
  return DMCG_OK;
}

int dmcg_plan_stats(const dmcg_plan* p, dmcg_stats* out) {
  if (!p || !out) return DMCG_E_CONFIG;
  *out = p->stats;
  return DMCG_OK;
}

int dmcg_ctx_stats(const dmcg_ctx* c, dmcg_stats* out) {
  if (!c || !out) return DMCG_E_CONFIG;
  *out = c->last_stats;
  return DMCG_OK;
}

void* dmcg_plan_stream(dmcg_plan* p) { return p ? (void*)p->ctx->stream : nullptr; }

int dmcg_plan_set_kernel_timing(dmcg_plan* p, int on) {
  if (!p) return DMCG_E_CONFIG;
  p->kernel_timing = on != 0;
  return DMCG_OK;
}

// ---- drop-in encode / decode -------------------------------------------------

// A pending decode plan may still have its factor in flight on aux2.
static void drop_pending_decode(dmcg_ctx* ctx) {
  if (!ctx->pending_dec) return;
  cudaStreamSynchronize(ctx->aux2);
  if (ctx->pending_dec->plan) dmcg_plan_destroy(ctx->pending_dec->plan);
  ctx->pending_dec.reset();
}

// The decode plan's config from a stream (dmcg_decode; the encode's
// pending decode plan uses the same function on its own output).
static Status decode_config(const dmcg_encoded* in, dmcg_config* cfg, std::vector<int>* rb) {
  const uint32_t nb = in->n_b > 1 ? in->n_b : 1;
  dmcg_config_default(cfg);
  cfg->variant = in->variant;
  cfg->k_l = in->k_l;
  cfg->n_b = (uint16_t)nb;
  rb->assign(in->k_l, 16);
  for (uint32_t r = 0; r < in->k_l; ++r) (*rb)[r] = in->row_bits[0][r];
  for (uint32_t r = 0; r < nb * in->k_l; ++r)
    for (int a = 0; a < 3; ++a)
      if (in->row_bits[a][r] < 1 || in->row_bits[a][r] > 16)
        return {DMCG_E_CORRUPT, "CorruptStream: row bit depth outside 1..16"};
  cfg->row_bits = rb->data();
  cfg->n_row_bits = in->k_l;
  cfg->anchor_bits = in->anchor_bits;
  cfg->dict_bits = in->dict_bits;
  cfg->diff_bits = in->diff_bits ? in->diff_bits : 8;
  return Status::ok();
}
int dmcg_encode(dmcg_ctx* ctx, const dmcg_seq* seq, const dmcg_config* cfg, dmcg_encoded* out) {
  if (!ctx || !seq || !cfg || !out) return DMCG_E_CONFIG;
  cudaSetDevice(ctx->device);
  PhaseTimer tm("encode");
  // Started below, once the mesh CSR exists: the decoder's analysis of this
  // mesh (normal matrix + symbolic Cholesky) on a host thread.  It needs only
  // the Laplacian structure and the anchor set (dmcg_select_anchors is a
  // function of n and the config), so it runs under the rest of the encode
  // (input H2D, plan, kernels, download).
  ctx->pending.reset();
  auto start_analysis = [&](const MeshHost& built) {
    static const bool off = std::getenv("DMCG_NO_OVERLAP") != nullptr;
    if (off || cfg->variant == DMCG_V2V || !seq->faces || !seq->n_faces || !seq->n) return;
    auto pa = std::make_unique<PendingAnalysis>();
    pa->n = seq->n;
    pa->n_faces = seq->n_faces;
    pa->faces_hash = hash_faces(seq->faces, seq->n_faces);
    pa->reduced = variant_uses_means(cfg->variant);
    if (!pa->reduced) {
      const uint32_t n_c = dmcg_anchor_count(seq->n, cfg->anchor_fraction);
      pa->anchors.resize(n_c);
      if (n_c == 0 || dmcg_select_anchors(seq->n, n_c, cfg->anchor_strategy, cfg->seed,
                                          pa->anchors.data()) != DMCG_OK)
        return;
    }
    // its own copy of the structure: the thread may outlive the encode plan
    pa->mesh.n = built.n;
    pa->mesh.lap_rp = built.lap_rp;
    pa->mesh.lap_ci = built.lap_ci;
    PendingAnalysis* raw = pa.get();
    pa->th = std::thread([raw] {
      const auto t0 = std::chrono::steady_clock::now();
      PhaseTimer ta("analysis-thread");
      MeshHost& m = raw->mesh;
      m.anchor_pos.assign(raw->n, -1);
      for (uint32_t t = 0; t < raw->anchors.size(); ++t)
        m.anchor_pos[raw->anchors[t]] = (int32_t)t;
      m.anchors = raw->anchors;
      if (raw->reduced) {
        build_reduced_normal(&m);
        ta.lap("normal matrix");
        chol_analyze(raw->n - 1, m.m_rp, m.m_ci, m.m_val, &raw->chol);
      } else {
        // the nested-dissection ordering needs only the 1-ring graph: it runs
        // (on its own threads) beside the normal-matrix build (host pool)
        CholOrdering ord;
        std::thread order_thread([&] { chol_order_graph(raw->n, m.lap_rp, m.lap_ci, &ord); });
        build_normal_matrix(&m);
        ta.lap("normal matrix");
        order_thread.join();
        ta.lap("ordering (rest)");
        chol_analyze(raw->n, m.m_rp, m.m_ci, m.m_val, &raw->chol, &m.lap_rp, &m.lap_ci, &ord);
      }
      ta.lap("chol_analyze");
      raw->seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
    ctx->pending = std::move(pa);
  };
  // The input upload goes first, into pool buffers: with pinned host memory
  // it runs on the copy engine while the host builds the mesh (CSR,
  // validation, anchors) for the plan below.
  const size_t in_bytes =
      (seq->n && seq->F) ? (size_t)seq->n * seq->F * (seq->dtype == DMCG_F32 ? 4 : 8) : 0;
  void* d_in[3] = {nullptr, nullptr, nullptr};
  struct InGuard {
    dmcg_ctx* c;
    void** d;
    size_t bytes;
    ~InGuard() {
      cudaStreamSynchronize(c->copy);
      cudaStreamSynchronize(c->stream);
      for (int a = 0; a < 3; ++a)
        if (d[a]) c->pool.put(d[a], bytes);
    }
  } in_guard{ctx, d_in, in_bytes};
  // On its own stream, axis by axis in 32 MB pieces with an event after each
  // axis: the plan's small (pageable) uploads slip between the pieces instead
  // of queueing behind a whole axis on the copy engine, and the encode starts
  // an axis' first kernels (K1, Gram) while the next axis is still in flight.
  if (in_bytes && seq->axes[0] && seq->axes[1] && seq->axes[2] &&
      (seq->dtype == DMCG_F64 || seq->dtype == DMCG_F32)) {
    bool ok = true;
    for (int a = 0; a < 3 && ok; ++a) {
      d_in[a] = ctx->pool.get(in_bytes);
      ok = d_in[a] != nullptr;
    }
    if (!ok) return ctx->set_error({DMCG_E_CUDA, "CudaError: device allocation failed"});
    auto issue_axis = [ctx, seq, in_bytes](void* dst, int a) {
      const size_t piece = (size_t)32 << 20;
      bool good = true;
      for (size_t off = 0; off < in_bytes && good; off += piece)
        good = cudaMemcpyAsync((uint8_t*)dst + off, (const uint8_t*)seq->axes[a] + off,
                               std::min(piece, in_bytes - off), cudaMemcpyHostToDevice,
                               ctx->copy) == cudaSuccess;
      return cudaEventRecord(ctx->ev_in[a], ctx->copy) == cudaSuccess && good;
    };
    // axis 0 now; axes 1 and 2 once the plan's uploads are queued (see
    // dmcg_ctx::after_plan_uploads), or below if no plan gets that far
    if (!issue_axis(d_in[0], 0)) return ctx->set_error({DMCG_E_CUDA, "CudaError: H2D copy failed"});
    void* d1 = d_in[1];
    void* d2 = d_in[2];
    ctx->after_plan_uploads = [issue_axis, d1, d2] {
      issue_axis(d1, 1);
      issue_axis(d2, 2);
    };
  }
  tm.lap("h2d issue");
  // One mesh build (host pool) serves the plan and the analysis thread; the
  // thread starts as soon as the CSR is there and then has the pool to itself
  // (the rest of plan creation is serial host work and uploads).
  // (Invalid input: plan_create_impl repeats the build and reports the error.)
  MeshHost built;
  const bool have_mesh = seq->faces && seq->n && seq->n_faces &&
                         build_mesh(seq->faces, seq->n_faces, seq->n, &built).good();
  tm.lap("mesh");
  if (have_mesh) start_analysis(built);
  dmcg_plan* p = nullptr;
  Status st = plan_create_impl(ctx, seq->n, seq->F, seq->dtype, seq->faces, seq->n_faces, cfg,
                               nullptr, 0, &p, have_mesh ? &built : nullptr);
  if (ctx->after_plan_uploads) {  // plan creation failed before its uploads
    ctx->after_plan_uploads();
    ctx->after_plan_uploads = nullptr;
  }
  if (!st.good()) return ctx->set_error(st);
  // the early analysis keys on the plan's anchor set: drop it if they differ
  if (ctx->pending && !std::equal(ctx->pending->anchors.begin(), ctx->pending->anchors.end(),
                                  p->mesh.anchors.begin(), p->mesh.anchors.end()))
    ctx->pending.reset();
  tm.lap("plan");
  // The next dmcg_decode of this stream -- its plan, decode structures and M's
  // numeric factor -- is prepared while the encode's kernels run: the host
  // waits for the analysis thread, uploads on the low-priority stream aux2 and
  // launches the factor there (it depends on mesh and anchors only, not on
  // anything the encode computes).  See PendingDecode.
  drop_pending_decode(ctx);
  static const bool no_prep = std::getenv("DMCG_NO_OVERLAP") || std::getenv("DMCG_NO_PREFACTOR");
  const std::function<void()> prepare_decode = [&] {
    if (no_prep || !ctx->pending || cfg->variant == DMCG_V2V || p->nb != 1) return;
    std::unique_ptr<PendingAnalysis> pa = std::move(ctx->pending);
    PhaseTimer tp("prepare-decode");
    if (pa->th.joinable()) pa->th.join();
    tp.lap("wait for the analysis");
    // what decode_config() will read from the stream this encode writes
    dmcg_config dc;
    dmcg_config_default(&dc);
    dc.variant = p->variant;
    dc.k_l = p->k_l;
    dc.n_b = 1;
    std::vector<int> drb(p->row_bits.begin(), p->row_bits.begin() + p->k_l);
    dc.row_bits = drb.data();
    dc.n_row_bits = p->k_l;
    dc.anchor_bits = p->anchor_bits;
    dc.dict_bits = p->dict_bits;
    dc.diff_bits = p->diff_bits ? p->diff_bits : 8;
    dmcg_plan* pdp = nullptr;
    const uint32_t no_anchor = 0;  // anchors "given" (empty) for the anchor-free variants
    Status sp = pa->failed ? Status{DMCG_E_CONFIG, "analysis failed"} : Status::ok();
    if (sp.good())
      sp = plan_create_impl(ctx, seq->n, seq->F, seq->dtype, seq->faces, seq->n_faces, &dc,
                            p->n_c ? p->mesh.anchors.data() : &no_anchor, p->n_c, &pdp,
                            &pa->mesh, false, ctx->aux2);
    if (sp.good()) {
      pdp->mesh.m_rp = std::move(pa->mesh.m_rp);
      pdp->mesh.m_ci = std::move(pa->mesh.m_ci);
      pdp->mesh.m_val = std::move(pa->mesh.m_val);
      pdp->chol = std::move(pa->chol);
      pdp->analyze_seconds = pa->seconds;
      pdp->chol_given = true;
      sp = plan_prepare_decode(pdp);
      pdp->up_stream = nullptr;  // the decode itself runs on the context stream
      if (sp.good()) sp = plan_prefactor_async(pdp, false);
    }
    if (sp.good()) {
      auto pd = std::make_unique<PendingDecode>();
      pd->plan = pdp;
      pd->n = seq->n;
      pd->F = seq->F;
      pd->n_faces = seq->n_faces;
      pd->faces_hash = pa->faces_hash;
      pd->dtype = seq->dtype;
      pd->variant = (int)p->variant;
      pd->k_l = p->k_l;
      pd->n_b = 1;
      pd->anchor_bits = (int)p->anchor_bits;
      pd->dict_bits = (int)p->dict_bits;
      pd->diff_bits = dc.diff_bits;
      pd->row_bits = drb;
      pd->anchors = p->mesh.anchors;
      ctx->pending_dec = std::move(pd);
    } else if (pdp) {
      cudaStreamSynchronize(ctx->aux2);
      dmcg_plan_destroy(pdp);
    }
    tp.lap("plan + uploads + factor launch");
  };
  // between the launches and the wait: the stream's D2H copies queued behind
  // the kernels (single-block streams; the blocks download reads pageable
  // staging and stays after the wait), then the decode preparation
  Status st_dl = Status::ok();
  const bool early_dl = p->nb == 1;
  const std::function<void()> between = [&] {
    // the preparation first: a D2H copy into pageable memory (small header
    // arrays of a caller that did not page-lock them) returns only once the
    // kernels ahead of it have run
    prepare_decode();
    if (early_dl) {
      if (!out->faces) out->faces = seq->faces;
      st_dl = download_issue(p, out);
      out->faces = seq->faces;
    }
  };
  p->in_events = true;
  if (early_dl && p->k > 0) {  // page-locked coefficient arrays: stream them per axis
    bool pinned = true;
    for (int a = 0; a < 3 && pinned; ++a) {
      cudaPointerAttributes at;
      pinned = out->coeff_q[a] && cudaPointerGetAttributes(&at, out->coeff_q[a]) == cudaSuccess &&
               at.type == cudaMemoryTypeHost;
    }
    cudaGetLastError();  // an unregistered pointer is not an error here
    if (pinned)
      for (int a = 0; a < 3; ++a) p->h_coeff_dst[a] = out->coeff_q[a];
  }
  if (st.good()) st = plan_encode(p, d_in, &between);
  tm.lap("h2d+kernels+download");
  if (st.good() && early_dl) {
    st = st_dl;
    if (st.good()) download_finish(p, out);
  } else if (st.good()) {
    if (!out->faces) out->faces = seq->faces;
    st = download_impl(p, out);
    out->faces = seq->faces;
  }
  tm.lap("download finish");
  if (!st.good()) drop_pending_decode(ctx);
  if (st.good()) {
    const dmcg_stats& e = p->stats;
    ctx->last_stats.ms_encode = e.ms_encode;
    ctx->last_stats.ms_delta = e.ms_delta;
    ctx->last_stats.ms_gram = e.ms_gram;
    ctx->last_stats.ms_basis = e.ms_basis;
    ctx->last_stats.ms_project = e.ms_project;
    ctx->last_stats.kernel_launches_encode = e.kernel_launches_encode;
    ctx->last_stats.ms_oi = e.ms_oi;
    ctx->last_stats.flops_oi = e.flops_oi;
  }
  dmcg_plan_destroy(p);
  return ctx->set_error(st);
}

int dmcg_decode(dmcg_ctx* ctx, const dmcg_encoded* in, const dmcg_decode_options* opt,
                void* const out_axes[3], int out_dtype) {
  if (!ctx || !in || !out_axes) return DMCG_E_CONFIG;
  cudaSetDevice(ctx->device);
  // Header sanity (the same bounds parse() enforces, stream.cpp:322-336).
  if (in->n < 1 || in->F < 1) return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: empty animation"});
  if (in->variant > DMCG_BLOCKS)
    return ctx->set_error({DMCG_E_UNSUPPORTED,
                           "Unsupported: only the variants pca, pca_q, v2v, pca_qs, pca_qp, blocks "
                           "are on the B200 path"});
  const uint32_t nb = in->n_b > 1 ? in->n_b : 1;
  if (nb > 1 && in->variant != DMCG_BLOCKS)
    return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: block count > 1 requires the blocks variant"});
  if (nb > 1 && (in->pad != (nb - in->F % nb) % nb))
    return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: padding does not match the block count"});
  if (nb > 1 && in->k_l > (in->F + in->pad) / nb)
    return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: retained row count exceeds dictionary dimension"});
  if (in->k_l > in->F)
    return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: retained row count exceeds dictionary dimension"});
  if (variant_uses_anchors(in->variant) ? (in->n_c < 1 || in->n_c > in->n) : in->n_c != 0)
    return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: anchor count out of range"});
  if (variant_uses_means(in->variant))
    for (int a = 0; a < 3; ++a)
      if (!in->means[a])
        return ctx->set_error({DMCG_E_CORRUPT, "CorruptPayload: missing frame means"});
  for (uint32_t t = 0; t < in->n_c; ++t)
    if (in->anchor_idx[t] >= in->n || (t && in->anchor_idx[t] <= in->anchor_idx[t - 1]))
      return ctx->set_error({DMCG_E_CORRUPT, "CorruptStream: anchor indices invalid"});
  dmcg_config cfg;
  std::vector<int> rb;
  {
    Status sc = decode_config(in, &cfg, &rb);
    if (!sc.good()) return ctx->set_error(sc);
  }
  dmcg_decode_options o;
  dmcg_decode_options_default(&o);
  if (opt) o = *opt;
  // The decode plan the last dmcg_encode prepared for its own stream (factor
  // already running on aux2), taken on an exact match of what it depends on.
  std::unique_ptr<PendingDecode> pd = std::move(ctx->pending_dec);
  if (pd && !(o.solver == 0 && pd->n == in->n && pd->F == in->F && pd->dtype == out_dtype &&
              pd->n_faces == in->n_faces && pd->variant == (int)in->variant &&
              pd->k_l == in->k_l && pd->n_b == nb && pd->anchor_bits == (int)in->anchor_bits &&
              pd->dict_bits == (int)in->dict_bits && pd->diff_bits == cfg.diff_bits &&
              pd->row_bits == rb && pd->anchors.size() == in->n_c &&
              std::equal(pd->anchors.begin(), pd->anchors.end(), in->anchor_idx) &&
              pd->faces_hash == hash_faces(in->faces, in->n_faces))) {
    // keep its host analysis (M, symbolic factor) when only the plan differs
    // (e.g. another output dtype): it depends on mesh and anchors alone
    if (pd->n == in->n && pd->n_faces == in->n_faces && pd->anchors.size() == in->n_c &&
        std::equal(pd->anchors.begin(), pd->anchors.end(), in->anchor_idx) &&
        variant_uses_means(pd->variant) == variant_uses_means(in->variant) &&
        pd->faces_hash == hash_faces(in->faces, in->n_faces) && !ctx->pending) {
      cudaStreamSynchronize(ctx->aux2);
      auto pa2 = std::make_unique<PendingAnalysis>();
      pa2->n = pd->n;
      pa2->n_faces = pd->n_faces;
      pa2->faces_hash = pd->faces_hash;
      pa2->reduced = variant_uses_means(pd->variant);
      pa2->anchors = pd->anchors;
      pa2->mesh = std::move(pd->plan->mesh);
      pa2->chol = std::move(pd->plan->chol);
      pa2->seconds = pd->plan->analyze_seconds;
      ctx->pending = std::move(pa2);
    }
    ctx->pending_dec = std::move(pd);
    drop_pending_decode(ctx);
  }
  // The analysis started by the last dmcg_encode (normal matrix, symbolic
  // Cholesky, and the Laplacian structure it was built from) is taken once,
  // and only when mesh and anchors match.
  std::unique_ptr<PendingAnalysis> pa = std::move(ctx->pending);
  if (pd) pa.reset();  // the prepared plan already holds it
  if (pa && !(pa->n == in->n && pa->n_faces == in->n_faces &&
              pa->reduced == variant_uses_means(in->variant) &&
              pa->anchors.size() == in->n_c &&
              std::equal(pa->anchors.begin(), pa->anchors.end(), in->anchor_idx) &&
              pa->faces_hash == hash_faces(in->faces, in->n_faces)))
    pa.reset();
  if (pa && pa->th.joinable()) pa->th.join();
  if (pa && pa->failed) pa.reset();
  dmcg_plan* p = pd ? pd->plan : nullptr;
  Status st = Status::ok();
  if (!p) {
    st = plan_create_impl(ctx, in->n, in->F, out_dtype, in->faces, in->n_faces, &cfg,
                          in->anchor_idx, in->n_c, &p, pa ? &pa->mesh : nullptr, false);
    if (!st.good()) return ctx->set_error(st);
  }
  PhaseTimer tm("decode");
  if (pa) {
    p->mesh.m_rp = std::move(pa->mesh.m_rp);
    p->mesh.m_ci = std::move(pa->mesh.m_ci);
    p->mesh.m_val = std::move(pa->mesh.m_val);
    p->chol = std::move(pa->chol);
    p->analyze_seconds = pa->seconds;
    p->chol_given = true;
  }
  tm.lap("plan");
  st = upload_impl(p, in, o.solver == 0 && !o.frame_count);
  tm.lap("upload");
  if (st.good() && o.solver == 0) st = plan_prepare_decode(p);
  tm.lap("prepare(analyze)");
  for (int a = 0; a < 3 && st.good(); ++a) {  // output staging (drop-in decode only)
    p->d_x_out[a] = plan_alloc(p, (size_t)in->n * in->F * (out_dtype == DMCG_F32 ? 4 : 8));
    if (!p->d_x_out[a]) st = {DMCG_E_CUDA, "CudaError: device allocation failed"};
  }
  // D2H of the decoded frame window only (all frames by default): columns
  // outside the window of the caller's arrays are left untouched.
  const size_t es = out_dtype == DMCG_F32 ? 4 : 8;
  auto d2h = [&](size_t f0, size_t fw, cudaStream_t cs) {
    for (int a = 0; a < 3 && st.good(); ++a)
      if (cudaMemcpy2DAsync((uint8_t*)out_axes[a] + f0 * es, in->F * es,
                            (const uint8_t*)p->d_x_out[a] + f0 * es, in->F * es, fw * es, in->n,
                            cudaMemcpyDeviceToHost, cs) != cudaSuccess)
        st = {DMCG_E_CUDA, "CudaError: D2H copy failed"};
  };
  // The whole sequence in two frame windows (the solve is column-separable:
  // each window decodes to the bits of the full decode, and the second reuses
  // the factor), so the first window's D2H runs under the second's kernels.
  static const bool no_split = std::getenv("DMCG_NO_DECODE_SPLIT") != nullptr;
  const bool split = !no_split && st.good() && o.solver == 0 && !o.frame_count && p->nb == 1 &&
                     in->F >= 64 && p->variant != DMCG_V2V;
  if (split) {
    static const int nwin_env = [] {
      const char* e = std::getenv("DMCG_DECODE_WINDOWS");
      return e ? std::max(2, std::min(8, std::atoi(e))) : 2;
    }();
    const uint32_t nwin = std::min<uint32_t>((uint32_t)nwin_env, in->F / 32);
    // two windows: the first one larger (in 64-frame steps), so that its D2H
    // (which hides under the second window's kernels) carries more of the
    // output and the exposed tail copy less
    static const int first_pct = [] {
      const char* e = std::getenv("DMCG_DECODE_FIRST_PCT");
      return e ? std::max(10, std::min(90, std::atoi(e))) : 75;
    }();
    // DMCG_DECODE_BOUNDS="f1,f2,...": explicit window boundaries (experiments)
    static const std::vector<uint32_t> env_bounds = [] {
      std::vector<uint32_t> v;
      if (const char* e = std::getenv("DMCG_DECODE_BOUNDS"))
        for (const char* q = e; *q;) {
          char* end = nullptr;
          const unsigned long x = std::strtoul(q, &end, 10);
          if (end == q) break;
          v.push_back((uint32_t)x);
          q = *end ? end + 1 : end;
        }
      return v;
    }();
    bool use_env = !env_bounds.empty() && env_bounds.back() < in->F;
    for (size_t i = 1; i < env_bounds.size(); ++i) use_env = use_env && env_bounds[i] > env_bounds[i - 1];
    // long sequences: three windows F/2 | F/2 - 64 | 64 frames (the copies of the
    // first two hide under kernels, the exposed tail copy is 64 frames; the
    // reconstruction's coefficient operand is sliced once, see rec_a_valid)
    const bool three = !use_env && nwin == 2 && in->F >= 512 && in->F % 128 == 0 &&
                       !std::getenv("DMCG_DECODE_FIRST_PCT") && !std::getenv("DMCG_DECODE_WINDOWS");
    const uint32_t nwin_eff = use_env ? (uint32_t)env_bounds.size() + 1 : (three ? 3u : nwin);
    auto bound = [&](uint32_t w) -> uint32_t {
      if (w == 0) return 0;
      if (w >= nwin_eff) return in->F;
      if (use_env) return env_bounds[w - 1];
      if (three) return w == 1 ? in->F / 2 : in->F - 64;
      if (nwin == 2 && in->F >= 256) {
        const uint32_t b = (uint32_t)((uint64_t)in->F * first_pct / 100 + 32) / 64 * 64;
        return std::max<uint32_t>(64, std::min<uint32_t>(b, in->F - 64));
      }
      return (uint32_t)((uint64_t)in->F * w / nwin);
    };
    for (uint32_t w = 0; w < nwin_eff && st.good(); ++w) {
      const uint32_t f0 = bound(w);
      const uint32_t f1 = bound(w + 1);
      dmcg_decode_options ow = o;
      ow.frame_begin = f0;
      ow.frame_count = f1 - f0;
      if (w) ow.reuse_factor = 1;
      st = plan_decode(p, &ow, p->d_x_out);  // returns after its stream sync
      tm.lap(w + 1 == nwin_eff ? "kernels (last window)" : "kernels (window)");
      if (st.good()) d2h(f0, f1 - f0, w + 1 == nwin_eff ? ctx->stream : ctx->aux2);
    }
    if (cudaStreamSynchronize(ctx->aux2) != cudaSuccess && st.good())
      st = {DMCG_E_CUDA, "CudaError: stream sync failed"};
  } else {
    if (st.good()) st = plan_decode(p, &o, p->d_x_out);
    tm.lap("kernels");
    const size_t f0 = o.frame_count ? o.frame_begin : 0;
    const size_t fw = o.frame_count ? o.frame_count : in->F;
    d2h(f0, fw, ctx->stream);
  }
  if (st.good() && cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    st = {DMCG_E_CUDA, "CudaError: stream sync failed"};
  tm.lap("d2h");
  if (st.good()) {  // keep the encode fields of the last dmcg_encode
    dmcg_stats e = ctx->last_stats;
    ctx->last_stats = p->stats;
    ctx->last_stats.ms_encode = e.ms_encode;
    ctx->last_stats.ms_delta = e.ms_delta;
    ctx->last_stats.ms_gram = e.ms_gram;
    ctx->last_stats.ms_basis = e.ms_basis;
    ctx->last_stats.ms_project = e.ms_project;
    ctx->last_stats.kernel_launches_encode = e.kernel_launches_encode;
    ctx->last_stats.ms_oi = e.ms_oi;
    ctx->last_stats.flops_oi = e.flops_oi;
  }
  dmcg_plan_destroy(p);
  return ctx->set_error(st);
}

// build_connectivity (src/mesh.cpp:60-86): sorted, deduplicated one-ring CSR.
// row_ptr: n + 1 entries; col: cap entries (cap >= 6 * n_faces always
// suffices); *nnz receives the neighbour count.  Errors as build_mesh, the
// message in dmcg_host_error().
static thread_local std::string g_host_error;
int dmcg_build_connectivity(const uint32_t* faces, uint32_t n_faces, uint32_t n, uint32_t* row_ptr,
                            uint32_t* col, size_t cap, size_t* nnz) {
  MeshHost m;
  Status st = build_mesh(faces, n_faces, n, &m);
  if (!st.good()) {
    g_host_error = st.msg;
    return st.code;
  }
  if (nnz) *nnz = m.adj_ci.size();
  if (m.adj_ci.size() > cap) {
    g_host_error = "DimensionMismatch: neighbour buffer too small";
    return DMCG_E_CONFIG;
  }
  std::copy(m.adj_rp.begin(), m.adj_rp.end(), row_ptr);
  std::copy(m.adj_ci.begin(), m.adj_ci.end(), col);
  return 0;
}
const char* dmcg_host_error(void) { return g_host_error.c_str(); }

}  // extern "C"

// ---- diagnostics ----------------------------------------------------------------
#include <chrono>

#include "chol.h"

extern "C" int dmcg_debug_chol(uint32_t n, const uint32_t* faces, uint32_t n_faces, uint32_t n_c,
                               const uint32_t* anchors, uint32_t W, const double* b, double* x,
                               double stats[8]) {
  MeshHost m;
  PhaseTimer tm("debug_chol");
  Status st = build_mesh(faces, n_faces, n, &m);
  if (!st.good()) return st.code;
  tm.lap("mesh");
  m.anchors.assign(anchors, anchors + n_c);
  m.anchor_pos.assign(n, -1);
  for (uint32_t t = 0; t < n_c; ++t) m.anchor_pos[anchors[t]] = (int32_t)t;
  build_normal_matrix(&m);
  tm.lap("normal");
  CholPlan p;
  const auto t0 = std::chrono::steady_clock::now();
  if (std::getenv("DMCG_DEBUG_PREORDER")) {  // the drop-in's split: ordering ahead of M
    CholOrdering ord;
    chol_order_graph(n, m.lap_rp, m.lap_ci, &ord);
    chol_analyze(n, m.m_rp, m.m_ci, m.m_val, &p, &m.lap_rp, &m.lap_ci, &ord);
  } else {
    chol_analyze(n, m.m_rp, m.m_ci, m.m_val, &p, &m.lap_rp, &m.lap_ci);
  }
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (stats) {
    stats[0] = p.nsup;
    stats[1] = p.nlevels;
    stats[2] = (double)p.nnz_l;
    stats[3] = p.flops_factor;
    stats[4] = p.flops_solve_per_rhs;
    stats[5] = p.max_front;
    stats[6] = p.max_width;
    stats[7] = secs;
    if (W == 0 && x) {  // memory footprint query: x[0..2] = sum m^2, sum w^2, sum m
      x[0] = (double)p.front_off[p.nsup];
      x[1] = (double)p.inv_off[p.nsup];
      x[2] = (double)p.rhs_off[p.nsup];
    }
  }
  if (const char* path = std::getenv("DMCG_DUMP_FRONTS")) {  // "level w m" per supernode
    if (FILE* f = std::fopen(path, "w")) {
      for (uint32_t l = 0; l + 1 < p.level_ptr.size(); ++l)
        for (uint32_t q = p.level_ptr[l]; q < p.level_ptr[l + 1]; ++q)
          std::fprintf(f, "%u %u %u\n", l, p.w(p.level_sup[q]), p.m(p.level_sup[q]));
      std::fclose(f);
    }
  }
  if (W > 0) {
    std::vector<double> F, Linv;
    if (!chol_factor_cpu(p, &F, &Linv)) return DMCG_E_NUMERICAL;
    chol_solve_cpu(p, F, Linv, W, b, x);
  }
  return DMCG_OK;
}
