// Internal host-side structures shared by host.cpp (C ABI, mesh / stream
// logic) and pipeline.cu (device orchestration).  Not installed.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dmcg.h"
#include "chol.h"
#include "chol_dev.h"

namespace dmcg {

// Variant predicates (include/dmc/stream.hpp:77-84).
inline bool variant_uses_anchors(int v) {
  return v == DMCG_PCA_QS || v == DMCG_PCA_QP || v == DMCG_BLOCKS;
}
inline bool variant_uses_means(int v) { return v == DMCG_PCA || v == DMCG_PCA_Q; }
inline bool variant_uses_delta(int v) { return v != DMCG_V2V; }

struct Status {
  int code = 0;
  std::string msg;
  static Status ok() { return {}; }
  bool good() const { return code == 0; }
};

// Caching device allocator owned by a context: blocks are recycled by size
// so repeated drop-in calls do not pay cudaMalloc (like a stream-ordered
// pool; all work of a context runs on its single stream).
class DevicePool {
 public:
  void* get(size_t bytes);
  void put(void* p, size_t bytes);
  void release_all();
  ~DevicePool() { release_all(); }

 private:
  std::multimap<size_t, void*> free_;
};

// Host-side mesh artefacts derived from the faces (reference src/mesh.cpp,
// src/laplacian.cpp, src/solver.cpp:25-39).
struct MeshHost {
  uint32_t n = 0;
  std::vector<uint32_t> adj_rp, adj_ci;   // one-ring CSR (sorted, dedup)
  std::vector<uint32_t> lap_rp, lap_ci;   // Laplacian structure incl. diagonal
  std::vector<uint32_t> m_rp, m_ci;       // M = L^T L + S^T S
  std::vector<float> m_val;
  std::vector<uint32_t> anchors;
  std::vector<int32_t> anchor_pos;        // vertex -> anchor slot or -1
};

Status build_mesh(const uint32_t* faces, uint32_t n_faces, uint32_t n, MeshHost* out);
Status validate_mesh(const MeshHost& m);   // isolated / connected (mesh.cpp:108-136)
void build_normal_matrix(MeshHost* m);     // needs anchors set
// (L^T L)[1:, 1:]: the normal matrix of solve_mean_constrained
// (solver.cpp:116-117), n - 1 rows (vertex i at row i - 1).
void build_reduced_normal(MeshHost* m);

}  // namespace dmcg

struct dmcg_plan;
namespace dmcg {
// Host phase timer, printed to stderr when DMCG_TIMING is set.
struct PhaseTimer {
  const char* scope;
  bool on;
  double t0;
  explicit PhaseTimer(const char* s);
  void lap(const char* what);
};
// Device allocation owned by the plan (returned to the context pool on destroy).
void* plan_alloc(dmcg_plan* p, size_t bytes);
// Builds the decode-side state on first use (host.cpp).
Status plan_prepare_decode(dmcg_plan* p);
// M's numeric factor on ctx->aux2 now (decode structures must exist); the
// next decode of the plan takes it and waits for it before its solves.
Status plan_prefactor_async(dmcg_plan* p, bool after_stream = true);
Status plan_prepare_normal(dmcg_plan* p);
}  // namespace dmcg

namespace dmcg {
// The decoder's host analysis (normal matrix M = L^T L + S^T S and the
// symbolic Cholesky of M) depends only on the mesh and the anchor set, both
// known when dmcg_encode starts.  The drop-in encode therefore runs it on a
// host thread while its GPU work executes; the next dmcg_decode on the same
// mesh and anchors takes the result (once) instead of recomputing it.
struct PendingAnalysis {
  uint32_t n = 0, n_faces = 0;
  bool reduced = false;  // (L^T L)[1:, 1:] of the anchor-free variants, else L^T L + S^T S
  uint64_t faces_hash = 0;
  std::vector<uint32_t> anchors;
  MeshHost mesh;    // lap_rp / lap_ci / anchor_pos in, m_rp / m_ci / m_val out
  CholPlan chol;
  double seconds = 0.0;
  bool failed = false;  // the mesh did not validate (the encode reports it)
  std::thread th;
  ~PendingAnalysis() {
    if (th.joinable()) th.join();
  }
};
uint64_t hash_faces(const uint32_t* faces, uint32_t n_faces);

// Byte offsets of the bit-packed payload sections of a DMC1 stream.
struct PayloadSpans {
  size_t dict[3], coeff[3], anchor[3];
};
size_t serialize_stream(const dmcg_encoded* e, uint8_t* out, size_t cap, dmcg_sections* s,
                        PayloadSpans* spans);
}  // namespace dmcg

namespace dmcg {
// The decode plan a drop-in dmcg_encode prepares for the next dmcg_decode of
// its own stream: created from the stream's config once the overlapped
// analysis is done, decode structures uploaded, and M's numeric factor
// launched on ctx->aux2 — so the factor runs while the encode returns and the
// decode uploads the stream and reconstructs.  Taken once, only on an exact
// match of everything the decode plan depends on; otherwise discarded.
struct PendingDecode {
  dmcg_plan* plan = nullptr;
  uint32_t n = 0, F = 0, n_faces = 0, k_l = 0, n_b = 0;
  int dtype = 0, variant = 0, anchor_bits = 0, dict_bits = 0, diff_bits = 0;
  uint64_t faces_hash = 0;
  std::vector<int> row_bits;
  std::vector<uint32_t> anchors;
};
}  // namespace dmcg

struct dmcg_ctx {
  int device = 0;
  std::unique_ptr<dmcg::PendingAnalysis> pending;  // see PendingAnalysis
  std::unique_ptr<dmcg::PendingDecode> pending_dec;  // see PendingDecode
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;  // fork/join side stream (independent encode / decode phases)
  cudaStream_t aux2 = nullptr; // low-priority stream: the decoder's factor during an encode
  cudaStream_t copy = nullptr; // the drop-in encode's input H2D (chunked, one event per axis)
  cudaEvent_t ev_in[3] = {nullptr, nullptr, nullptr};  // axis a of the input has arrived
  cudaEvent_t ev_q[3] = {nullptr, nullptr, nullptr};   // axis a's coefficient symbols are quantised
  cudaEvent_t ev_cp = nullptr;                         // the copy stream's D2H of them is done
  // run once by the next plan creation right after it has issued its uploads
  // (the drop-in encode queues input axes 1 and 2 there: queued earlier they
  // would hold the copy engine's FIFO ahead of the plan's small uploads)
  std::function<void()> after_plan_uploads;
  std::string err;
  dmcg::DevicePool pool;
  dmcg_stats last_stats = {};  // stats of the last drop-in encode / decode
  // CUDA events recycled across the plans of this context (timing events,
  // and fork / join events without timing): creating ~10 events per drop-in
  // call costs ~0.1 ms of host time.
  std::vector<cudaEvent_t> ev_timing, ev_plain;
  cudaEvent_t take_event(bool timing) {
    auto& v = timing ? ev_timing : ev_plain;
    if (!v.empty()) {
      cudaEvent_t e = v.back();
      v.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
    return e;
  }
  void give_event(cudaEvent_t e, bool timing) {
    if (e) (timing ? ev_timing : ev_plain).push_back(e);
  }
  int set_error(const dmcg::Status& s) {
    err = s.msg;
    return s.code;
  }
};

namespace dmcg {
// An instantiated CUDA graph of one plan call, keyed by the caller's
// pointers / options (pipeline.cu run_graph).
struct PlanGraph {
  cudaGraphExec_t exec = nullptr;
  const void* key[4] = {nullptr, nullptr, nullptr, nullptr};
  long long opt_key = 0;
};
}  // namespace dmcg

struct dmcg_comm;  // NCCL communicator (shard.cpp)
namespace dmcg {
// Vertex-row shard of one large sequence.  Rank q owns the
// contiguous rows [r0[q], r0[q+1]); its local input holds those rows
// followed by the halo rows (one-ring neighbours owned by other ranks) that
// K1 needs.  The local Laplacian CSR keeps each row's global column order, so
// the shard's delta rows equal the single-GPU rows bit for bit.
struct ShardState {
  int nranks = 1, rank = 0;
  std::vector<uint32_t> r0;                  // nranks + 1 row boundaries
  std::vector<uint32_t> a0;                  // nranks + 1 anchor-slot boundaries
  std::vector<unsigned long long> stage_off; // nranks + 1 offsets (u16) into the gather buffer
  uint32_t n_own = 0, n_loc = 0;
  std::vector<uint32_t> halo;                // global ids of local rows n_own..n_loc-1
  std::vector<uint32_t> loc_rp, loc_ci;      // local CSR of the owned rows
  uint32_t* d_loc_rp = nullptr;
  uint32_t* d_loc_ci = nullptr;
  uint32_t* d_loc_anchor = nullptr;          // local rows of the owned anchors
  unsigned long long* d_keys = nullptr;      // (3 k + 3) x (min, max) ordered keys
  uint16_t* d_gather = nullptr;              // every rank's symbols (rank q at stage_off[q])
  dmcg_comm* comm = nullptr;                 // not owned
};
// Row split, halo and local CSR of rank `rank` (needs m.lap_* and m.anchors).
void shard_layout(const MeshHost& m, uint32_t F, uint32_t k, int nranks, int rank,
                  ShardState* out);
// Collectives on the plan stream (NCCL, shard.cpp).
Status comm_allreduce_sum_f64(dmcg_comm* c, double* buf, size_t count, cudaStream_t s);
Status comm_allreduce_max_u64(dmcg_comm* c, unsigned long long* buf, size_t count,
                              cudaStream_t s);
// Every rank q broadcasts buf[off[q] .. off[q+1]) (u16) in place to all ranks.
Status comm_allgatherv_u16(dmcg_comm* c, uint16_t* buf, const unsigned long long* off,
                           cudaStream_t s);
int comm_size(const dmcg_comm* c);
int comm_rank(const dmcg_comm* c);
}  // namespace dmcg

struct dmcg_plan {
  dmcg_ctx* ctx = nullptr;
  std::unique_ptr<dmcg::ShardState> shard;  // vertex-row shard plans only
  // geometry / config
  uint32_t n = 0, F = 0, k = 0, n_c = 0, n_faces = 0;
  int dtype = DMCG_F64;
  int rounds = 0;
  int anchor_bits = 16, dict_bits = 16, diff_bits = 8;
  uint64_t oi_seed = 0;
  int variant = DMCG_PCA_QP;        // pca / pca_q / v2v / pca_qs / pca_qp
  bool implicit = false;            // dmcg_config.oi_implicit
  std::vector<int> row_bits;
  std::vector<uint32_t> faces;
  dmcg::MeshHost mesh;
  uint32_t W = 0, W_pad = 0, nblk = 0;   // CG columns (3F), padded to kCB

  // device buffers (owned; returned to ctx->pool on destroy)
  std::vector<std::pair<void*, size_t>> owned;
  uint32_t *d_lap_rp = nullptr, *d_lap_ci = nullptr;
  uint32_t *d_m_rp = nullptr, *d_m_ci = nullptr;
  float* d_m_val = nullptr;
  uint32_t* d_anchor_idx = nullptr;
  int32_t* d_anchor_pos = nullptr;
  void* d_x_out[3] = {nullptr, nullptr, nullptr};  // output staging of the drop-in decode
  double* d_delta = nullptr;       // 3 x n x F
  double* d_R = nullptr;           // 3 x F x F
  double* d_part = nullptr;        // split-K partials
  size_t part_elems = 0;
  // Ozaki INT8 tensor-core Gram (ozaki.h; f32 storage, n_b = 1): the s
  // slices of X (rows = frames, K = vertex rows) and their row maxima
  int oz_slices = 0;               // 0: DMMA Gram
  int oz_proj_slices = 0;          // Ozaki projection U_k^T delta^T (0: DMMA)
  int oz_rec_slices = 0;           // Ozaki reconstruction U~ c~ (0: DMMA)
  size_t oz_q_bytes = 0;           // d_oz_q capacity
  size_t oz_max_elems = 0;         // d_oz_max capacity
  int8_t* d_oz_q = nullptr;        // 3 x s x F_pad x n_pad
  unsigned long long* d_oz_max = nullptr;  // 3 x F_pad
  double* d_U = nullptr;           // 3 x F x F (col-major)
  double* d_evals = nullptr;       // 3 x F
  double *d_Q = nullptr, *d_Z = nullptr, *d_tau = nullptr;  // 3 x F x k, 3 x F
  double *d_H = nullptr, *d_V = nullptr, *d_w = nullptr;    // jacobi work (3 x m2 x m2)
  double* d_qr_scr = nullptr;      // 3 x qr_scratch_doubles(F, k) blocked-QR scratch
  double* d_oi_mirror = nullptr;   // oi_mirror_doubles(F, 3): published OI block reflectors
  double* d_start = nullptr;       // 3 x F x k OI start matrices
  double* d_C = nullptr;           // 3 x k x n coefficients
  unsigned long long* d_keys = nullptr;  // 3 x k x 2 (min,max) ordered keys
  int* d_flags = nullptr;          // [0] non-finite axes mask, [1] corrupt payload, [2] cg fail
  // encoded (device-resident)
  uint16_t* d_dict_q = nullptr;    // 3 x F x F
  float *d_row_min = nullptr, *d_row_max = nullptr;  // 3 x k
  uint8_t* d_row_bits = nullptr;   // 3 x k
  uint16_t* d_coeff_q = nullptr;   // 3 x k x n
  float* d_anchor_rng = nullptr;   // 3 x 2
  float* d_means = nullptr;        // 3 x F per-frame vertex means (pca / pca_q)
  double* d_colsum = nullptr;      // column-sum partials (3 x 64 x 3F) of the means / shift
  uint16_t* d_anchor_q = nullptr;  // 3 x n_c x F
  // decode
  double* d_rowp = nullptr;        // 3 x k x 2 (min_, width) dequantiser params
  double* d_Ud = nullptr;          // 3 x k x F dequantised dictionary columns (decode)
  uint32_t* d_stream = nullptr;    // device DMC1 image for dmcg_plan_serialize
  double* d_metric = nullptr;      // 3 n F + F + F + n doubles (dmcg_plan_distortion)
  size_t stream_cap = 0;
  unsigned long long* d_row_bitoff = nullptr;  // 3 x k payload bit offsets
  double *d_cg_x = nullptr, *d_cg_r = nullptr, *d_cg_p = nullptr, *d_cg_q = nullptr;
  int* d_cg_iters = nullptr;       // per column
  double* d_cg_res = nullptr;      // per column relative residual
  // direct solver (supernodal Cholesky, chol.h)
  dmcg::CholPlan chol;
  dmcg::CholLevels levels;
  dmcg::CholDev cdev;
  double *d_rm_delta = nullptr, *d_rm_b = nullptr, *d_rm_x = nullptr;  // n x 3F, original order
  double *d_rm_y = nullptr, *d_rm_xp = nullptr, *d_rm_r = nullptr;     // permuted / residual
  double analyze_seconds = 0.0;
  bool decode_ready = false;
  bool chol_given = false;
  bool factor_valid = false;        // cdev.F / Linv hold the numeric factor of M          // chol / mesh.m_* were filled by a PendingAnalysis
  bool oi_timed = false;            // ev[6..7] bracket k_oi_fused in the last encode
  float h_anchor_rng[6] = {};        // download staging (anchor ranges)
  // drop-in encode: the input axes arrive on ctx->copy; the encode waits for
  // ctx->ev_in[a] before the first kernel that reads axis a
  bool in_events = false;
  // drop-in encode with page-locked output arrays: axis a's coefficient
  // symbols go to h_coeff_dst[a] on ctx->copy as soon as they are quantised
  // (per-axis projection + quantisation), under the next axes' kernels
  void* h_coeff_dst[3] = {nullptr, nullptr, nullptr};
  // the reconstruction's A operand (dequantised coefficients, their Ozaki
  // slices) is still in place from an earlier frame window of the same stream
  bool rec_a_valid = false;
  // drop-in decode from page-locked arrays: axis a's coefficient symbols arrive
  // on ctx->copy (event ctx->ev_in[a]); the first reconstruction waits per axis
  bool coeff_events = false;
  bool coeff_streamed = false;  // set by the encode when it did so (download skips them)
  cudaStream_t up_stream = nullptr;  // plan / decode-structure uploads (default: aux / ctx stream)
  bool use_graphs = false;          // reused plans replay CUDA graphs (dmcg_plan_create)
  dmcg::PlanGraph g_encode, g_decode;

  // blocks variant (n_b > 1, codec.cpp:149-172, 290-349): F above is the
  // padded frame count F_in + pad = nb * kf, k = nb * k_l coefficient rows
  // per axis (block b at rows [b k_l, (b+1) k_l)); d_R / d_U / d_dict_q hold
  // the nb per-block k_f x k_f matrices of each axis back to back.
  uint32_t nb = 1, kf = 0, k_l = 0, F_in = 0, pad = 0;
  int t_max = 4;
  double oi_tol = -1.0;
  double* d_bUeig = nullptr;       // 3 x nb x kf^2 eigenbases of every block
  double* d_bwork = nullptr;       // 3 x block_work_doubles(kf)
  double* d_bUd = nullptr;         // 3 x nb x kf^2 decoded dictionaries
  float* d_diff_rng = nullptr;     // 3 x (nb - 1) x 2 difference ranges
  void* d_xpad = nullptr;          // 3 x n x F padded input (pad > 0)
  int oi_fallbacks = 0;            // blocks that fell back to full_eigenbasis (last encode)

  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // ctx->stream <-> ctx->aux
  bool forked = false;
  // Decoder factor overlapped with the encode (pipeline.cu prefactor_on):
  // M = L^T L + S^T S depends only on the mesh and the plan's anchor set, so
  // once the decode structures exist an encode factors M on ctx->aux2 while
  // its own latency-bound basis phase leaves most SMs idle; the next decode
  // takes that factor instead of refactoring.
  cudaEvent_t ev_pf_fork = nullptr, ev_pf_join = nullptr, ev_pf0 = nullptr, ev_pf1 = nullptr;
  int* d_pf_flag = nullptr;        // non-positive pivot of the overlapped factor
  bool factor_pending = false;     // the last encode left a factor of M for the next decode
  bool pf_unjoined = false;        // ... launched outside any graph: the decode waits ev_pf_join
  bool kernel_timing = false;      // dmcg_plan_set_kernel_timing
  std::vector<cudaEvent_t> solve_ev;  // (1 + refine) x 4 nlevels timing events
  float ms_prefactor = 0.0f;
  dmcg_stats stats = {};
};
