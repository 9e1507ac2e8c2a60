// Multi-GPU: vertex-row shards of one large sequence and the
// NCCL communicator they use.
//
// One process per GPU.  Rank q owns the contiguous vertex rows
// [q n / N, (q+1) n / N) (the generators number vertices in spatially
// coherent order, so a row block is a compact patch and its halo is thin).
// Encode per rank: K1 delta of the owned rows from the local input (owned +
// halo rows), the partial Gram of the owned rows, then
//   ncclAllReduce(sum) of the 3 F x F partials (the Gram is a sum over
//   vertices: src/spectral.cpp:37),
// the basis on every rank (replicated: NCCL leaves identical bits on every
// rank), the projection of the owned rows and their per-row min / max keys,
//   ncclAllReduce(max) of the (3 k + 3) key pairs (row ranges of
//   quantize_rows, codec.cpp:253, and the anchor range, codec.cpp:449-455),
// quantisation of the owned rows / anchors, and
//   grouped ncclBroadcast of every rank's symbols (an all-gather with
//   per-rank counts), so every rank holds the whole stream for decode.
// Decode splits frames across ranks instead (dmcg_decode_options frame
// window: the anchored solve is column-separable), so it needs no exchange.
//
// NCCL is loaded with dlopen at first use (libnccl.so.2: the copy torch has
// already loaded, else the system one) so libdmcg itself has no link-time
// NCCL dependency; a missing NCCL is reported by dmcg_comm_create.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.h"

struct dmcg_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

namespace dmcg {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("NCCL not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))sym("ncclAllReduce");
    api.broadcast = (decltype(api.broadcast))sym("ncclBroadcast");
    api.groupStart = (decltype(api.groupStart))sym("ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))sym("ncclGroupEnd");
    api.errorString = (decltype(api.errorString))sym("ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce &&
             api.broadcast && api.groupStart && api.groupEnd && api.errorString;
    if (!api.ok) api.why = "NCCL library lacks a required symbol";
  });
  return api;
}

Status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return Status::ok();
  return {DMCG_E_CUDA, std::string("NcclError: ") + what + ": " + nccl().errorString(r)};
}

}  // namespace

void shard_layout(const MeshHost& m, uint32_t F, uint32_t k, int nranks, int rank,
                  ShardState* out) {
  ShardState& sh = *out;
  const uint32_t n = m.n;
  sh.nranks = nranks;
  sh.rank = rank;
  sh.r0.assign(nranks + 1, 0);
  sh.a0.assign(nranks + 1, 0);
  for (int q = 0; q <= nranks; ++q) {
    sh.r0[q] = (uint32_t)((unsigned long long)n * q / nranks);
    sh.a0[q] = (uint32_t)(std::lower_bound(m.anchors.begin(), m.anchors.end(), sh.r0[q]) -
                          m.anchors.begin());
  }
  sh.stage_off.assign(nranks + 1, 0);
  for (int q = 0; q < nranks; ++q)
    sh.stage_off[q + 1] = sh.stage_off[q] + 3ull * k * (sh.r0[q + 1] - sh.r0[q]) +
                          3ull * (sh.a0[q + 1] - sh.a0[q]) * F;
  const uint32_t b = sh.r0[rank], e = sh.r0[rank + 1];
  sh.n_own = e - b;
  sh.halo.clear();
  for (uint32_t i = b; i < e; ++i)
    for (uint32_t p = m.lap_rp[i]; p < m.lap_rp[i + 1]; ++p)
      if (m.lap_ci[p] < b || m.lap_ci[p] >= e) sh.halo.push_back(m.lap_ci[p]);
  std::sort(sh.halo.begin(), sh.halo.end());
  sh.halo.erase(std::unique(sh.halo.begin(), sh.halo.end()), sh.halo.end());
  sh.n_loc = sh.n_own + (uint32_t)sh.halo.size();
  // Local CSR: same entries in the same (global column) order, renumbered.
  sh.loc_rp.assign(sh.n_own + 1, 0);
  sh.loc_ci.clear();
  sh.loc_ci.reserve(m.lap_rp[e] - m.lap_rp[b]);
  for (uint32_t i = b; i < e; ++i) {
    for (uint32_t p = m.lap_rp[i]; p < m.lap_rp[i + 1]; ++p) {
      const uint32_t j = m.lap_ci[p];
      if (j >= b && j < e)
        sh.loc_ci.push_back(j - b);
      else
        sh.loc_ci.push_back(sh.n_own + (uint32_t)(std::lower_bound(sh.halo.begin(),
                                                                   sh.halo.end(), j) -
                                                  sh.halo.begin()));
    }
    sh.loc_rp[i - b + 1] = (uint32_t)sh.loc_ci.size();
  }
}

Status comm_allreduce_sum_f64(dmcg_comm* c, double* buf, size_t count, cudaStream_t s) {
  if (c->nranks == 1) return Status::ok();
  return nccl_status(nccl().allReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, s),
                     "allreduce(sum)");
}

Status comm_allreduce_max_u64(dmcg_comm* c, unsigned long long* buf, size_t count,
                              cudaStream_t s) {
  if (c->nranks == 1) return Status::ok();
  return nccl_status(nccl().allReduce(buf, buf, count, ncclUint64, ncclMax, c->comm, s),
                     "allreduce(max)");
}

Status comm_allgatherv_u16(dmcg_comm* c, uint16_t* buf, const unsigned long long* off,
                           cudaStream_t s) {
  if (c->nranks == 1) return Status::ok();
  const NcclApi& api = nccl();
  Status st = nccl_status(api.groupStart(), "group start");
  for (int q = 0; q < c->nranks && st.good(); ++q)
    st = nccl_status(api.broadcast(buf + off[q], buf + off[q], (off[q + 1] - off[q]) * 2,
                                   ncclUint8, q, c->comm, s),
                     "broadcast");
  Status ge = nccl_status(api.groupEnd(), "group end");
  return st.good() ? ge : st;
}

int comm_size(const dmcg_comm* c) { return c->nranks; }
int comm_rank(const dmcg_comm* c) { return c->rank; }

Status shard_encode(dmcg_plan* p, const void* const x[3]);        // pipeline.cu
Status shard_phase(dmcg_plan* p, int phase, const void* const x[3]);

}  // namespace dmcg

using dmcg::Status;

extern "C" {

int dmcg_comm_unique_id(uint8_t id[128]) {
  const auto& api = dmcg::nccl();
  if (!api.ok) return DMCG_E_UNSUPPORTED;
  ncclUniqueId u;
  if (api.getUniqueId(&u) != ncclSuccess) return DMCG_E_CUDA;
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return DMCG_OK;
}

int dmcg_comm_create(int device, const uint8_t id[128], int nranks, int rank, dmcg_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return DMCG_E_CONFIG;
  *out = nullptr;
  auto* c = new dmcg_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (nranks > 1) {  // a one-rank job needs no communicator (collectives are identities)
    const auto& api = dmcg::nccl();
    if (!api.ok) {
      delete c;
      return DMCG_E_UNSUPPORTED;
    }
    cudaSetDevice(device);
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (api.commInitRank(&c->comm, nranks, u, rank) != ncclSuccess) {
      delete c;
      return DMCG_E_CUDA;
    }
  }
  *out = c;
  return DMCG_OK;
}

void dmcg_comm_destroy(dmcg_comm* c) {
  if (!c) return;
  if (c->comm) dmcg::nccl().commDestroy(c->comm);
  delete c;
}

static void fill_info(const dmcg::ShardState& sh, dmcg_shard_info* info, uint32_t* halo) {
  if (info) {
    info->nranks = sh.nranks;
    info->rank = sh.rank;
    info->row_begin = sh.r0[sh.rank];
    info->row_end = sh.r0[sh.rank + 1];
    info->n_own = sh.n_own;
    info->n_halo = (uint32_t)sh.halo.size();
    info->n_loc = sh.n_loc;
    info->anchor_begin = sh.a0[sh.rank];
    info->anchor_end = sh.a0[sh.rank + 1];
    info->stage_begin = sh.stage_off[sh.rank];
    info->stage_count = sh.stage_off[sh.rank + 1] - sh.stage_off[sh.rank];
    info->gather_count = sh.stage_off[sh.nranks];
  }
  if (halo && !sh.halo.empty()) std::memcpy(halo, sh.halo.data(), sh.halo.size() * 4);
}

int dmcg_shard_layout(uint32_t n, uint32_t F, const uint32_t* faces, uint32_t n_faces,
                      const dmcg_config* cfg, int nranks, int rank, dmcg_shard_info* info,
                      uint32_t* halo) {
  if (!faces || !cfg || nranks < 1 || rank < 0 || rank >= nranks || n < (uint32_t)nranks)
    return DMCG_E_CONFIG;
  dmcg::MeshHost m;
  Status st = dmcg::build_mesh(faces, n_faces, n, &m);
  if (!st.good()) return st.code;
  const uint32_t n_c = dmcg_anchor_count(n, cfg->anchor_fraction);
  m.anchors.resize(n_c);
  if (dmcg_select_anchors(n, n_c, cfg->anchor_strategy, cfg->seed, m.anchors.data()))
    return DMCG_E_CONFIG;
  dmcg::ShardState sh;
  dmcg::shard_layout(m, F, cfg->k_l, nranks, rank, &sh);
  fill_info(sh, info, halo);
  return DMCG_OK;
}

int dmcg_shard_info_get(const dmcg_plan* p, dmcg_shard_info* info, uint32_t* halo) {
  if (!p || !p->shard) return DMCG_E_CONFIG;
  fill_info(*p->shard, info, halo);
  return DMCG_OK;
}

int dmcg_shard_encode_device(dmcg_plan* p, const void* const d_loc_axes[3]) {
  if (!p || !p->shard || !d_loc_axes) return DMCG_E_CONFIG;
  if (!p->shard->comm)
    return p->ctx->set_error({DMCG_E_CONFIG, "ConfigError: shard plan has no communicator"});
  cudaSetDevice(p->ctx->device);
  return p->ctx->set_error(dmcg::shard_encode(p, d_loc_axes));
}

int dmcg_shard_encode_phase(dmcg_plan* p, int phase, const void* const d_loc_axes[3]) {
  if (!p || !p->shard || phase < 0 || phase > 3) return DMCG_E_CONFIG;
  cudaSetDevice(p->ctx->device);
  return p->ctx->set_error(dmcg::shard_phase(p, phase, d_loc_axes));
}

int dmcg_shard_buffer(dmcg_plan* p, int which, void** dptr, size_t* count) {
  if (!p || !p->shard || !dptr || !count) return DMCG_E_CONFIG;
  const dmcg::ShardState& sh = *p->shard;
  switch (which) {
    case DMCG_SHARD_GRAM:
      *dptr = p->d_R;
      *count = 3ull * p->F * p->F;
      return DMCG_OK;
    case DMCG_SHARD_KEYS:
      *dptr = sh.d_keys;
      *count = (3ull * p->k + 3) * 2;
      return DMCG_OK;
    case DMCG_SHARD_SYMBOLS:
      *dptr = sh.d_gather;
      *count = sh.stage_off[sh.nranks];
      return DMCG_OK;
    default:
      return DMCG_E_CONFIG;
  }
}

}  // extern "C"
