// DMC1 wire format for the pca_qp / n_b = 1 path: serialize, strict parse
// and exact rate accounting.  Reference: src/stream.cpp:172-469 (format and
// checks), src/quantize.cpp:50-87 (MSB-first bit packing), src/metrics.cpp:
// 46-59 (rate_exact).  Bit packing here works a byte / 64-bit word at a time
// instead of the reference's bit-at-a-time loop; the bytes are identical.
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace {

struct ByteOut {
  uint8_t* o;
  size_t cap, pos = 0;
  bool overflow = false;
  void u8(uint8_t v) {
    if (o) {
      if (pos < cap)
        o[pos] = v;
      else
        overflow = true;
    }
    ++pos;
  }
  void u16(uint16_t v) {
    u8((uint8_t)v);
    u8((uint8_t)(v >> 8));
  }
  void u32(uint32_t v) {
    for (int i = 0; i < 4; ++i) u8((uint8_t)(v >> (8 * i)));
  }
  void f32(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    u32(u);
  }
};

// BitWriter (quantize.cpp:50-69): MSB first, final partial byte zero padded.
struct BitOut {
  ByteOut& w;
  uint64_t acc = 0;
  int fill = 0;
  explicit BitOut(ByteOut& bw) : w(bw) {}
  void put(uint32_t v, int bits) {
    acc = (acc << bits) | (v & ((1u << bits) - 1u));
    fill += bits;
    while (fill >= 8) {
      fill -= 8;
      w.u8((uint8_t)(acc >> fill));
    }
  }
  void flush() {
    if (fill > 0) w.u8((uint8_t)(acc << (8 - fill)));
    fill = 0;
    acc = 0;
  }
};

struct ByteIn {
  const uint8_t* d;
  size_t size, pos = 0;
  std::string err;
  bool need(size_t c) {
    if (size - pos < c) {
      if (err.empty()) err = "unexpected end of stream at byte " + std::to_string(pos);
      return false;
    }
    return true;
  }
  uint8_t u8() { return need(1) ? d[pos++] : 0; }
  uint16_t u16() {
    if (!need(2)) return 0;
    uint16_t v = (uint16_t)(d[pos] | (d[pos + 1] << 8));
    pos += 2;
    return v;
  }
  uint32_t u32() {
    if (!need(4)) return 0;
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)d[pos + i] << (8 * i);
    pos += 4;
    return v;
  }
  float f32() {
    uint32_t u = u32();
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  const uint8_t* slice(size_t c) {
    if (!need(c)) return nullptr;
    const uint8_t* p = d + pos;
    pos += c;
    return p;
  }
};

// BitReader over an exact byte span (quantize.cpp:71-87).
void unpack(const uint8_t* src, size_t count, int bits, uint16_t* out) {
  uint64_t acc = 0;
  int fill = 0;
  size_t pos = 0;
  const uint32_t mask = (1u << bits) - 1u;
  for (size_t t = 0; t < count; ++t) {
    while (fill < bits) {
      acc = (acc << 8) | src[pos++];
      fill += 8;
    }
    fill -= bits;
    out[t] = (uint16_t)((acc >> fill) & mask);
  }
}

size_t packed_bytes(size_t count, int bits) { return (count * (size_t)bits + 7) / 8; }

// Skips `bytes` payload bytes (their content is written elsewhere).
void skip(ByteOut& w, size_t bytes) {
  if (w.o && w.pos + bytes > w.cap) w.overflow = true;
  w.pos += bytes;
}

}  // namespace

// Writes the DMC1 stream of e.  With spans == nullptr the payload sections
// (dictionary, coefficient and anchor levels) are bit-packed here; otherwise
// they are only sized and their byte offsets reported in spans (the GPU
// packer fills them: dmcg_plan_serialize).
size_t dmcg::serialize_stream(const dmcg_encoded* e, uint8_t* out, size_t cap, dmcg_sections* s,
                             PayloadSpans* spans) {
  dmcg_sections sz;
  std::memset(&sz, 0, sizeof(sz));
  ByteOut w{out, cap};
  const char magic[4] = {'D', 'M', 'C', '1'};
  for (char c : magic) w.u8((uint8_t)c);
  w.u16(1);  // kStreamVersion
  w.u8(e->variant);
  w.u8(0);   // flags
  w.u32(e->n);
  w.u32(e->F);
  const uint32_t nb = e->n_b > 1 ? e->n_b : 1, pad = nb > 1 ? e->pad : 0;
  const uint32_t kf = (e->F + pad) / nb;
  w.u16((uint16_t)nb);
  w.u16((uint16_t)pad);
  w.u32(e->k_l);
  w.u32(e->n_c);
  w.u8(e->anchor_bits);
  w.u8(e->dict_bits);
  w.u8(e->diff_bits ? e->diff_bits : 8);
  w.u8(0);
  sz.header = w.pos;
  w.u32(e->n_faces);
  for (size_t t = 0; t < 3 * (size_t)e->n_faces; ++t) w.u32(e->faces[t]);
  sz.connectivity = w.pos - sz.header;
  const size_t FF = (size_t)kf * kf;
  if (spans && nb > 1) return 0;  // device packing serves n_b = 1 streams only
  for (int a = 0; a < 3; ++a) {
    size_t start = w.pos;
    if (spans) {
      spans->dict[a] = w.pos;
      skip(w, packed_bytes(FF, e->dict_bits));
    } else {
      BitOut b(w);
      for (size_t t = 0; t < FF; ++t) b.put(e->dict_q[a][t], e->dict_bits);
      b.flush();
    }
    sz.dict_payload += w.pos - start;
    for (uint32_t blk = 1; blk < nb; ++blk) {  // dict_diffs (stream.cpp:218-227)
      start = w.pos;
      w.f32(e->diff_min[a][blk - 1]);
      w.f32(e->diff_max[a][blk - 1]);
      sz.dict_ranges += w.pos - start;
      start = w.pos;
      BitOut b(w);
      for (size_t t = 0; t < FF; ++t) b.put(e->dict_q[a][blk * FF + t], e->diff_bits);
      b.flush();
      sz.dict_payload += w.pos - start;
    }
    for (uint32_t blk = 0; blk < nb; ++blk) {  // one CoeffBlock per block (stream.cpp:229-251)
      const size_t ro = (size_t)blk * e->k_l;
      const float* row_min = e->row_min[a] + ro;
      const float* row_max = e->row_max[a] + ro;
      const uint8_t* row_bits = e->row_bits[a] + ro;
      const uint16_t* coeff_q = e->coeff_q[a] + ro * e->n;
      start = w.pos;
      for (uint32_t r = 0; r < e->k_l; ++r) {
        w.f32(row_min[r]);
        w.f32(row_max[r]);
        w.u8(row_bits[r]);
      }
      sz.coeff_headers += w.pos - start;
      start = w.pos;
      if (spans) {
        spans->coeff[a] = w.pos;
        size_t bits = 0;
        for (uint32_t r = 0; r < e->k_l; ++r)
          if (row_min[r] != row_max[r]) bits += (size_t)e->n * row_bits[r];
        skip(w, (bits + 7) / 8);
      } else {
        BitOut b(w);
        for (uint32_t r = 0; r < e->k_l; ++r) {
          if (row_min[r] == row_max[r]) continue;  // no payload (stream.cpp:114)
          const uint16_t* q = coeff_q + (size_t)r * e->n;
          const int bits = row_bits[r];
          for (uint32_t i = 0; i < e->n; ++i) b.put(q[i], bits);
        }
        b.flush();
      }
      sz.coeff_payload += w.pos - start;
    }  // blocks
    if (variant_uses_means(e->variant)) {  // stream.cpp:255-263
      start = w.pos;
      for (uint32_t f = 0; f < e->F; ++f) w.f32(e->means[a][f]);
      sz.means += w.pos - start;
    }
  }
  if (!variant_uses_anchors(e->variant)) {
    if (s) *s = sz;
    return w.overflow ? 0 : w.pos;
  }
  size_t start = w.pos;
  for (uint32_t t = 0; t < e->n_c; ++t) w.u32(e->anchor_idx[t]);
  sz.anchor_indices = w.pos - start;
  for (int a = 0; a < 3; ++a) {
    start = w.pos;
    w.f32(e->anchor_min[a]);
    w.f32(e->anchor_max[a]);
    sz.anchor_ranges += w.pos - start;
    start = w.pos;
    if (spans) {
      spans->anchor[a] = w.pos;
      skip(w, packed_bytes((size_t)e->n_c * e->F, e->anchor_bits));
    } else {
      BitOut b(w);
      for (size_t t = 0; t < (size_t)e->n_c * e->F; ++t) b.put(e->anchor_q[a][t], e->anchor_bits);
      b.flush();
    }
    sz.anchor_payload += w.pos - start;
  }
  if (s) *s = sz;
  if (w.overflow) return 0;
  return w.pos;
}

extern "C" {

size_t dmcg_serialize(const dmcg_encoded* e, uint8_t* out, size_t cap, dmcg_sections* s) {
  if (!e) return 0;
  return dmcg::serialize_stream(e, out, cap, s, nullptr);
}

// Header fields + the reference's header checks (stream.cpp:299-336).
static int parse_header_impl(ByteIn& r, dmcg_encoded* c, std::string* msg) {
  static const char magic[4] = {'D', 'M', 'C', '1'};
  for (char ch : magic)
    if ((char)r.u8() != ch) {
      *msg = r.err.empty() ? "CorruptStream: bad magic" : "CorruptStream: " + r.err;
      return DMCG_E_CORRUPT;
    }
  const uint16_t version = r.u16();
  if (!r.err.empty()) return *msg = "CorruptStream: " + r.err, DMCG_E_CORRUPT;
  if (version != 1) {
    *msg = "VersionMismatch: stream version " + std::to_string(version) +
           ", supported version is 1";
    return DMCG_E_VERSION;
  }
  const uint8_t variant = r.u8();
  const uint8_t flags = r.u8();
  const uint32_t n = r.u32(), k = r.u32();
  const uint16_t n_b = r.u16(), pad = r.u16();
  const uint32_t k_l = r.u32(), n_c = r.u32();
  const uint8_t ab = r.u8(), db = r.u8(), fb = r.u8();
  r.u8();
  auto corrupt = [&](const char* what) {
    *msg = std::string("CorruptStream: ") + what;
    return DMCG_E_CORRUPT;
  };
  if (!r.err.empty()) return corrupt(r.err.c_str());
  if (variant > 6) return corrupt("unknown variant");
  if (flags & ~0x03) return corrupt("unknown flag bits");
  if (!(n >= 1 && k >= 1)) return corrupt("empty animation");
  if (n_b < 1) return corrupt("block count must be >= 1");
  if ((k + pad) % n_b != 0) return corrupt("padded frame count not divisible by block count");
  const uint32_t k_f = (k + pad) / n_b;
  if (!(pad < k_f || (pad == 0 && n_b == 1))) return corrupt("padding exceeds one block");
  if (variant == 6 && n_b != 1) return corrupt("per-mesh variant is unblocked");
  const uint32_t max_rows = variant == 6 ? n : k_f;
  if (k_l > max_rows) return corrupt("retained row count exceeds dictionary dimension");
  const bool anchors = variant == 3 || variant == 4 || variant == 5;
  if (anchors) {
    if (!(n_c >= 1 && n_c <= n)) return corrupt("anchor count out of range");
    if (!(ab >= 1 && ab <= 16)) return corrupt("anchor bit depth outside 1..16");
  } else if (n_c != 0) {
    return corrupt("anchor count nonzero for anchor-free variant");
  }
  if (!(db >= 1 && db <= 16)) return corrupt("dictionary bit depth outside 1..16");
  if (!(fb >= 1 && fb <= 16)) return corrupt("difference bit depth outside 1..16");
  if (variant > DMCG_BLOCKS || flags != 0 || (n_b == 1 && pad != 0)) {
    *msg = "Unsupported: only the variants pca, pca_q, v2v, pca_qs, pca_qp, blocks with "
           "quantised payloads are on the B200 path";
    return DMCG_E_UNSUPPORTED;
  }
  c->n_b = n_b;
  c->pad = pad;
  c->n = n;
  c->F = k;
  c->k_l = k_l;
  c->n_c = n_c;
  c->variant = variant;
  c->flags = flags;
  c->anchor_bits = ab;
  c->dict_bits = db;
  c->diff_bits = fb;
  c->n_faces = r.u32();
  if (!r.err.empty()) return corrupt(r.err.c_str());
  if (c->n_faces < 1) return corrupt("no faces");
  return DMCG_OK;
}

static thread_local std::string g_parse_error;

int dmcg_parse_header(const uint8_t* data, size_t size, dmcg_encoded* hdr) {
  if (!data || !hdr) return DMCG_E_CONFIG;
  ByteIn r{data, size, 0, {}};
  return parse_header_impl(r, hdr, &g_parse_error);
}

int dmcg_parse(const uint8_t* data, size_t size, dmcg_encoded* c, dmcg_sections* s) {
  if (!data || !c) return DMCG_E_CONFIG;
  ByteIn r{data, size, 0, {}};
  dmcg_sections sz;
  std::memset(&sz, 0, sizeof(sz));
  dmcg_encoded hdr = *c;
  int rc = parse_header_impl(r, &hdr, &g_parse_error);
  if (rc) return rc;
  auto corrupt = [&](const std::string& what) {
    g_parse_error = "CorruptStream: " + what;
    return DMCG_E_CORRUPT;
  };
  if (hdr.n != c->n || hdr.F != c->F || hdr.k_l != c->k_l || hdr.n_c != c->n_c ||
      hdr.n_faces != c->n_faces || hdr.n_b != (c->n_b ? c->n_b : 1) ||
      (hdr.n_b > 1 && hdr.pad != c->pad))
    return corrupt("buffers sized for a different header");
  *c = hdr;
  sz.header = 32;
  uint32_t* faces = const_cast<uint32_t*>(c->faces);
  for (uint32_t t = 0; t < c->n_faces; ++t) {
    uint32_t f[3];
    for (int j = 0; j < 3; ++j) {
      f[j] = r.u32();
      if (!r.err.empty()) return corrupt(r.err);
      if (f[j] >= c->n) return corrupt("face index out of range");
      faces[3 * (size_t)t + j] = f[j];
    }
    if (f[0] == f[1] || f[1] == f[2] || f[0] == f[2]) return corrupt("degenerate face");
  }
  sz.connectivity = r.pos - sz.header;
  const uint32_t nb = c->n_b, kf = (c->F + c->pad) / nb;
  const size_t FF = (size_t)kf * kf;
  for (int a = 0; a < 3; ++a) {
    size_t start = r.pos;
    const size_t db = packed_bytes(FF, c->dict_bits);
    const uint8_t* p = r.slice(db);
    if (!p) return corrupt(r.err);
    unpack(p, FF, c->dict_bits, c->dict_q[a]);
    sz.dict_payload += r.pos - start;
    for (uint32_t blk = 1; blk < nb; ++blk) {  // dict_diffs (stream.cpp:370-385)
      start = r.pos;
      const float mn = r.f32(), mx = r.f32();
      if (!r.err.empty()) return corrupt(r.err);
      if (!(mn <= mx)) return corrupt("difference range has min > max");
      c->diff_min[a][blk - 1] = mn;
      c->diff_max[a][blk - 1] = mx;
      sz.dict_ranges += r.pos - start;
      start = r.pos;
      const uint8_t* pd = r.slice(packed_bytes(FF, c->diff_bits));
      if (!pd) return corrupt(r.err);
      unpack(pd, FF, c->diff_bits, c->dict_q[a] + blk * FF);
      sz.dict_payload += r.pos - start;
    }
    for (uint32_t blk = 0; blk < nb; ++blk) {  // coeffs, one CoeffBlock per block
      const size_t ro = (size_t)blk * c->k_l;
      float* row_min = c->row_min[a] + ro;
      float* row_max = c->row_max[a] + ro;
      uint8_t* row_bits = c->row_bits[a] + ro;
      uint16_t* coeff_q = c->coeff_q[a] + ro * c->n;
      start = r.pos;
      size_t bits_total = 0;
      for (uint32_t q = 0; q < c->k_l; ++q) {
        row_min[q] = r.f32();
        row_max[q] = r.f32();
        row_bits[q] = r.u8();
        if (!r.err.empty()) return corrupt(r.err);
        if (row_bits[q] < 1 || row_bits[q] > 16)
          return corrupt("row bit depth outside 1..16");
        if (!(row_min[q] <= row_max[q])) return corrupt("row range has min > max");
        if (!(row_min[q] == row_max[q])) bits_total += (size_t)row_bits[q] * c->n;
      }
      sz.coeff_headers += r.pos - start;
      start = r.pos;
      const size_t pb = (bits_total + 7) / 8;
      const uint8_t* pp = r.slice(pb);
      if (!pp) return corrupt(r.err);
      // rows are contiguous in the bit stream: unpack sequentially
      uint64_t acc = 0;
      int fill = 0;
      size_t pos = 0;
      for (uint32_t q = 0; q < c->k_l; ++q) {
        uint16_t* o = coeff_q + (size_t)q * c->n;
        if (row_min[q] == row_max[q]) {
          std::memset(o, 0, (size_t)c->n * 2);
          continue;
        }
        const int bits = row_bits[q];
        const uint32_t mask = (1u << bits) - 1u;
        for (uint32_t i = 0; i < c->n; ++i) {
          while (fill < bits) {
            acc = (acc << 8) | pp[pos++];
            fill += 8;
          }
          fill -= bits;
          o[i] = (uint16_t)((acc >> fill) & mask);
        }
      }
      sz.coeff_payload += r.pos - start;
    }  // blocks
    if (dmcg::variant_uses_means(c->variant)) {
      start = r.pos;
      for (uint32_t f = 0; f < c->F; ++f) {
        const float m = r.f32();
        if (c->means[a]) c->means[a][f] = m;
      }
      if (!r.err.empty()) return corrupt(r.err);
      sz.means += r.pos - start;
    }
  }
  if (!dmcg::variant_uses_anchors(c->variant)) {
    if (r.pos != size) return corrupt("trailing bytes after stream end");
    if (s) *s = sz;
    return DMCG_OK;
  }
  size_t start = r.pos;
  uint32_t prev = 0;
  for (uint32_t t = 0; t < c->n_c; ++t) {
    const uint32_t v = r.u32();
    if (!r.err.empty()) return corrupt(r.err);
    if (v >= c->n) return corrupt("anchor index out of range");
    if (t > 0 && v <= prev) return corrupt("anchor indices not strictly increasing");
    c->anchor_idx[t] = prev = v;
  }
  sz.anchor_indices = r.pos - start;
  const size_t vals = (size_t)c->n_c * c->F;
  for (int a = 0; a < 3; ++a) {
    start = r.pos;
    c->anchor_min[a] = r.f32();
    c->anchor_max[a] = r.f32();
    if (!r.err.empty()) return corrupt(r.err);
    if (!(c->anchor_min[a] <= c->anchor_max[a])) return corrupt("anchor range has min > max");
    sz.anchor_ranges += r.pos - start;
    start = r.pos;
    const size_t pb = packed_bytes(vals, c->anchor_bits);
    const uint8_t* p = r.slice(pb);
    if (!p) return corrupt(r.err);
    unpack(p, vals, c->anchor_bits, c->anchor_q[a]);
    sz.anchor_payload += r.pos - start;
  }
  if (r.pos != size) return corrupt("trailing bytes after stream end");
  if (s) *s = sz;
  return DMCG_OK;
}

const char* dmcg_parse_error(void) { return g_parse_error.c_str(); }

void dmcg_rate_exact(const dmcg_sections* s, uint32_t n, uint32_t F, double out[5]) {
  const double tv = (double)n * F;
  out[0] = 8.0 * s->coeff_payload / tv;
  out[1] = 8.0 * (s->anchor_indices + s->anchor_payload) / tv;
  out[2] = 8.0 * s->dict_payload / tv;
  out[3] = 8.0 *
           (s->header + s->connectivity + s->dict_ranges + s->coeff_headers + s->means +
            s->anchor_ranges) /
           tv;
  out[4] = out[0] + out[1] + out[2] + out[3];
}

}  // extern "C"
