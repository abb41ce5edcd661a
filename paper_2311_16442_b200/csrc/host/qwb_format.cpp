// qwb_format.cpp -- packed-layer format: pack, validate, QWL1 container,
// tensor-parallel shards.
//
// pack_layer / validate_layer restate bitpack.cpp:91-147 and 212-247;
// the container restates container.cpp:112-471 (same bytes on disk, so files
// written by the reference load here and vice versa).
#include <algorithm>
#include <cstring>

#include "qwb_host.hpp"

namespace qwb {

namespace {

void put_codes2(const uint8_t* codes, uint8_t* dst, size_t n) {  // LSB-first
  std::memset(dst, 0, n / 4);
  for (size_t k = 0; k < n; ++k) {
    if (codes[k] > 3) throw Error("pack: 2-bit code out of range");
    dst[k >> 2] |= (uint8_t)(codes[k] << ((k & 3) * 2));
  }
}

void put_nibbles(const uint8_t* codes, uint8_t* dst) {  // even index low
  for (size_t i = 0; i < 4; ++i) {
    if (codes[2 * i] > 15 || codes[2 * i + 1] > 15) throw Error("pack: 4-bit code out of range");
    dst[i] = (uint8_t)(codes[2 * i] | (codes[2 * i + 1] << 4));
  }
}

uint16_t meta_word(const uint8_t* z, const uint8_t* s) {  // bitpack.cpp:45-56
  if (z[0] > 3 || z[1] > 3 || z[2] > 3) throw Error("pack_meta: zero-point out of range");
  if (s[0] > 15 || s[1] > 7 || s[2] > 7) throw Error("pack_meta: scale code out of range");
  return (uint16_t)(z[0] | (z[1] << 2) | (z[2] << 4) | (s[0] << 6) | (s[1] << 10) | (s[2] << 13));
}

void validate_csr(const CsrOutliers& csr, uint32_t rows, uint32_t padded) {  // outliers.cpp:175-190
  if (csr.row_ptr.size() != (size_t)rows + 1 || csr.row_ptr[0] != 0)
    throw Error("csr: row_ptr malformed");
  for (size_t r = 0; r < rows; ++r)
    if (csr.row_ptr[r] > csr.row_ptr[r + 1]) throw Error("csr: row_ptr not monotone");
  if (csr.col_ind.size() != csr.nnz() || csr.values.size() != csr.nnz())
    throw Error("csr: index/value lengths disagree with row_ptr");
  for (size_t r = 0; r < rows; ++r)
    for (uint32_t i = csr.row_ptr[r]; i < csr.row_ptr[r + 1]; ++i) {
      if (csr.col_ind[i] >= padded) throw Error("csr: column out of range");
      if (i > csr.row_ptr[r] && csr.col_ind[i] <= csr.col_ind[i - 1])
        throw Error("csr: columns not strictly increasing");
    }
}

}  // namespace

// plan.cpp:75-105
void validate_plan(const ChannelPlan& p) {
  if (p.in_channels == 0 || p.in_channels % kG1 != 0)
    throw Error("plan: channel count must be a positive multiple of 16");
  if (p.n4 > p.in_channels || p.n4 % kTile4 != 0) throw Error("plan: bad 4-bit channel count");
  if (p.pad2 != (kTile2 - p.n2() % kTile2) % kTile2) throw Error("plan: bad pad count");
  if (p.padded_channels() > kMaxSlots) throw Error("plan: padded channel count exceeds 65536");
  if (p.bits.size() != p.in_channels || p.perm.size() != p.padded_channels())
    throw Error("plan: field sizes inconsistent");
  std::vector<uint8_t> seen(p.in_channels, 0);
  for (uint32_t slot = 0; slot < p.perm.size(); ++slot) {
    const uint32_t c = p.perm[slot];
    const bool in_pads = slot >= p.n2() && slot < p.n2_padded();
    if (c == kPad) {
      if (!in_pads) throw Error("plan: pad channel outside pad region");
      continue;
    }
    if (in_pads || c >= p.in_channels || seen[c]++) throw Error("plan: permutation is not a bijection");
    if (p.bits[c] != (slot < p.n2() ? 2 : 4))
      throw Error("plan: bits[] disagrees with permutation regions");
  }
  for (uint8_t s : seen)
    if (!s) throw Error("plan: permutation is not a bijection");
}

// bitpack.cpp:212-247
void validate_layer(const PackedLayer& L) {
  const LayerConfig& c = L.cfg;
  if (c.n != 2 || c.n2 != 4 || c.group1 != kG1 || c.tile != kTile || c.group2 == 0)
    throw Error("layer: unsupported config constants");
  if (c.rows == 0 || c.cols == 0 || c.cols % kG1 != 0) throw Error("layer: rows/cols malformed");
  if (c.n4 > c.cols || c.n4 % kTile4 != 0) throw Error("layer: bad 4-bit channel count");
  if (c.pad2 != (kTile2 - (c.cols - c.n4) % kTile2) % kTile2) throw Error("layer: bad pad count");
  validate_plan(L.plan);
  if (L.plan.in_channels != c.cols || L.plan.n4 != c.n4 || L.plan.pad2 != c.pad2)
    throw Error("layer: plan disagrees with config");
  if (L.main.size() != c.main_bytes() || L.tail2.size() != c.tail2_bytes() ||
      L.tail4.size() != c.tail4_bytes() || L.secondary.size() != c.secondary_bytes() ||
      L.meta.size() != c.meta_count() || L.sorder.size() != c.sorder_count() ||
      L.fourbit.size() != c.fourbit_count())
    throw Error("layer: stream sizes disagree with config");
  for (const SorderParam& p : L.sorder)
    if (p.zero2 > 15) throw Error("layer: second-order zero out of range");
  for (const FourBitParam& p : L.fourbit)
    if (p.zero > 15) throw Error("layer: four-bit zero out of range");
  validate_csr(L.csr, c.rows, c.padded_cols());
  if (L.csr.nnz() != c.outlier_count) throw Error("layer: outlier count disagrees with config");
  for (uint16_t col : L.csr.col_ind)
    if (col >= c.n2_padded() || L.plan.perm[col] == kPad)
      throw Error("layer: outlier outside the 2-bit region");
}

// bitpack.cpp:91-147
PackedLayer pack_layer(const LayerConfig& cfg, const ChannelPlan& plan,
                       const LayerGroups& g, CsrOutliers csr) {
  const uint32_t t2 = cfg.triples(), t4 = cfg.blocks4(), pr = cfg.paired();
  const uint32_t gpr = cfg.groups_per_row(), n2p = cfg.n2_padded();
  if (g.codes2.size() != (size_t)cfg.rows * n2p || g.zeros2.size() != (size_t)cfg.rows * gpr ||
      g.scodes.size() != (size_t)cfg.rows * gpr || g.sorder.size() != cfg.sorder_count() ||
      g.codes4.size() != (size_t)cfg.rows * cfg.n4 || g.fourbit.size() != cfg.fourbit_count())
    throw Error("pack_layer: group field sizes disagree with config");
  if (csr.row_ptr.empty()) csr.row_ptr.assign((size_t)cfg.rows + 1, 0);
  PackedLayer L;
  L.cfg = cfg;
  L.plan = plan;
  L.main.assign(cfg.main_bytes(), 0);
  L.tail2.assign(cfg.tail2_bytes(), 0);
  L.tail4.assign(cfg.tail4_bytes(), 0);
  L.secondary.assign(cfg.secondary_bytes(), 0);
  L.meta.assign(cfg.meta_count(), 0);
  L.sorder = g.sorder;
  L.fourbit = g.fourbit;
  L.csr = std::move(csr);
  for (size_t r = 0; r < cfg.rows; ++r) {
    for (uint32_t t = 0; t < t2; ++t) {
      L.meta[r * t2 + t] = meta_word(&g.zeros2[r * gpr + 3 * t], &g.scodes[r * gpr + 3 * t]);
      uint8_t* dst = t < pr ? &L.main[(r * pr + t) * 16] : &L.tail2[(r * (t2 - pr) + (t - pr)) * 12];
      put_codes2(&g.codes2[r * n2p + (size_t)t * kTile2], dst, kTile2);
    }
    for (uint32_t b = 0; b < t4; ++b) {
      const uint8_t* c4 = &g.codes4[r * cfg.n4 + (size_t)b * kTile4];
      put_nibbles(c4, b < pr ? &L.main[(r * pr + b) * 16 + 12] : &L.tail4[(r * (t4 - pr) + (b - pr)) * 4]);
      put_nibbles(c4 + 8, &L.secondary[(r * t4 + b) * 4]);
    }
  }
  validate_layer(L);
  return L;
}

// container.cpp:252-279, 466-471: every section except the plan's
uint64_t payload_bytes(const LayerConfig& c, uint64_t nnz) {
  return c.main_bytes() + c.tail2_bytes() + c.tail4_bytes() + c.secondary_bytes() +
         c.meta_count() * 2 + c.sorder_count() * 3 + c.fourbit_count() * 3 +
         (nnz ? ((uint64_t)c.rows + 1) * 4 : 0) + nnz * 4;
}

// ------------------------------------------------------------------ QWL1
namespace {

constexpr uint32_t kSections = 12;

struct Out {
  std::vector<uint8_t> b;
  void u8(uint8_t v) { b.push_back(v); }
  void u16(uint16_t v) { u8((uint8_t)v), u8((uint8_t)(v >> 8)); }
  void u32(uint32_t v) { u16((uint16_t)v), u16((uint16_t)(v >> 16)); }
  void u64(uint64_t v) { u32((uint32_t)v), u32((uint32_t)(v >> 32)); }
  void f32(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    u32(u);
  }
  void raw(const std::vector<uint8_t>& v) { b.insert(b.end(), v.begin(), v.end()); }
};

struct In {
  std::span<const uint8_t> b;
  size_t at = 0;
  const char* what = "header";
  void need(size_t n) const {
    if (at + n > b.size()) throw Error(std::string("container: truncated ") + what);
  }
  uint8_t u8() { return need(1), b[at++]; }
  uint16_t u16() {
    const uint16_t lo = u8();
    return (uint16_t)(lo | (u8() << 8));
  }
  uint32_t u32() {
    const uint32_t lo = u16();
    return lo | ((uint32_t)u16() << 16);
  }
  uint64_t u64() {
    const uint64_t lo = u32();
    return lo | ((uint64_t)u32() << 32);
  }
  float f32() {
    const uint32_t u = u32();
    float v;
    std::memcpy(&v, &u, 4);
    return v;
  }
};

const char* section_label(uint32_t id) {
  static const char* names[] = {"?",         "plan_bits", "plan_perm", "main",
                                "tail2",     "tail4",     "secondary", "meta",
                                "sorder",    "fourbit",   "csr_row_ptr",
                                "csr_col_ind", "csr_values"};
  return id <= kSections ? names[id] : "unknown";
}

uint64_t section_length(const LayerConfig& c, uint32_t id) {  // container.cpp:182-211
  switch (id) {
    case 1: return (c.cols + 7) / 8;
    case 2: return (uint64_t)c.padded_cols() * 4;
    case 3: return c.main_bytes();
    case 4: return c.tail2_bytes();
    case 5: return c.tail4_bytes();
    case 6: return c.secondary_bytes();
    case 7: return c.meta_count() * 2;
    case 8: return c.sorder_count() * 3;
    case 9: return c.fourbit_count() * 3;
    case 10: return c.outlier_count ? ((uint64_t)c.rows + 1) * 4 : 0;
    default: return (uint64_t)c.outlier_count * 2;
  }
}

std::vector<uint8_t> encode(const PackedLayer& L, uint32_t id) {
  Out o;
  switch (id) {
    case 1:
      o.b.assign((L.cfg.cols + 7) / 8, 0);
      for (uint32_t c = 0; c < L.cfg.cols; ++c)
        if (L.plan.bits[c] == 4) o.b[c / 8] |= (uint8_t)(1u << (c % 8));
      break;
    case 2: for (uint32_t v : L.plan.perm) o.u32(v); break;
    case 3: o.b = L.main; break;
    case 4: o.b = L.tail2; break;
    case 5: o.b = L.tail4; break;
    case 6: o.b = L.secondary; break;
    case 7: for (uint16_t m : L.meta) o.u16(m); break;
    case 8: for (auto& p : L.sorder) o.u8(p.zero2), o.u16(p.scale2); break;
    case 9: for (auto& p : L.fourbit) o.u16(p.scale), o.u8(p.zero); break;
    case 10: if (L.csr.nnz()) for (uint32_t v : L.csr.row_ptr) o.u32(v); break;
    case 11: for (uint16_t v : L.csr.col_ind) o.u16(v); break;
    case 12: for (uint16_t v : L.csr.values) o.u16(v); break;
  }
  return o.b;
}

void decode(PackedLayer& L, uint32_t id, std::span<const uint8_t> b) {
  In in{b, 0, section_label(id)};
  const LayerConfig& c = L.cfg;
  switch (id) {
    case 1:
      L.plan.bits.assign(c.cols, 2);
      for (uint32_t k = 0; k < c.cols; ++k)
        if (b[k / 8] & (1u << (k % 8))) L.plan.bits[k] = 4;
      in.at = b.size();
      break;
    case 2: L.plan.perm.resize(c.padded_cols()); for (auto& v : L.plan.perm) v = in.u32(); break;
    case 3: L.main.assign(b.begin(), b.end()), in.at = b.size(); break;
    case 4: L.tail2.assign(b.begin(), b.end()), in.at = b.size(); break;
    case 5: L.tail4.assign(b.begin(), b.end()), in.at = b.size(); break;
    case 6: L.secondary.assign(b.begin(), b.end()), in.at = b.size(); break;
    case 7: L.meta.resize(b.size() / 2); for (auto& m : L.meta) m = in.u16(); break;
    case 8:
      L.sorder.resize(b.size() / 3);
      for (auto& p : L.sorder) p.zero2 = in.u8(), p.scale2 = in.u16();
      break;
    case 9:
      L.fourbit.resize(b.size() / 3);
      for (auto& p : L.fourbit) p.scale = in.u16(), p.zero = in.u8();
      break;
    case 10:
      if (b.empty()) {
        L.csr.row_ptr.assign((size_t)c.rows + 1, 0);
        break;
      }
      L.csr.row_ptr.resize(b.size() / 4);
      for (auto& v : L.csr.row_ptr) v = in.u32();
      break;
    case 11: L.csr.col_ind.resize(b.size() / 2); for (auto& v : L.csr.col_ind) v = in.u16(); break;
    case 12: L.csr.values.resize(b.size() / 2); for (auto& v : L.csr.values) v = in.u16(); break;
  }
  if (in.at != b.size())
    throw Error(std::string("container: section ") + section_label(id) + " has unexpected length");
}

}  // namespace

uint32_t crc32(std::span<const uint8_t> bytes) {  // IEEE, reflected 0xEDB88320
  static uint32_t table[256];
  static const bool ready = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
      table[i] = c;
    }
    return true;
  }();
  (void)ready;
  uint32_t c = 0xFFFFFFFFu;
  for (uint8_t v : bytes) c = table[(c ^ v) & 0xFFu] ^ (c >> 8);
  return ~c;
}

std::vector<uint8_t> serialize_layer(const PackedLayer& L) {
  validate_layer(L);
  Out o;
  const char magic[4] = {'Q', 'W', 'L', '1'};
  o.b.insert(o.b.end(), magic, magic + 4);
  const LayerConfig& c = L.cfg;
  o.u16(1), o.u16(0);
  o.u16(c.n), o.u16(c.n2), o.u16(c.group1), o.u16(c.group2), o.u16(c.tile), o.u16(0);
  o.u32(c.rows), o.u32(c.cols), o.u32(c.n4), o.u32(c.pad2), o.u32(c.outlier_count);
  o.f32(c.alpha), o.f32(c.outlier_ratio);
  std::vector<std::vector<uint8_t>> body;
  for (uint32_t id = 1; id <= kSections; ++id) body.push_back(encode(L, id));
  o.u32(kSections);
  uint64_t off = o.b.size() + kSections * 20;
  for (uint32_t id = 1; id <= kSections; ++id) {
    o.u32(id), o.u64(off), o.u64(body[id - 1].size());
    off += body[id - 1].size();
  }
  for (auto& s : body) o.raw(s);
  o.u32(crc32(o.b));
  return o.b;
}

PackedLayer deserialize_layer(std::span<const uint8_t> bytes) {
  if (bytes.size() < 8 || std::memcmp(bytes.data(), "QWL1", 4) != 0) throw Error("container: bad magic");
  if (bytes.size() < 48 + 4 + kSections * 20 + 4) throw Error("container: truncated header");
  const size_t n = bytes.size();
  const uint32_t stored = (uint32_t)bytes[n - 4] | ((uint32_t)bytes[n - 3] << 8) |
                          ((uint32_t)bytes[n - 2] << 16) | ((uint32_t)bytes[n - 1] << 24);
  if (crc32(bytes.subspan(0, n - 4)) != stored) throw Error("container: checksum mismatch");
  In in{bytes, 4};
  if (in.u16() != 1) throw Error("container: unsupported version");
  in.u16();
  PackedLayer L;
  LayerConfig& c = L.cfg;
  c.n = in.u16(), c.n2 = in.u16(), c.group1 = in.u16(), c.group2 = in.u16(), c.tile = in.u16();
  in.u16();
  c.rows = in.u32(), c.cols = in.u32(), c.n4 = in.u32(), c.pad2 = in.u32(), c.outlier_count = in.u32();
  c.alpha = in.f32(), c.outlier_ratio = in.f32();
  if (c.cols == 0 || c.cols % kG1 != 0 || c.n4 > c.cols || c.group2 == 0 || c.rows == 0)
    throw Error("container: malformed config");
  if (in.u32() != kSections) throw Error("container: unexpected section count");
  uint64_t off[kSections + 1], len[kSections + 1];
  uint64_t end = in.at + kSections * 20;
  for (uint32_t id = 1; id <= kSections; ++id) {
    if (in.u32() != id) throw Error("container: section table out of order");
    off[id] = in.u64(), len[id] = in.u64();
    if (off[id] != end) throw Error("container: section offsets not contiguous");
    if (len[id] != section_length(c, id))
      throw Error(std::string("container: section ") + section_label(id) + " has unexpected length");
    if (off[id] + len[id] + 4 > n)
      throw Error(std::string("container: truncated section ") + section_label(id));
    end = off[id] + len[id];
  }
  if (end + 4 != n) throw Error("container: trailing bytes after sections");
  L.plan.in_channels = c.cols, L.plan.n4 = c.n4, L.plan.pad2 = c.pad2;
  for (uint32_t id = 1; id <= kSections; ++id) decode(L, id, bytes.subspan(off[id], len[id]));
  validate_layer(L);
  return L;
}

// ------------------------------------------------------------------ shards
// Column-parallel split: rows [r0, r1) with whole 2-order row blocks.
PackedLayer shard_rows(const PackedLayer& L, uint32_t r0, uint32_t r1) {
  const LayerConfig& c = L.cfg;
  if (r0 >= r1 || r1 > c.rows) throw Error("shard_rows: empty or out-of-range row range");
  if (r0 % c.group2 != 0 || (r1 % c.group2 != 0 && r1 != c.rows))
    throw Error("shard_rows: shard boundaries must align to group2 row blocks");
  PackedLayer S;
  S.cfg = c;
  S.cfg.rows = r1 - r0;
  S.plan = L.plan;
  auto slice = [](const auto& v, uint64_t per_row, uint32_t a, uint32_t b) {
    return std::remove_cvref_t<decltype(v)>(v.begin() + a * per_row, v.begin() + b * per_row);
  };
  S.main = slice(L.main, (uint64_t)c.paired() * 16, r0, r1);
  S.tail2 = slice(L.tail2, (uint64_t)c.tail2_blocks() * 12, r0, r1);
  S.tail4 = slice(L.tail4, (uint64_t)c.tail4_blocks() * 4, r0, r1);
  S.secondary = slice(L.secondary, (uint64_t)c.blocks4() * 4, r0, r1);
  S.meta = slice(L.meta, c.triples(), r0, r1);
  S.fourbit = slice(L.fourbit, c.blocks4(), r0, r1);
  const uint32_t b0 = r0 / c.group2, b1 = (r1 + c.group2 - 1) / c.group2;
  S.sorder = slice(L.sorder, c.groups_per_row(), b0, b1);
  const uint32_t e0 = L.csr.row_ptr[r0], e1 = L.csr.row_ptr[r1];
  S.csr.row_ptr.resize((size_t)(r1 - r0) + 1);
  for (uint32_t r = r0; r <= r1; ++r) S.csr.row_ptr[r - r0] = L.csr.row_ptr[r] - e0;
  S.csr.col_ind.assign(L.csr.col_ind.begin() + e0, L.csr.col_ind.begin() + e1);
  S.csr.values.assign(L.csr.values.begin() + e0, L.csr.values.begin() + e1);
  S.cfg.outlier_count = e1 - e0;
  validate_layer(S);
  return S;
}

// Row-parallel split: tiles [t0, t1) of a layer whose 2-bit triples and
// 4-bit blocks pair one to one (every Llama shape).  The shard's channels are
// numbered in the parent's permuted order, real 2-bit slots first.
PackedLayer shard_tiles(const PackedLayer& L, uint32_t t0, uint32_t t1) {
  const LayerConfig& c = L.cfg;
  const uint32_t T = c.triples();
  if (T != c.blocks4()) throw Error("shard_tiles: layer has unpaired tail tiles");
  if (t0 >= t1 || t1 > T) throw Error("shard_tiles: empty or out-of-range tile range");
  const uint32_t nt = t1 - t0;
  const uint32_t lo2 = 48 * t0, hi2 = 48 * t1;
  uint32_t real2 = 0;
  for (uint32_t s = lo2; s < hi2; ++s) real2 += L.plan.perm[s] != kPad;
  PackedLayer S;
  S.cfg = c;
  S.cfg.n4 = 16 * nt;
  S.cfg.cols = real2 + S.cfg.n4;
  S.cfg.pad2 = 48 * nt - real2;
  if (S.cfg.cols % kG1 != 0) throw Error("shard_tiles: shard channel count not a multiple of 16");
  S.plan.in_channels = S.cfg.cols;
  S.plan.n4 = S.cfg.n4;
  S.plan.pad2 = S.cfg.pad2;
  S.plan.bits.assign(S.cfg.cols, 2);
  for (uint32_t k = real2; k < S.cfg.cols; ++k) S.plan.bits[k] = 4;
  for (uint32_t k = 0; k < real2; ++k) S.plan.perm.push_back(k);
  S.plan.perm.insert(S.plan.perm.end(), S.cfg.pad2, kPad);
  for (uint32_t k = 0; k < S.cfg.n4; ++k) S.plan.perm.push_back(real2 + k);
  const uint32_t rows = c.rows;
  for (uint32_t r = 0; r < rows; ++r) {
    S.main.insert(S.main.end(), L.main.begin() + ((size_t)r * T + t0) * 16, L.main.begin() + ((size_t)r * T + t1) * 16);
    S.secondary.insert(S.secondary.end(), L.secondary.begin() + ((size_t)r * T + t0) * 4,
                       L.secondary.begin() + ((size_t)r * T + t1) * 4);
    S.meta.insert(S.meta.end(), L.meta.begin() + (size_t)r * T + t0, L.meta.begin() + (size_t)r * T + t1);
    S.fourbit.insert(S.fourbit.end(), L.fourbit.begin() + (size_t)r * T + t0, L.fourbit.begin() + (size_t)r * T + t1);
  }
  const uint32_t gpr = c.groups_per_row();
  for (uint32_t b = 0; b < c.row_blocks(); ++b)
    S.sorder.insert(S.sorder.end(), L.sorder.begin() + (size_t)b * gpr + 3 * t0,
                    L.sorder.begin() + (size_t)b * gpr + 3 * t1);
  S.csr.row_ptr.assign((size_t)rows + 1, 0);
  for (uint32_t r = 0; r < rows; ++r) {
    for (uint32_t i = L.csr.row_ptr[r]; i < L.csr.row_ptr[r + 1]; ++i) {
      const uint32_t col = L.csr.col_ind[i];
      if (col < lo2 || col >= hi2) continue;
      S.csr.col_ind.push_back((uint16_t)(col - lo2));
      S.csr.values.push_back(L.csr.values[i]);
    }
    S.csr.row_ptr[r + 1] = (uint32_t)S.csr.col_ind.size();
  }
  S.cfg.outlier_count = (uint32_t)S.csr.col_ind.size();
  validate_layer(S);
  return S;
}

}  // namespace qwb
