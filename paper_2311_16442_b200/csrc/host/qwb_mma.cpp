// qwb_mma.cpp -- host repack of a validated PackedLayer into the tile format
// of the tensor-core batch-1 kernel (K2m, qw_mma.cu; layout in qw_device.hpp).
//
// Reads the reference streams (bitpack.hpp:15-22, bitpack.cpp:175-210):
// 2-bit group j of row r is bytes 4 sub .. 4 sub + 3 of tile j / 3's main
// block (or tail2), code k at bits 2k; 4-bit block b is main bytes 12-15 (or
// tail4) + secondary, nibble k at bits 4k; meta / sorder / fourbit as the
// reference structs.  Nothing is re-quantized: every code, zero and scale is
// moved bit for bit, and the 2-order pair (scale2, zero2) of each group is
// stored as the two fp16 constants the kernel's s1 evaluation uses.
#include <cmath>
#include <cstring>

#include "../device/qw_device.hpp"
#include "qwb_host.hpp"

namespace qwb {

namespace {

struct Src {
  const PackedLayer& L;
  uint32_t T2, T4, G2, P;
  uint32_t code2(uint32_t r, uint32_t j) const {  // 16 codes of 2-bit group j, code k at bits 2k
    if (r >= L.cfg.rows || j >= G2) return 0;
    const uint32_t t = j / 3, sub = j % 3;
    const uint8_t* b = t < P ? &L.main[((size_t)r * P + t) * 16]
                             : &L.tail2[((size_t)r * L.cfg.tail2_blocks() + (t - P)) * 12];
    uint32_t w;
    std::memcpy(&w, b + 4 * sub, 4);
    return w;
  }
  uint32_t code4(uint32_t r, uint32_t blk, uint32_t k) const {  // code k of 4-bit block blk
    if (r >= L.cfg.rows || blk >= T4) return 0;
    const uint8_t* p;
    if (k < 8)
      p = blk < P ? &L.main[((size_t)r * P + blk) * 16 + 12]
                  : &L.tail4[((size_t)r * L.cfg.tail4_blocks() + (blk - P)) * 4];
    else
      p = &L.secondary[((size_t)r * T4 + blk) * 4];
    uint32_t w;
    std::memcpy(&w, p, 4);
    return (w >> (4 * (k & 7))) & 15u;
  }
  uint32_t meta(uint32_t r, uint32_t t) const {
    return (r < L.cfg.rows && t < T2) ? L.meta[(size_t)r * T2 + t] : 0u;
  }
};

// channel 2s (even half) / 2s + 1 (odd half) of a 16-code group at bits 2s
uint32_t even_half(uint32_t w) {
  uint32_t h = 0;
  for (uint32_t s = 0; s < 8; ++s) h |= ((w >> (4 * s)) & 3u) << (2 * s);
  return h;
}
uint32_t odd_half(uint32_t w) {
  uint32_t h = 0;
  for (uint32_t s = 0; s < 8; ++s) h |= ((w >> (4 * s + 2)) & 3u) << (2 * s);
  return h;
}

void put32(uint8_t* p, uint32_t v) { std::memcpy(p, &v, 4); }

}  // namespace

// group of 2-bit column n of block b of super-block sb (rows' lane t owns
// triples 8 sb + 2t, 8 sb + 2t + 1: columns 2t, 2t+1 of the 3 blocks)
static inline uint32_t mma_group2(uint32_t sb, uint32_t b, uint32_t n) {
  return 24u * sb + 6u * (n >> 1) + 2u * b + (n & 1u);
}

void repack_mma(const PackedLayer& L, const qwdev::MmaGeometry& m, float s_scale, std::vector<uint8_t>& out) {
  const auto& c = L.cfg;
  Src src{L, c.triples(), c.blocks4(), c.groups_per_row(), c.paired()};
  out.assign((size_t)m.RT * m.nchunks * m.rec_stride, 0);
  const uint32_t nb2 = 3 * m.SB;
  for (uint32_t ch = 0; ch < m.nchunks; ++ch) {
    const qwdev::MmaChunk& C = m.chunk[ch];
    for (uint32_t tile = 0; tile < m.RT; ++tile) {
      uint8_t* rec = &out[((size_t)ch * m.RT + tile) * m.rec_stride];
      const uint32_t r0 = 16 * tile, rb = r0 / c.group2;
      for (uint32_t i = 0; i < C.nblk; ++i) {
        const uint32_t kind = C.kind[i], grp = C.grp[i];
        if (kind < 3) {
          const uint32_t sb = grp, b = kind;
          uint8_t* hdr = rec + C.hdr_off[i];
          for (uint32_t lane = 0; lane < 32; ++lane) {
            const uint32_t g = lane >> 2, t = lane & 3;
            // meta words of the lane's two triples, rows g and g + 8
            for (uint32_t h = 0; h < 2; ++h) {
              const uint32_t r = r0 + g + 8 * h;
              put32(hdr + 8 * lane + 4 * h, src.meta(r, 8 * sb + 2 * t) | (src.meta(r, 8 * sb + 2 * t + 1) << 16));
            }
            // codes: E_g, E_g+8, O_g, O_g+8; low half column 2t, high half 2t + 1
            const uint32_t j0 = mma_group2(sb, b, 2 * t), j1 = mma_group2(sb, b, 2 * t + 1);
            uint8_t* cw = rec + C.code_off[i] + 16 * lane;
            for (uint32_t h = 0; h < 2; ++h) {
              const uint32_t r = r0 + g + 8 * h;
              const uint32_t w0 = src.code2(r, j0), w1 = src.code2(r, j1);
              put32(cw + 4 * h, even_half(w0) | (even_half(w1) << 16));
              put32(cw + 8 + 4 * h, odd_half(w0) | (odd_half(w1) << 16));
            }
          }
          // sorder of the tile's 2-order row block: (a, c) per column, as
          // fp16: a = scale2 2^-P, c = -(2^(10 - pe) + zero2); the masked eff
          // field ORed into 1024 reads 1024 + eff 2^pe (pe = 6 / 2 / 5 for
          // sub 0 / 1 / 2, the 4/3/3 rule, quantizer.cpp:103-104)
          for (uint32_t bb = 0; bb < 3; ++bb)
            for (uint32_t t = 0; t < 4; ++t)
              for (uint32_t e = 0; e < 2; ++e) {
                const uint32_t j = mma_group2(sb, bb, 2 * t + e);
                uint32_t v = 0;
                if (j < src.G2) {
                  const SorderParam& sp = L.sorder[(size_t)rb * src.G2 + j];
                  const int pe = (j % 3) == 0 ? 6 : ((j % 3) == 1 ? 2 : 5);
                  const uint16_t a = f32_to_f16(f16_to_f32(sp.scale2) * s_scale);
                  const uint16_t cc = f32_to_f16(-(std::ldexp(1.0f, 10 - pe) + (float)sp.zero2));
                  v = (uint32_t)a | ((uint32_t)cc << 16);
                }
                put32(hdr + 256 + 8 * (4 * bb + t) + 4 * e, v);
              }
        } else {
          const uint32_t bb = grp;
          uint8_t* cw = rec + C.code_off[i];
          uint8_t* s4 = rec + C.hdr_off[i];
          uint8_t* z4 = s4 + qwdev::kMmaS4;
          for (uint32_t lane = 0; lane < 32; ++lane) {
            const uint32_t g = lane >> 2, t = lane & 3;
            const uint32_t b0 = 8 * bb + 2 * t, b1 = b0 + 1;
            // W(row, e, h): nibble i = code 2(4h + i) + e; low half block b0, high b1
            for (uint32_t h = 0; h < 2; ++h)
              for (uint32_t e = 0; e < 2; ++e)
                for (uint32_t rr = 0; rr < 2; ++rr) {
                  const uint32_t r = r0 + g + 8 * rr;
                  uint32_t q0 = 0, q1 = 0;
                  for (uint32_t ii = 0; ii < 4; ++ii) {
                    const uint32_t k = 2 * (4 * h + ii) + e;
                    q0 |= src.code4(r, b0, k) << (4 * ii);
                    q1 |= src.code4(r, b1, k) << (4 * ii);
                  }
                  put32(cw + 32 * lane + 16 * h + 8 * e + 4 * rr, q0 | (q1 << 16));
                }
            uint32_t zz = 0;
            for (uint32_t rr = 0; rr < 2; ++rr) {
              const uint32_t r = r0 + g + 8 * rr;
              uint32_t sv[2] = {0, 0}, zv[2] = {0, 0};
              for (uint32_t e = 0; e < 2; ++e) {
                const uint32_t blk = b0 + e;
                if (r < c.rows && blk < src.T4) {
                  const FourBitParam& fb = L.fourbit[(size_t)r * src.T4 + blk];
                  sv[e] = fb.scale, zv[e] = fb.zero & 15u;
                }
              }
              put32(s4 + 8 * lane + 4 * rr, sv[0] | (sv[1] << 16));
              zz |= (zv[0] << (4 * rr)) | (zv[1] << (8 + 4 * rr));
            }
            const uint16_t z16 = (uint16_t)zz;
            std::memcpy(z4 + 2 * lane, &z16, 2);
          }
        }
      }
    }
  }
}

}  // namespace qwb
