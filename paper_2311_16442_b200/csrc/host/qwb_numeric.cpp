// qwb_numeric.cpp -- IEEE half conversion and the Eq. 1-4 group fits.
//
// Bit-identical restatements of reference proj/src/fp16.cpp and
// proj/src/quant.cpp.  Built with -ffp-contract=off and without -march so the
// float expressions round exactly like the reference's default build.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "qwb_host.hpp"

namespace qwb {

// fp16.cpp:8-38 -- round-to-nearest-even, subnormals kept, NaN quieted to
// sign|0x7E00, overflow to infinity.
uint16_t f32_to_f16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, sizeof u);
  const uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
  const uint32_t fexp = (u >> 23) & 0xFFu;
  uint32_t mant = u & 0x7FFFFFu;
  if (fexp == 0xFFu) return (uint16_t)(sign | 0x7C00u | (mant ? 0x200u : 0u));
  const int hexp = (int)fexp - 112;  // rebias 127 -> 15
  if (hexp >= 31) return (uint16_t)(sign | 0x7C00u);
  if (hexp <= 0) {
    if (hexp < -10) return sign;
    mant |= 0x800000u;
    const uint32_t drop = (uint32_t)(14 - hexp);  // bits shifted out
    const uint32_t kept = mant >> drop;
    const uint32_t rest = mant & ((1u << drop) - 1u);
    const uint32_t half = 1u << (drop - 1);
    const uint32_t up = (rest > half || (rest == half && (kept & 1u))) ? 1u : 0u;
    return (uint16_t)(sign | (kept + up));
  }
  const uint32_t kept = ((uint32_t)hexp << 10) | (mant >> 13);
  const uint32_t rest = mant & 0x1FFFu;
  const uint32_t up = (rest > 0x1000u || (rest == 0x1000u && (kept & 1u))) ? 1u : 0u;
  return (uint16_t)(sign | (kept + up));  // carry may walk into inf, as intended
}

// fp16.cpp:40-64
float f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t hexp = (h >> 10) & 0x1Fu;
  const uint32_t mant = h & 0x3FFu;
  uint32_t u;
  if (hexp == 31) {
    u = sign | 0x7F800000u | (mant << 13);
  } else if (hexp != 0) {
    u = sign | ((hexp + 112u) << 23) | (mant << 13);
  } else if (mant == 0) {
    u = sign;
  } else {
    int lead = 9;  // position of the leading one of the 10-bit subnormal
    while (!(mant & (1u << lead))) --lead;
    const uint32_t frac = (mant << (10 - lead)) & 0x3FFu;
    u = sign | ((uint32_t)(103 + lead) << 23) | (frac << 13);
  }
  float f;
  std::memcpy(&f, &u, sizeof f);
  return f;
}

namespace {
void require_bits(int bits) {
  if (bits < 1 || bits > 8) throw Error("quant: unsupported bit width");
}
}  // namespace

// quant.cpp:18-52 -- asymmetric min/max fit with the degenerate-group rules.
ScaleZero fit_scale_zero(std::span<const float> v, int bits) {
  require_bits(bits);
  if (v.empty()) throw Error("fit_scale_zero: empty group");
  float lo = v[0], hi = v[0];
  for (float x : v) {
    if (!std::isfinite(x)) throw Error("fit_scale_zero: non-finite value");
    lo = std::min(lo, x);
    hi = std::max(hi, x);
  }
  const float top = (float)((1 << bits) - 1);
  if (lo == hi) {
    if (lo == 0.0f) return {1.0f, 0};
    const float mag = std::fabs(lo);
    const uint8_t z = lo > 0.0f ? (uint8_t)0 : (uint8_t)top;
    const float step = mag / top;
    return (step * top == mag) ? ScaleZero{step, z} : ScaleZero{mag, z};
  }
  float s = (hi - lo) / top;
  if (!std::isfinite(s)) throw Error("fit_scale_zero: range overflows float32");
  if (s == 0.0f) s = hi - lo;
  const float zr = std::round(-lo / s);
  const uint8_t z = zr <= 0.0f ? (uint8_t)0 : (zr >= top ? (uint8_t)top : (uint8_t)zr);
  return {s, z};
}

// quant.cpp:54-68 -- round half away from zero, clamp to the code range.
void quantize_values(std::span<const float> v, float scale, uint8_t zero,
                     int bits, uint8_t* codes) {
  require_bits(bits);
  if (!(scale > 0.0f) || !std::isfinite(scale))
    throw Error("quantize_values: scale must be positive and finite");
  const float top = (float)((1 << bits) - 1);
  if ((float)zero > top) throw Error("quantize_values: zero-point out of range");
  for (size_t i = 0; i < v.size(); ++i) {
    const float c = std::round(v[i] / scale) + (float)zero;
    codes[i] = c <= 0.0f ? (uint8_t)0 : (c >= top ? (uint8_t)top : (uint8_t)c);
  }
}

}  // namespace qwb
