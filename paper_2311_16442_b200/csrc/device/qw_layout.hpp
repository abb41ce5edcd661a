// qw_layout.hpp -- row-pair packing of the code words inside a quad record.
//
// The reference keeps one 32-bit word of 2-bit codes per (row, group)
// (codes 0-7 in the low half, 8-15 in the high half) and two words of 4-bit
// codes per (row, block) (codes 0-7, 8-15; nibble n at bits 4n).  The device
// record interleaves rows 2p and 2p+1 at 16-bit granularity so that one
// fp16x2 lane pair of an HFMA2 holds the same channel of two rows:
//
//   2-bit, pair p:  word 0 = rowA codes 0-7  | rowB codes 0-7  << 16
//                   word 1 = rowA codes 8-15 | rowB codes 8-15 << 16
//   4-bit, pair p:  word j = rowA codes 4j..4j+3 | rowB codes 4j..4j+3 << 16
//
// Host (repack) and device (decode kernels) share these helpers.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define QW_HD __host__ __device__ __forceinline__
#else
#define QW_HD inline
#endif

namespace qwdev {

// 2-bit: reference words of rows A, B -> the pair's two device words
QW_HD void pack_pair2(uint32_t a, uint32_t b, uint32_t out[2]) {
  out[0] = (a & 0xFFFFu) | (b << 16);
  out[1] = (a >> 16) | (b & 0xFFFF0000u);
}
// device words of a 2-bit pair -> reference word of row `side` (0 = A)
QW_HD uint32_t unpack_pair2(const uint32_t w[2], uint32_t side) {
  const uint32_t s = 16u * side;
  return ((w[0] >> s) & 0xFFFFu) | (((w[1] >> s) & 0xFFFFu) << 16);
}
// 4-bit: reference words (lo = codes 0-7, hi = codes 8-15) of rows A, B ->
// four device words
QW_HD void pack_pair4(uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi, uint32_t out[4]) {
  out[0] = (a_lo & 0xFFFFu) | (b_lo << 16);
  out[1] = (a_lo >> 16) | (b_lo & 0xFFFF0000u);
  out[2] = (a_hi & 0xFFFFu) | (b_hi << 16);
  out[3] = (a_hi >> 16) | (b_hi & 0xFFFF0000u);
}
QW_HD void unpack_pair4(const uint32_t w[4], uint32_t side, uint32_t* lo, uint32_t* hi) {
  const uint32_t s = 16u * side;
  *lo = ((w[0] >> s) & 0xFFFFu) | (((w[1] >> s) & 0xFFFFu) << 16);
  *hi = ((w[2] >> s) & 0xFFFFu) | (((w[3] >> s) & 0xFFFFu) << 16);
}

}  // namespace qwdev
