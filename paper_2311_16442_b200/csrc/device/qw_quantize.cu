// qw_quantize.cu -- the offline producer's data-parallel passes on the GPU
// (SURVEY §8(f) rank 3): quantize_layer (quantizer.cpp:132-146) with every
// per-element / per-group pass on the device and the decisions that need a
// global order (the channel plan, the final top-K ranking, CSR, pack) on the
// host (csrc/host/qwb_gpu_producer.cpp).  Bit-identical to the reference:
// every float / double operation is the same IEEE operation in the same
// order, written with explicit round-to-nearest intrinsics so nothing is
// contracted into an FMA (the reference builds without -march: SURVEY H8).
//
//   amplitudes_kernel  compute_amplitudes (plan.cpp:10-30): per column,
//                      sum over rows ascending of (w/h)^2 in double
//   score_kernel       score_outliers (outliers.cpp:30-44, 61-79) on every
//                      real 2-bit slot: the baseline 2-bit group fit, its
//                      residual^2 / h^2 in double; pass 1 histograms the
//                      scores by their top 16 bits, pass 2 emits the
//                      candidates at or above the bucket holding rank k
//   fit1_kernel        quantize_groups' first-order fits (quantizer.cpp:38-80):
//                      2-bit groups refit without their outlier slots, 4-bit
//                      blocks, codes
//   fit2_kernel        the 2-order pass down each group column of a row block
//                      (quantizer.cpp:82-107, 4/3/3 rule)
#include <cuda_runtime.h>

#include <cstdint>

#include "qw_device.hpp"

namespace qwdev {
namespace {

constexpr uint32_t kPadCh = 0xFFFFFFFFu;

// fit_scale_zero (quant.cpp:18-52) on n values; returns false on a
// non-finite input (the host raises the reference's error)
__device__ __forceinline__ bool fit(const float* v, int n, int bits, float& s_out, uint32_t& z_out) {
  float lo = v[0], hi = v[0];
  bool ok = true;
  for (int i = 0; i < n; ++i) {  // std::min / std::max semantics (first wins on ties)
    ok = ok && isfinite(v[i]);
    lo = v[i] < lo ? v[i] : lo;
    hi = hi < v[i] ? v[i] : hi;
  }
  const float top = (float)((1 << bits) - 1);
  if (lo == hi) {
    if (lo == 0.0f) {
      s_out = 1.0f, z_out = 0;
      return ok;
    }
    const float mag = fabsf(lo);
    const uint32_t z = lo > 0.0f ? 0u : (uint32_t)top;
    const float step = __fdiv_rn(mag, top);
    s_out = (__fmul_rn(step, top) == mag) ? step : mag, z_out = z;
    return ok;
  }
  float s = __fdiv_rn(__fsub_rn(hi, lo), top);
  ok = ok && isfinite(s);
  if (s == 0.0f) s = __fsub_rn(hi, lo);
  const float zr = roundf(__fdiv_rn(-lo, s));  // round half away from zero (std::round)
  z_out = zr <= 0.0f ? 0u : (zr >= top ? (uint32_t)top : (uint32_t)zr);
  s_out = s;
  return ok;
}

// quantize_values (quant.cpp:54-68)
__device__ __forceinline__ uint32_t qcode(float v, float s, uint32_t z, int bits) {
  const float top = (float)((1 << bits) - 1);
  const float c = __fadd_rn(roundf(__fdiv_rn(v, s)), (float)z);
  return c <= 0.0f ? 0u : (c >= top ? (uint32_t)top : (uint32_t)c);
}

__global__ void amplitudes_kernel(const float* __restrict__ w, const float* __restrict__ h, uint32_t rows,
                                  uint32_t cols, double* __restrict__ amp) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const double b = h[c];
  const double bb = __dmul_rn(b, b);
  double acc = 0.0;
  for (uint32_t r = 0; r < rows; ++r) {  // ascending rows, as the reference
    const double a = w[(size_t)r * cols + c];
    acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(a, a), bb));
  }
  amp[c] = acc;
}

// the permuted value of slot k (apply_permutation, plan.cpp:107-116)
__device__ __forceinline__ float wp_at(const float* __restrict__ wrow, const uint32_t* __restrict__ perm,
                                       uint32_t k) {
  const uint32_t o = perm[k];
  return o == kPadCh ? 0.0f : wrow[o];
}
__device__ __forceinline__ uint32_t bucket_of(double s) { return (uint32_t)(__double_as_longlong(s) >> 48); }

// One thread per (row, 2-bit group).  mode 0: histogram; mode 1: candidates
// with bucket >= floor_bucket (score, row, slot) appended.
__global__ void score_kernel(const float* __restrict__ w, const float* __restrict__ h,
                             const uint32_t* __restrict__ perm, uint32_t rows, uint32_t cols, uint32_t n2p,
                             uint32_t mode, unsigned long long* __restrict__ hist, uint32_t floor_bucket,
                             double* __restrict__ cs, uint32_t* __restrict__ crow, uint32_t* __restrict__ ccol,
                             unsigned long long* __restrict__ ncand, uint32_t* __restrict__ bad) {
  const uint32_t groups = n2p / 16;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint64_t)rows * groups) return;
  const uint32_t r = (uint32_t)(i / groups), base = (uint32_t)(i % groups) * 16;
  const float* wrow = w + (size_t)r * cols;
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = wp_at(wrow, perm, base + k);
  float s;
  uint32_t z;
  if (!fit(v, 16, 2, s, z)) atomicOr(bad, 1u);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t orig = perm[base + k];
    if (orig == kPadCh) continue;
    const uint32_t c = qcode(v[k], s, z, 2);
    const float deq = __fmul_rn((float)((int)c - (int)z), s);  // dequantize_one (quant.hpp:30-32)
    const double res = __dsub_rn((double)deq, (double)v[k]);
    const double dh = h[orig];
    const double sc = __ddiv_rn(__dmul_rn(res, res), __dmul_rn(dh, dh));
    if (!(sc > 0.0)) continue;
    const uint32_t b = bucket_of(sc);
    if (mode == 0) {
      atomicAdd(hist + b, 1ull);
    } else if (b >= floor_bucket) {
      const unsigned long long at = atomicAdd(ncand, 1ull);
      cs[at] = sc, crow[at] = r, ccol[at] = base + k;
    }
  }
}

// One thread per (row, group): 2-bit groups g < G2 (outlier slots -> 0 and
// out of the refit), then 4-bit blocks.
__global__ void fit1_kernel(const float* __restrict__ w, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ outmask, uint32_t rows, uint32_t cols, uint32_t n2p,
                            uint32_t n4, uint8_t* __restrict__ codes2, uint8_t* __restrict__ zeros2,
                            float* __restrict__ scale1, uint8_t* __restrict__ codes4, float* __restrict__ s4,
                            uint8_t* __restrict__ z4, uint32_t* __restrict__ bad) {
  const uint32_t G2 = n2p / 16, T4 = n4 / 16, G = G2 + T4, pc = n2p + n4, mw = (pc + 31) / 32;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint64_t)rows * G) return;
  const uint32_t r = (uint32_t)(i / G), j = (uint32_t)(i % G);
  const float* wrow = w + (size_t)r * cols;
  float v[16];
  if (j < G2) {
    const uint32_t base = 16 * j;
    const uint32_t m = (outmask[(size_t)r * mw + base / 32] >> (base % 32)) & 0xFFFFu;
    float keep[16];
    int kept = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const bool out = (m >> k) & 1u;
      v[k] = out ? 0.0f : wp_at(wrow, perm, base + k);
      if (!out) keep[kept++] = v[k];
    }
    if (kept == 0) keep[kept++] = 0.0f;
    float s;
    uint32_t z;
    if (!fit(keep, kept, 2, s, z)) atomicOr(bad, 1u);
    scale1[(size_t)r * G2 + j] = s;
    zeros2[(size_t)r * G2 + j] = (uint8_t)z;
#pragma unroll
    for (int k = 0; k < 16; ++k) codes2[(size_t)r * n2p + base + k] = (uint8_t)qcode(v[k], s, z, 2);
  } else {
    const uint32_t b = j - G2, base = n2p + 16 * b;
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = wp_at(wrow, perm, base + k);
    float s;
    uint32_t z;
    if (!fit(v, 16, 4, s, z)) atomicOr(bad, 1u);
    s4[(size_t)r * T4 + b] = s;
    z4[(size_t)r * T4 + b] = (uint8_t)z;
#pragma unroll
    for (int k = 0; k < 16; ++k) codes4[(size_t)r * n4 + 16 * b + k] = (uint8_t)qcode(v[k], s, z, 4);
  }
}

// One thread per (row block, 2-bit group column): quantize_scales_2order
// (quant.cpp:87-107) on the block's first-order scales, then the 4/3/3 rule.
__global__ void fit2_kernel(const float* __restrict__ scale1, uint32_t rows, uint32_t G2, uint32_t group2,
                            uint8_t* __restrict__ scodes, float* __restrict__ s2, uint8_t* __restrict__ zero2,
                            uint32_t* __restrict__ bad) {
  const uint32_t rbs = (rows + group2 - 1) / group2;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint64_t)rbs * G2) return;
  const uint32_t rb = (uint32_t)(i / G2), j = (uint32_t)(i % G2);
  const uint32_t r0 = rb * group2, rn = min(group2, rows - r0);
  float hi = 0.0f;
  for (uint32_t k = 0; k < rn; ++k) {
    const float sv = scale1[(size_t)(r0 + k) * G2 + j];
    if (!(sv >= 0.0f) || !isfinite(sv)) atomicOr(bad, 2u);
    hi = hi < sv ? sv : hi;
  }
  const float ends[2] = {0.0f, hi};
  float s;
  uint32_t z;
  fit(ends, 2, 4, s, z);
  s2[i] = s, zero2[i] = (uint8_t)z;
  for (uint32_t k = 0; k < rn; ++k) {
    const uint32_t c = qcode(scale1[(size_t)(r0 + k) * G2 + j], s, z, 4);
    scodes[(size_t)(r0 + k) * G2 + j] = (uint8_t)((j % 3 == 0) ? c : (c >> 1));
  }
}

__global__ void outmask_kernel(const uint32_t* __restrict__ row_ptr, const uint16_t* __restrict__ col_ind,
                               uint32_t rows, uint32_t mw, uint32_t* __restrict__ outmask) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (uint32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
    const uint32_t c = col_ind[e];
    outmask[(size_t)r * mw + c / 32] |= 1u << (c % 32);  // one thread per row: no race
  }
}

uint32_t blocks_for(uint64_t n, uint32_t t) { return (uint32_t)((n + t - 1) / t); }

}  // namespace

int producer_amplitudes(const float* w, const float* h, uint32_t rows, uint32_t cols, double* amp) {
  if (cols) amplitudes_kernel<<<blocks_for(cols, 128), 128>>>(w, h, rows, cols, amp);
  return (int)cudaGetLastError();
}
int producer_scores(const float* w, const float* h, const uint32_t* perm, uint32_t rows, uint32_t cols,
                    uint32_t n2p, uint32_t mode, unsigned long long* hist, uint32_t floor_bucket, double* cs,
                    uint32_t* crow, uint32_t* ccol, unsigned long long* ncand, uint32_t* bad) {
  // A zero-sized grid is a launch error, so empty stages are skipped (alpha = 1: no 2-bit columns).
  if (const uint32_t nb = blocks_for((uint64_t)rows * (n2p / 16), 256))
    score_kernel<<<nb, 256>>>(w, h, perm, rows, cols, n2p, mode, hist,
                                                                     floor_bucket, cs, crow, ccol, ncand, bad);
  return (int)cudaGetLastError();
}
int producer_fits(const float* w, const uint32_t* perm, const uint32_t* row_ptr, const uint16_t* col_ind,
                  uint32_t* outmask, uint32_t rows, uint32_t cols, uint32_t n2p, uint32_t n4, uint32_t group2,
                  uint8_t* codes2, uint8_t* zeros2, float* scale1, uint8_t* codes4, float* s4, uint8_t* z4,
                  uint8_t* scodes, float* s2, uint8_t* zero2, uint32_t* bad) {
  const uint32_t pc = n2p + n4, mw = (pc + 31) / 32, G2 = n2p / 16;
  cudaError_t e = cudaMemset(outmask, 0, (size_t)rows * mw * 4);
  if (e != cudaSuccess) return (int)e;
  if (rows) outmask_kernel<<<blocks_for(rows, 128), 128>>>(row_ptr, col_ind, rows, mw, outmask);
  if (const uint32_t nb = blocks_for((uint64_t)rows * (G2 + n4 / 16), 256))
    fit1_kernel<<<nb, 256>>>(w, perm, outmask, rows, cols, n2p, n4, codes2, zeros2, scale1, codes4, s4, z4, bad);
  if (const uint32_t nb = blocks_for((uint64_t)((rows + group2 - 1) / group2) * G2, 128))
    fit2_kernel<<<nb, 128>>>(scale1, rows, G2, group2, scodes, s2, zero2, bad);
  return (int)cudaGetLastError();
}

}  // namespace qwdev
