// qw_kernels.cu -- sm_100a kernels of the quantized linear layer y = W_q x.
//
//   K5 prologue  x (original order) -> permuted fp32 xp + per-16-group fp16
//                x' (power-of-two scaled) + sum(x') + unscale factor
//                (apply_permutation plan.cpp:107-116, checked_permute
//                engine.cpp:124-132)
//   K2/K3 gemv   batch-1 GEMV with the 2-order scale decode, LOP3 unpack,
//                fp16x2 dot products, warp-shuffle reduce and the fp16 CSR
//                outliers fused into the same output accumulation
//                (matvec_oracle engine.cpp:169-183, row_* 40-122)
//   K1 dequant   bit-exact reconstruct_dense (engine.cpp:151-167)
//   K0 unpack    bit-exact unpack_layer codes (bitpack.cpp:149-173)
//
// The GEMV is a persistent, warp-specialised kernel: one producer warp
// streams whole 4-row quad records HBM -> shared memory with cp.async.bulk
// (TMA bulk copies) into an mbarrier ring; 8 consumer warps decode them.
// Algorithm 1 of the paper (asynchronous dequantization) maps onto this ring:
// 2-order parameters ride in the same bulk transaction as the weight words,
// so first-order scale reconstruction overlaps the streaming of later quads.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "qw_device.hpp"

namespace qwdev {
namespace {

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Programmatic dependent launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;  // (a & b) | c
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ half2 as_h2(uint32_t u) { return *reinterpret_cast<half2*>(&u); }
__device__ __forceinline__ float half_bits_to_float(uint32_t h) {
  return __half2float(__ushort_as_half((unsigned short)(h & 0xFFFFu)));
}
// small non-negative integer -> exact float without I2F (2^23 magic)
__device__ __forceinline__ float small_int_to_float(uint32_t v) {
  return __int_as_float(0x4B000000u | v) - 8388608.0f;
}

// ------------------------------------------------ code unpack + dot product
// A code c sitting at mantissa bits [j, j+width) of an fp16 whose exponent
// makes bit j worth 1 reads as magic + c exactly; subtracting the magic is
// exact, so one LOP3 + one HSUB2 turns two codes into two fp16 integers.
//
// 2-bit word (reference main bytes 4*sub..4*sub+3): code k at bits 2k, so the
// low half holds codes 0-7 and the high half codes 8-15.  Masks at bit 2k of
// each half, k = 0..3, applied to w and w >> 8, yield the pairs (p, p+8),
// p = 0..7; X[p] = {x'_p, x'_{p+8}}.
__device__ __forceinline__ half2 code_step(half2 acc, uint32_t src, uint32_t mask, uint32_t magic,
                                           half2 x) {
  return __hfma2(__hsub2(as_h2(lop3_and_or(src, mask, magic)), as_h2(magic)), x, acc);
}
__device__ __forceinline__ float dot_2bit(uint32_t w, const half2* X) {
  const uint32_t hi = w >> 8;
  half2 acc = __float2half2_rn(0.0f);
  acc = code_step(acc, w, 0x00030003u, 0x64006400u, X[0]);
  acc = code_step(acc, w, 0x000C000Cu, 0x5C005C00u, X[1]);
  acc = code_step(acc, w, 0x00300030u, 0x54005400u, X[2]);
  acc = code_step(acc, w, 0x00C000C0u, 0x4C004C00u, X[3]);
  acc = code_step(acc, hi, 0x00030003u, 0x64006400u, X[4]);
  acc = code_step(acc, hi, 0x000C000Cu, 0x5C005C00u, X[5]);
  acc = code_step(acc, hi, 0x00300030u, 0x54005400u, X[6]);
  acc = code_step(acc, hi, 0x00C000C0u, 0x4C004C00u, X[7]);
  const float2 f = __half22float2(acc);
  return f.x + f.y;
}
// 4-bit block: word 0 holds codes 0-7 (nibble n at bits 4n), word 1 codes
// 8-15.  Masks at bits 0 and 4 of each half on w and w >> 8 give the pairs
// (0,4) (1,5) (2,6) (3,7) of each word.
__device__ __forceinline__ float dot_4bit(uint32_t w0, uint32_t w1, const half2* X) {
  const uint32_t h0 = w0 >> 8, h1 = w1 >> 8;
  half2 acc = __float2half2_rn(0.0f);
  acc = code_step(acc, w0, 0x000F000Fu, 0x64006400u, X[0]);
  acc = code_step(acc, w0, 0x00F000F0u, 0x54005400u, X[1]);
  acc = code_step(acc, h0, 0x000F000Fu, 0x64006400u, X[2]);
  acc = code_step(acc, h0, 0x00F000F0u, 0x54005400u, X[3]);
  acc = code_step(acc, w1, 0x000F000Fu, 0x64006400u, X[4]);
  acc = code_step(acc, w1, 0x00F000F0u, 0x54005400u, X[5]);
  acc = code_step(acc, h1, 0x000F000Fu, 0x64006400u, X[6]);
  acc = code_step(acc, h1, 0x00F000F0u, 0x54005400u, X[7]);
  const float2 f = __half22float2(acc);
  return f.x + f.y;
}

// ------------------------------------------------------------ K5 prologue
// One 16-lane segment per group.  The scale 2^-sh puts max|x'| in [64, 128)
// so the fp16 partial sums of a 16-wide group cannot overflow (|P| <
// 15*16*128) while keeping fp16's full relative precision.
__global__ void __launch_bounds__(256) prologue_kernel(const float* __restrict__ x,
                                                       const uint32_t* __restrict__ perm,
                                                       uint32_t cols, uint32_t G2, uint32_t G,
                                                       uint8_t* __restrict__ xprep,
                                                       uint32_t block_stride, float* __restrict__ xp,
                                                       uint32_t xp_stride, uint32_t* flags) {
  pdl_launch_dependents();
  pdl_wait();  // x may be produced by the previous kernel
  const uint32_t col = blockIdx.y;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t g = tid >> 4, k = tid & 15u;
  const bool live = g < G;
  float v = 0.0f;
  if (live) {
    const uint32_t s = 16u * g + k;
    const uint32_t src = perm[s];
    v = src == 0xFFFFFFFFu ? 0.0f : x[(size_t)col * cols + src];
    if (!isfinite(v)) atomicOr(flags, 1u);
    xp[(size_t)col * xp_stride + s] = v;
  }
  float m = fabsf(v);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o, 16));
  int sh = 0;
  if (m > 0.0f && isfinite(m)) sh = ilogbf(m) - 6;
  const __half h = __float2half_rn(ldexpf(v, -sh));
  float s = __half2float(h);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o, 16);
  if (!live) return;
  uint8_t* blk = xprep + (size_t)col * block_stride;
  const uint32_t idx = g < G2 ? 2u * (k & 7u) + (k >> 3)
                              : 2u * ((k & 3u) + 4u * (k >> 3)) + ((k >> 2) & 1u);
  reinterpret_cast<__half*>(blk)[16u * g + idx] = h;
  if (k == 0) {
    float* sx = reinterpret_cast<float*>(blk + 32u * G);
    sx[g] = s;
    sx[G + g] = ldexpf(1.0f, sh);
  }
}

// ------------------------------------------------------------ K2/K3 GEMV
constexpr int kConsumerWarps = 8;
constexpr int kGemvThreads = (kConsumerWarps + 1) * 32;

struct GemvArgs {
  const uint8_t* quads;
  const uint32_t* sorder;
  const uint32_t* row_ptr;
  const uint32_t* csr;
  const uint8_t* xprep;
  const float* xp;
  float* y;
  Geometry g;
  uint32_t nslot, slot_stride, sorder_off, sorder_bytes_max;
  uint32_t xprep_bytes, xregion, nchunks, grid, nq_max;
  uint32_t uniform_rb;  // group2 % 4 == 0: a quad lies in one 2-order block
};

// Sum the 4 row partials of a warp: afterwards lanes 8i..8i+7 hold row i.
__device__ __forceinline__ float reduce4(float a0, float a1, float a2, float a3, uint32_t lane) {
  const bool up = lane & 16u;
  float k0 = up ? a2 : a0, k1 = up ? a3 : a1;
  const float s0 = up ? a0 : a2, s1 = up ? a1 : a3;
  k0 += __shfl_xor_sync(0xFFFFFFFFu, s0, 16);
  k1 += __shfl_xor_sync(0xFFFFFFFFu, s1, 16);
  const bool mid = lane & 8u;
  float v = mid ? k1 : k0;
  v += __shfl_xor_sync(0xFFFFFFFFu, mid ? k0 : k1, 8);
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 4);
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
  return v;
}

__global__ void __launch_bounds__(kGemvThreads, 2) gemv_kernel(const __grid_constant__ GemvArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Geometry& G = a.g;
  uint8_t* s_x = smem;
  uint8_t* s_slots = smem + a.xregion;
  float* s_part = reinterpret_cast<float*>(s_slots + (size_t)a.nslot * a.slot_stride);
  float* s_csr = s_part + a.nslot * a.nchunks * 4;
  uint32_t* s_done = reinterpret_cast<uint32_t*>(s_csr + a.nq_max * 4);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(s_done + a.nq_max) + 7) & ~uintptr_t(7));
  uint64_t* s_empty = s_full + a.nslot;
  uint64_t* s_xbar = s_empty + a.nslot;

  const uint32_t q0 = (uint32_t)((uint64_t)blockIdx.x * G.quads / a.grid);
  const uint32_t q1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * G.quads / a.grid);
  const uint32_t nq = q1 - q0;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < a.nslot; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
    }
    mbar_init(s_xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (uint32_t i = threadIdx.x; i < nq; i += blockDim.x) s_done[i] = 0;
  __syncthreads();
  pdl_launch_dependents();

  if (warp == kConsumerWarps) {
    // ---------------- producer: stream quad records + their 2-order rows
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      auto issue = [&](uint32_t i) {
        const uint32_t q = q0 + i, slot = i % a.nslot;
        const uint32_t r_first = q * kRowsPerQuad;
        const uint32_t r_last = min(r_first + kRowsPerQuad, G.rows) - 1;
        const uint32_t rb0 = r_first / G.group2, rb1 = r_last / G.group2;
        const uint32_t sob = (rb1 - rb0 + 1) * G.G2s * 4u;
        uint8_t* dst = s_slots + (size_t)slot * a.slot_stride;
        mbar_expect_tx(&s_full[slot], G.dense_bytes + sob);
        bulk_load(dst, a.quads + (size_t)q * G.dense_bytes, G.dense_bytes, &s_full[slot], pol_w);
        bulk_load(dst + a.sorder_off, a.sorder + (size_t)rb0 * G.G2s, sob, &s_full[slot], pol_w);
      };
      const uint32_t first = min(nq, a.nslot);
      for (uint32_t i = 0; i < first; ++i) issue(i);
      // the activation block is written by the prologue kernel
      pdl_wait();
      mbar_expect_tx(s_xbar, a.xprep_bytes);
      bulk_load(s_x, a.xprep, a.xprep_bytes, s_xbar, policy_evict_last());
      for (uint32_t i = first; i < nq; ++i) {
        mbar_wait(&s_empty[i % a.nslot], ((i / a.nslot) - 1) & 1u);
        issue(i);
      }
    }
    return;
  }

  // ---------------- consumers
  const float* s_sx = reinterpret_cast<const float*>(s_x + 32u * G.G);
  const float* s_ex = s_sx + G.G;
  bool have_x = false;
  const uint32_t ntask = nq * (a.nchunks + 1);
  for (uint32_t task = warp; task < ntask; task += kConsumerWarps) {
    uint32_t lq, chunk;
    const bool is_csr = task < nq;
    if (is_csr) {
      lq = task;
      chunk = a.nchunks;
    } else {
      lq = (task - nq) / a.nchunks;
      chunk = (task - nq) - lq * a.nchunks;
    }
    const uint32_t q = q0 + lq, slot = lq % a.nslot;
    const uint32_t r0 = q * kRowsPerQuad;
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f, acc3 = 0.0f;

    if (is_csr) {
      // ---------- K3: fp16 outliers of the quad's rows (outliers.cpp:131-141)
      const uint32_t nrow = min((uint32_t)kRowsPerQuad, G.rows - r0);
      uint32_t rp = 0;
      if (lane <= (uint32_t)kRowsPerQuad) rp = a.row_ptr[r0 + min(lane, nrow)];
      const uint32_t base = __shfl_sync(0xFFFFFFFFu, rp, 0);
      const uint32_t c1 = __shfl_sync(0xFFFFFFFFu, rp, 1) - base;
      const uint32_t c2 = __shfl_sync(0xFFFFFFFFu, rp, 2) - base;
      const uint32_t c3 = __shfl_sync(0xFFFFFFFFu, rp, 3) - base;
      const uint32_t cnt = __shfl_sync(0xFFFFFFFFu, rp, 4) - base;
      if (cnt > 0) {
        pdl_wait();  // xp comes from the prologue kernel
        for (uint32_t e = lane; e < cnt; e += 32) {
          const uint32_t ent = a.csr[base + e];
          const float prod = half_bits_to_float(ent >> 16) * a.xp[ent & 0xFFFFu];
          const uint32_t row = (e >= c1) + (e >= c2) + (e >= c3);
          acc0 += row == 0 ? prod : 0.0f;
          acc1 += row == 1 ? prod : 0.0f;
          acc2 += row == 2 ? prod : 0.0f;
          acc3 += row == 3 ? prod : 0.0f;
        }
      }
      const float v = reduce4(acc0, acc1, acc2, acc3, lane);
      if ((lane & 7u) == 0) s_csr[lq * 4 + (lane >> 3)] = v;
    } else {
      if (!have_x) {
        mbar_wait(s_xbar, 0);
        have_x = true;
      }
      mbar_wait(&s_full[slot], (lq / a.nslot) & 1u);
      const uint8_t* sb = s_slots + (size_t)slot * a.slot_stride;
      const uint32_t* sso = reinterpret_cast<const uint32_t*>(sb + a.sorder_off);
      const uint32_t g = chunk * 32u + lane;
      if (g < G.G) {
        const uint4 xa = *reinterpret_cast<const uint4*>(s_x + 32u * g);
        const uint4 xb = *reinterpret_cast<const uint4*>(s_x + 32u * g + 16u);
        const half2 X[8] = {as_h2(xa.x), as_h2(xa.y), as_h2(xa.z), as_h2(xa.w),
                            as_h2(xb.x), as_h2(xb.y), as_h2(xb.z), as_h2(xb.w)};
        const float sx = s_sx[g], ex = s_ex[g];
        float acc[4];
        if (g < G.G2) {
          // ---------- 2-bit group: stages 1-4 of engine.cpp:40-122
          const uint4 w = *reinterpret_cast<const uint4*>(sb + 16u * g);
          const uint32_t t = g / 3u, sub = g - 3u * t;
          const uint2 m2 = *reinterpret_cast<const uint2*>(sb + G.off_meta + 8u * t);
          const uint32_t zsh = 2u * sub;
          const uint32_t esh = sub == 0 ? 6u : (sub == 1 ? 9u : 12u);  // 4/3/3 rule
          const uint32_t emask = sub == 0 ? 15u : 14u;
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
          const uint32_t ms[4] = {m2.x & 0xFFFFu, m2.x >> 16, m2.y & 0xFFFFu, m2.y >> 16};
          const uint32_t rbase = r0 / G.group2;
          float A = 0.0f, B = 0.0f;
          if (a.uniform_rb) {
            const uint32_t e = sso[g];
            A = half_bits_to_float(e) * ex;  // scale2 * 2^sh (exact)
            B = -small_int_to_float(e >> 16) * A;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (!a.uniform_rb) {
              const uint32_t rb = (r0 + i) / G.group2 - rbase;
              const uint32_t e = sso[rb * G.G2s + g];
              A = half_bits_to_float(e) * ex;
              B = -small_int_to_float(e >> 16) * A;
            }
            const float P = dot_2bit(ws[i], X);
            const float eff = small_int_to_float((ms[i] >> esh) & emask);
            const float z = small_int_to_float((ms[i] >> zsh) & 3u);
            const float s1 = fmaf(eff, A, B);  // (eff - zero2) * scale2 * 2^sh
            acc[i] = s1 * fmaf(-z, sx, P);     // sum (c - z) x' over the group
          }
        } else {
          // ---------- 4-bit block
          const uint32_t b = g - G.G2;
          const uint4 w0 = *reinterpret_cast<const uint4*>(sb + G.off_c4 + 32u * b);
          const uint4 w1 = *reinterpret_cast<const uint4*>(sb + G.off_c4 + 32u * b + 16u);
          const uint2 s4 = *reinterpret_cast<const uint2*>(sb + G.off_s4 + 8u * b);
          const uint32_t z4 = *reinterpret_cast<const uint16_t*>(sb + G.off_z4 + 2u * b);
          const uint32_t a0[4] = {w0.x, w0.y, w0.z, w0.w};
          const uint32_t a1[4] = {w1.x, w1.y, w1.z, w1.w};
          const uint32_t ss[4] = {s4.x, s4.x >> 16, s4.y, s4.y >> 16};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float P = dot_4bit(a0[i], a1[i], X);
            const float s = half_bits_to_float(ss[i]) * ex;
            const float z = small_int_to_float((z4 >> (4 * i)) & 15u);
            acc[i] = s * fmaf(-z, sx, P);
          }
        }
        acc0 = acc[0], acc1 = acc[1], acc2 = acc[2], acc3 = acc[3];
      }
      const float v = reduce4(acc0, acc1, acc2, acc3, lane);
      if ((lane & 7u) == 0) s_part[(slot * a.nchunks + chunk) * 4 + (lane >> 3)] = v;
    }

    // ---------- completion: the last of nchunks+1 tasks finalises the quad
    __syncwarp();
    uint32_t prev = 0;
    if (lane == 0) {
      __threadfence_block();
      prev = atomicAdd(&s_done[lq], 1u);
    }
    prev = __shfl_sync(0xFFFFFFFFu, prev, 0);
    if (prev == a.nchunks) {
      __threadfence_block();
      if (lane < (uint32_t)kRowsPerQuad) {
        float s = 0.0f;
        for (uint32_t c = 0; c < a.nchunks; ++c) s += s_part[(slot * a.nchunks + c) * 4 + lane];
        s += s_csr[lq * 4 + lane];  // outliers after the dense sum, as row_fma
        if (r0 + lane < G.rows) a.y[r0 + lane] = s;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[slot]);
    }
  }
}

// ------------------------------------------------------------ K1 dequant
// One thread per (row, group); products are exact in fp32, so any
// evaluation order reproduces reconstruct_dense bit for bit.
__global__ void dequant_kernel(const uint8_t* __restrict__ quads,
                               const uint32_t* __restrict__ sorder, Geometry G,
                               float* __restrict__ w) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)G.rows * G.G) return;
  const uint32_t r = (uint32_t)(tid / G.G), g = (uint32_t)(tid % G.G);
  const uint8_t* qr = quads + (size_t)(r / kRowsPerQuad) * G.dense_bytes;
  const uint32_t i = r % kRowsPerQuad;
  float out[16];
  if (g < G.G2) {
    const uint32_t word = *reinterpret_cast<const uint32_t*>(qr + 16u * g + 4u * i);
    const uint32_t t = g / 3u, sub = g - 3u * t;
    const uint32_t meta = *reinterpret_cast<const uint16_t*>(qr + G.off_meta + 8u * t + 2u * i);
    const int z = (int)((meta >> (2 * sub)) & 3u);
    const uint32_t sc = sub == 0 ? (meta >> 6) & 15u : ((meta >> (sub == 1 ? 10 : 13)) & 7u) << 1;
    const uint32_t e = sorder[(size_t)(r / G.group2) * G.G2s + g];
    const float s1 = (float)((int)sc - (int)(e >> 16)) * half_bits_to_float(e);
#pragma unroll
    for (int k = 0; k < 16; ++k) out[k] = (float)((int)((word >> (2 * k)) & 3u) - z) * s1;
  } else {
    const uint32_t b = g - G.G2;
    const uint32_t w0 = *reinterpret_cast<const uint32_t*>(qr + G.off_c4 + 32u * b + 4u * i);
    const uint32_t w1 = *reinterpret_cast<const uint32_t*>(qr + G.off_c4 + 32u * b + 16u + 4u * i);
    const float s4 = half_bits_to_float(*reinterpret_cast<const uint16_t*>(qr + G.off_s4 + 8u * b + 2u * i));
    const int z4 = (int)((*reinterpret_cast<const uint16_t*>(qr + G.off_z4 + 2u * b) >> (4 * i)) & 15u);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      out[k] = (float)((int)((w0 >> (4 * k)) & 15u) - z4) * s4;
      out[8 + k] = (float)((int)((w1 >> (4 * k)) & 15u) - z4) * s4;
    }
  }
  float4* dst = reinterpret_cast<float4*>(w + (size_t)r * G.padded_cols + 16u * g);
#pragma unroll
  for (int k = 0; k < 4; ++k) dst[k] = make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
}

// ------------------------------------------------------------ K0 unpack
__global__ void unpack_kernel(const uint8_t* __restrict__ quads, Geometry G, uint8_t* codes2,
                              uint8_t* zeros2, uint8_t* scodes, uint8_t* codes4) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)G.rows * G.G) return;
  const uint32_t r = (uint32_t)(tid / G.G), g = (uint32_t)(tid % G.G);
  const uint8_t* qr = quads + (size_t)(r / kRowsPerQuad) * G.dense_bytes;
  const uint32_t i = r % kRowsPerQuad;
  if (g < G.G2) {
    const uint32_t word = *reinterpret_cast<const uint32_t*>(qr + 16u * g + 4u * i);
    const uint32_t t = g / 3u, sub = g - 3u * t;
    const uint32_t meta = *reinterpret_cast<const uint16_t*>(qr + G.off_meta + 8u * t + 2u * i);
    for (int k = 0; k < 16; ++k) codes2[(size_t)r * G.n2p + 16u * g + k] = (word >> (2 * k)) & 3u;
    zeros2[(size_t)r * G.G2 + g] = (meta >> (2 * sub)) & 3u;
    scodes[(size_t)r * G.G2 + g] = sub == 0 ? (meta >> 6) & 15u : (meta >> (sub == 1 ? 10 : 13)) & 7u;
  } else {
    const uint32_t b = g - G.G2;
    const uint32_t w0 = *reinterpret_cast<const uint32_t*>(qr + G.off_c4 + 32u * b + 4u * i);
    const uint32_t w1 = *reinterpret_cast<const uint32_t*>(qr + G.off_c4 + 32u * b + 16u + 4u * i);
    for (int k = 0; k < 8; ++k) {
      codes4[(size_t)r * G.n4 + 16u * b + k] = (w0 >> (4 * k)) & 15u;
      codes4[(size_t)r * G.n4 + 16u * b + 8 + k] = (w1 >> (4 * k)) & 15u;
    }
  }
}

cudaError_t launch_ex(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      bool pdl, void** params) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelExC(&cfg, fn, params);
}

}  // namespace

int launch_prologue(const DeviceLayer& L, const float* x, uint32_t batch, const Workspace& ws,
                    void* stream, bool pdl) {
  const Geometry& G = L.g;
  const uint32_t threads = 256;
  dim3 grid((G.G * 16u + threads - 1) / threads, batch);
  uint32_t cols = G.cols, g2 = G.G2, gg = G.G, bs = ws.block_stride, xs = ws.xp_stride;
  uint8_t* xprep = ws.xprep;
  float* xp = ws.xp;
  uint32_t* flags = ws.flags;
  const uint32_t* perm = L.perm;
  void* params[] = {(void*)&x, (void*)&perm, &cols, &g2, &gg, &xprep, &bs, &xp, &xs, &flags};
  return (int)launch_ex((const void*)prologue_kernel, grid, dim3(threads), 0, (cudaStream_t)stream,
                        pdl, params);
}

int launch_gemv(const DeviceLayer& L, uint32_t batch, float* y, const Workspace& ws, void* stream,
                bool pdl, int num_sms) {
  const Geometry& G = L.g;
  GemvArgs a = {};
  a.quads = L.quads;
  a.sorder = L.sorder;
  a.row_ptr = L.row_ptr;
  a.csr = L.csr;
  a.g = G;
  a.nchunks = (G.G + 31u) / 32u;
  a.grid = min((uint32_t)num_sms, G.quads);
  a.nq_max = (G.quads + a.grid - 1) / a.grid;
  a.uniform_rb = (G.group2 % kRowsPerQuad) == 0;
  a.sorder_off = (G.dense_bytes + 15u) & ~15u;
  a.sorder_bytes_max = G.max_rb_per_quad * G.G2s * 4u;
  a.slot_stride = (a.sorder_off + a.sorder_bytes_max + 127u) & ~127u;
  a.xprep_bytes = XprepLayout{G.G}.block_bytes();
  a.xregion = (a.xprep_bytes + 127u) & ~127u;
  // shared memory: xprep | slots | partials | csr partials + counters | barriers
  auto need = [&](size_t nslot) {
    return (size_t)a.xregion + nslot * a.slot_stride + nslot * a.nchunks * 16u +
           (size_t)a.nq_max * 20u + 8u + (2 * nslot + 1) * 8u;
  };
  // two CTAs per SM (so a PDL successor can co-reside) when >= 3 slots fit in
  // half the SM, otherwise one CTA with the whole carve-out
  size_t nslot = 16;
  if (nslot > a.nq_max) nslot = a.nq_max;
  const size_t half_sm = 110 * 1024, full_sm = 220 * 1024;
  size_t budget = need(std::min<size_t>(nslot, 3)) <= half_sm ? half_sm : full_sm;
  while (nslot > 1 && need(nslot) > budget) --nslot;
  if (need(nslot) > full_sm) return (int)cudaErrorInvalidConfiguration;
  a.nslot = (uint32_t)nslot;
  const size_t smem = need(nslot);
  cudaError_t err = cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
  if (err != cudaSuccess) return (int)err;
  for (uint32_t col = 0; col < batch; ++col) {
    GemvArgs b = a;
    b.xprep = ws.xprep + (size_t)col * ws.block_stride;
    b.xp = ws.xp + (size_t)col * ws.xp_stride;
    b.y = y + (size_t)col * G.rows;
    void* params[] = {&b};
    err = launch_ex((const void*)gemv_kernel, dim3(a.grid), dim3(kGemvThreads), smem,
                    (cudaStream_t)stream, pdl, params);
    if (err != cudaSuccess) return (int)err;
  }
  return 0;
}

int launch_dequant(const DeviceLayer& L, float* w, void* stream) {
  const uint64_t n = (uint64_t)L.g.rows * L.g.G;
  const uint32_t threads = 256;
  dequant_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      L.quads, L.sorder, L.g, w);
  return (int)cudaGetLastError();
}

int launch_unpack(const DeviceLayer& L, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes,
                  uint8_t* codes4, void* stream) {
  const uint64_t n = (uint64_t)L.g.rows * L.g.G;
  const uint32_t threads = 256;
  unpack_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      L.quads, L.g, codes2, zeros2, scodes, codes4);
  return (int)cudaGetLastError();
}

}  // namespace qwdev
