// qw_gemv_common.cuh -- device helpers shared by the batch-1 kernels
// (gemv_kernel in qw_gemv.cu, chain_kernel in qw_chain.cu): fp32x2 / fp16x2
// arithmetic, the subnormal-code dot products, the exact fp16 1st-order
// scale, the reduction-window layout; host plan helpers.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "qw_device.hpp"
#include "qw_ptx.cuh"

namespace qwdev {
namespace {

// ------------------------------------------------------------ fp32x2
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float pow2f(int e) {  // 2^e for -126 <= e <= 127
  return __uint_as_float((uint32_t)(e + 127) << 23);
}
__device__ __forceinline__ float2 h2f2(uint32_t h) { return __half22float2(as_h2(h)); }

// ------------------------------------------------------------ unpack + dot
// 2-bit row pair: w0 = channels 0-7 of rows A|B, w1 = channels 8-15; channel
// j of a half at bits 2j.  X[k] = {x'_k, x'_k} 2^-2(k%4).  Two 8-long HFMA2
// chains; returns the fp16 pair {sum c x' 2^-24 for row A, for row B}.
__device__ __forceinline__ half2 dot2(uint32_t w0, uint32_t w1, const half2* X) {
  const uint32_t h0 = w0 >> 8, h1 = w1 >> 8;
  half2 a = __hmul2(as_h2(w0 & 0x00030003u), X[0]);
  half2 b = __hmul2(as_h2(w1 & 0x00030003u), X[8]);
  a = __hfma2(as_h2(w0 & 0x000C000Cu), X[1], a);
  b = __hfma2(as_h2(w1 & 0x000C000Cu), X[9], b);
  a = __hfma2(as_h2(w0 & 0x00300030u), X[2], a);
  b = __hfma2(as_h2(w1 & 0x00300030u), X[10], b);
  a = __hfma2(as_h2(w0 & 0x00C000C0u), X[3], a);
  b = __hfma2(as_h2(w1 & 0x00C000C0u), X[11], b);
  a = __hfma2(as_h2(h0 & 0x00030003u), X[4], a);
  b = __hfma2(as_h2(h1 & 0x00030003u), X[12], b);
  a = __hfma2(as_h2(h0 & 0x000C000Cu), X[5], a);
  b = __hfma2(as_h2(h1 & 0x000C000Cu), X[13], b);
  a = __hfma2(as_h2(h0 & 0x00300030u), X[6], a);
  b = __hfma2(as_h2(h1 & 0x00300030u), X[14], b);
  a = __hfma2(as_h2(h0 & 0x00C000C0u), X[7], a);
  b = __hfma2(as_h2(h1 & 0x00C000C0u), X[15], b);
  return __hadd2(a, b);
}
// 4-bit row pair: word j = channels 4j..4j+3 of rows A|B, nibble i of a half
// at bits 4i.  X[k] = {x'_k, x'_k} 2^-4(k%2).
__device__ __forceinline__ half2 dot4(uint4 w, const half2* X) {
  // chain a: channels 0-7 (w.x, w.y); chain b: channels 8-15 (w.z, w.w)
  const uint32_t ha0 = w.x >> 8, hb0 = w.z >> 8, ha1 = w.y >> 8, hb1 = w.w >> 8;
  half2 a = __hmul2(as_h2(w.x & 0x000F000Fu), X[0]);
  half2 b = __hmul2(as_h2(w.z & 0x000F000Fu), X[8]);
  a = __hfma2(as_h2(w.x & 0x00F000F0u), X[1], a);
  b = __hfma2(as_h2(w.z & 0x00F000F0u), X[9], b);
  a = __hfma2(as_h2(ha0 & 0x000F000Fu), X[2], a);
  b = __hfma2(as_h2(hb0 & 0x000F000Fu), X[10], b);
  a = __hfma2(as_h2(ha0 & 0x00F000F0u), X[3], a);
  b = __hfma2(as_h2(hb0 & 0x00F000F0u), X[11], b);
  a = __hfma2(as_h2(w.y & 0x000F000Fu), X[4], a);
  b = __hfma2(as_h2(w.w & 0x000F000Fu), X[12], b);
  a = __hfma2(as_h2(w.y & 0x00F000F0u), X[5], a);
  b = __hfma2(as_h2(w.w & 0x00F000F0u), X[13], b);
  a = __hfma2(as_h2(ha1 & 0x000F000Fu), X[6], a);
  b = __hfma2(as_h2(hb1 & 0x000F000Fu), X[14], b);
  a = __hfma2(as_h2(ha1 & 0x00F000F0u), X[7], a);
  b = __hfma2(as_h2(hb1 & 0x00F000F0u), X[15], b);
  return __hadd2(a, b);
}

// ------------------------------------------------------------ helpers
// acc += float(a) * float(b) for fp16 halves, one rounding (sm_100 mixed FMA)
__device__ __forceinline__ float fhfma_lo(half2 a, half2 b, float c) {
  float d;
  asm("{.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.f16 %0, al, bl, %3;}"
      : "=f"(d)
      : "r"(*reinterpret_cast<uint32_t*>(&a)), "r"(*reinterpret_cast<uint32_t*>(&b)), "f"(c));
  return d;
}
__device__ __forceinline__ float fhfma_hi(half2 a, half2 b, float c) {
  float d;
  asm("{.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.f16 %0, ah, bh, %3;}"
      : "=f"(d)
      : "r"(*reinterpret_cast<uint32_t*>(&a)), "r"(*reinterpret_cast<uint32_t*>(&b)), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t pack_h2(float2 v) {  // cvt.rn.f16x2.f32
  const half2 h = __float22half2_rn(v);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// 1st-order scales of a row pair (the 2-order dequant, engine.cpp:48-63):
// s1 = (eff - zero2) * scale2 2^-P rounded once to fp16.  The masked field
// eff 2^pe ORed into the fp16 1024 (0x6400) reads 1024 + eff 2^pe exactly; one
// HFMA2 with p2 = 2^-pe, c2 = -(2^(10 - pe) + zero2) leaves eff - zero2 exactly,
// one HMUL2 by a2 = scale2 2^-P (an fp16 value) rounds the exact product once
// -- the same fp16 as forming it in fp32 and converting.
__device__ __forceinline__ uint32_t s1_pair(uint32_t mm, uint32_t emask, half2 p2, half2 c2, half2 a2) {
  const half2 d = __hfma2(as_h2((mm & emask) | 0x64006400u), p2, c2);
  const half2 r = __hmul2(d, a2);
  return *reinterpret_cast<const uint32_t*>(&r);
}
__device__ __forceinline__ half2 h2_of(float lo, float hi) { return __floats2half2_rn(lo, hi); }

// Per-warp reduction window of 16 rows: lane l stores its partials of rows
// r..r+3 at win[wbase(l) + r] (16-byte stores, conflict-free per quarter
// warp), wbase(l) = 20 l + 16 (l >> 3).  When the window is full, lane l sums
// the row pair 2 (l & 7), +1 over source lanes 8 (l >> 3) .. +7 (8-byte reads:
// the two source groups of a half-warp sit 16 banks apart), two shuffles join
// the four source groups (a fixed tree: deterministic).
constexpr uint32_t kWinRows = 16, kWinWords = 688;
__device__ __forceinline__ uint32_t win_base(uint32_t l) { return l * 20u + (l >> 3) * 16u; }

// ------------------------------------------------------------ host helpers
uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* e = knob_str(name);
  return e ? (uint32_t)std::atoi(e) : dflt;
}
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace
}  // namespace qwdev
