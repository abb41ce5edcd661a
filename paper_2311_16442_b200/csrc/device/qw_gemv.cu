// qw_gemv.cu -- the hot path: y = W_q x for the mixed 2/4-bit layer (batch 1),
// one fused kernel per activation column.
//
// Reference semantics: matvec_oracle (engine.cpp:169-183) over the stages
// row_fetch_params / row_compute_scales / row_decode / row_fma
// (engine.cpp:40-122), the activation gather of checked_permute /
// apply_permutation (engine.cpp:124-132, plan.cpp:107-116) and the CSR
// outliers of sparse_matvec (outliers.cpp:131-141).
//
// CTA (persistent, one per SM, a contiguous range of 4-row quad records;
// small enough that the next layer's CTA sits beside it under programmatic
// dependent launch):
//   producer warp  TMA bulk copies: the CTA's 2-order rows once, then one
//                  quad record per ring slot.  It never waits on the
//                  previous kernel, so the weight stream of layer i+1
//                  starts while layer i still computes.
//   csr warp       the CTA's outliers: exact fp32 products with x, summed per
//                  row in CSR order.
//   T teams of W consumer warps.  Team t takes quads t, t+T, ...; inside a
//                  team lane l of warp w owns the groups (w + k W) * 32 + l,
//                  k < KG, for every quad, so the group's 16 activations stay
//                  in registers (prepared once: permuted, fp16, pre-scaled)
//                  and the 2-order scales of its group are re-read only when
//                  the quad enters a new 2-order row block.  Per quad a lane
//                  produces 4 row partials, one transpose-reduce over the
//                  warp leaves 4 row sums, and the CTA sums the W warps of a
//                  quad in a fixed order at the end (deterministic).
//
// Code unpack: a code masked into an fp16 whose exponent field is zero reads
// as c * 2^(bitpos-24) exactly (a subnormal).  Rows 2p and 2p+1 share each
// 32-bit word (qw_layout.hpp), so one LOP3 + one HFMA2 multiplies one channel
// of two rows by x'_k pre-scaled by 2^-bitpos; every product is c x' 2^-24
// and the accumulator's two halves are the two rows.  Zero points:
// sum((c - z) x') = sum(c x') - z sum(x'), applied with one HFMA2 per row
// pair; the 1st-order scale s1 = (eff - zero2) * scale2 (the 2-order
// dequant, engine.cpp:48-63) is formed exactly in fp32 per (row, group) and
// applied with packed fp32x2 FMAs.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <type_traits>
#include <vector>

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

// ------------------------------------------------------------ K2+K3 GEMV
struct GemvArgs {
  // per layer (segment) of the launch
  const uint8_t* quads[kMaxSeg];
  const uint32_t* sorder[kMaxSeg];
  const uint32_t* row_ptr[kMaxSeg];
  const uint32_t* csr[kMaxSeg];
  const uint16_t* perm[kMaxSeg];
  float* y[kMaxSeg];
  float s_scale[kMaxSeg];  // 2^-P: keeps (eff - zero2) scale2 2^-P inside fp16
  const float* x;
  Geometry g;
  uint32_t W, W2, T, S, grid, nq_max;  // warps per team, 2-bit warps, teams, ring slots
  uint32_t rb_magic, rb_one;  // row / group2 = rb_one ? row : umulhi(row, rb_magic)
  uint32_t repeat;  // diagnostics: consumers re-run the resident quads this many times
  uint32_t wait_x;  // x is the previous kernel's output: griddepcontrol.wait before reading it
  uint32_t pre;     // precompute 1st-order scales of resident units before x
  uint32_t npre_max;  // at most this many units precomputed
  uint32_t x_gate;    // the producer issues this many units, then waits for x
  uint32_t x_first; // stage x before the scale precompute (no predecessor overlap)
  uint32_t so_off, part_off, csr_off, x_off, win_off, pre_off, bar_off;
  uint32_t ent_off, csr_stage;  // the CTA's CSR entries staged in shared memory by one bulk copy
  const uint8_t* pf_ptr[GemvPlan::kMaxPf];  // next launch's weights -> L2 (a slice per CTA)
  uint32_t pf_bytes[GemvPlan::kMaxPf], pf_n, pf_late;
  unsigned long long* dbg;  // optional timeline: kTimelineEvents stamps per CTA
  uint32_t dbg_global;      // stamps from %globaltimer (ns) instead of clock64
  uint8_t cta_seg[kMaxGrid];
  uint32_t cta_q0[kMaxGrid], cta_q1[kMaxGrid], cta_e0[kMaxGrid], cta_e1[kMaxGrid];
};

__device__ __forceinline__ void stamp_impl(const GemvArgs& a, uint32_t ev) {
  unsigned long long t;
  if (a.dbg_global)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  else
    t = clock64();
  a.dbg[blockIdx.x * kTimelineEvents + ev] = t;
}
#define stamp(DBG, EV) \
  do {                 \
    if (DBG) stamp_impl(a, EV); \
  } while (0)

// Per-warp reduction window of 16 rows: lane l stores its partials of rows
// r..r+3 at win[wbase(l) + r] (16-byte stores, conflict-free per quarter
// warp), wbase(l) = 20 l + 16 (l >> 3).  When the window is full, lane l sums
// the row pair 2 (l & 7), +1 over source lanes 8 (l >> 3) .. +7 (8-byte reads:
// the two source groups of a half-warp sit 16 banks apart), two shuffles join
// the four source groups (a fixed tree: deterministic).
constexpr uint32_t kWinRows = 16, kWinWords = 688;
__device__ __forceinline__ uint32_t win_base(uint32_t l) { return l * 20u + (l >> 3) * 16u; }

// KG groups per lane, NQ quads per ring slot (decoded together for ILP),
// UNI: group2 % 4 == 0 (a quad never straddles 2-order blocks), XSM: x is
// staged in shared memory (TMA) before the gather.
// TM: two teams of consumer warps take alternate units (long quad ranges:
// group launches, wide layers); then the CTA owns the SM (no PDL co-residency).
template <int KG, int NQ, bool UNI, bool XSM, bool TM = false>
__global__ void __launch_bounds__(TM ? 576 : (KG <= 2 ? 320 : 544), (TM || KG > 2) ? 1 : 2)
    gemv_kernel(const __grid_constant__ GemvArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Geometry& G = a.g;
  const uint32_t W = a.W, T = TM ? a.T : 1u, NC = W * T, S = a.S, dense = G.dense_bytes;
  const uint32_t* s_so = reinterpret_cast<const uint32_t*>(smem + a.so_off);
  float* s_part = reinterpret_cast<float*>(smem + a.part_off);  // [row][warp]
  float* s_csr = reinterpret_cast<float*>(smem + a.csr_off);
  uint32_t* s_rp = reinterpret_cast<uint32_t*>(s_csr + a.nq_max * 4);
  float* s_prod = reinterpret_cast<float*>(s_rp + a.nq_max * 4 + 4);
  float* s_red = s_prod + 256;  // [warp] max |x|
  float* s_x = reinterpret_cast<float*>(smem + a.x_off);
  uint2* s_pre = reinterpret_cast<uint2*>(smem + a.pre_off);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* s_empty = s_full + S;
  uint64_t* s_sobar = s_empty + S;
  uint64_t* s_xbar = s_sobar + 1;
  uint64_t* s_cbar = s_xbar + 1;

  const uint32_t seg = a.cta_seg[blockIdx.x];
  const uint32_t q0 = a.cta_q0[blockIdx.x], q1 = a.cta_q1[blockIdx.x];
  const uint32_t nq = q1 - q0;
  const uint8_t* __restrict__ g_quads = a.quads[seg];
  const uint32_t* __restrict__ g_sorder = a.sorder[seg];
  const uint32_t* __restrict__ g_row_ptr = a.row_ptr[seg];
  const uint32_t* __restrict__ g_csr = a.csr[seg];
  const uint16_t* __restrict__ g_perm = a.perm[seg];
  float* __restrict__ g_y = a.y[seg];
  const float s_scale = a.s_scale[seg];
  const uint32_t nunit = (nq + NQ - 1) / NQ;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t r_begin = q0 * kRowsPerQuad;
  const uint32_t r_end = min(q1 * kRowsPerQuad, G.rows);
  const uint32_t nrows = r_end - r_begin;
  auto row_block = [&](uint32_t r) { return a.rb_one ? r : __umulhi(r, a.rb_magic); };
  const uint32_t rb_first = row_block(r_begin);

  if (threadIdx.x < S) {
    mbar_init(&s_full[threadIdx.x], 1);
    mbar_init(&s_empty[threadIdx.x], W);  // one team consumes a unit
  }
  if (threadIdx.x == 32) mbar_init(s_sobar, 1), mbar_init(s_xbar, NC), mbar_init(s_cbar, 1);
  if (XSM && threadIdx.x == 64) s_x[G.cols] = 0.0f;  // pads gather this zero (perm16 = cols)
  if (threadIdx.x == 0) stamp(a.dbg, 0);  // entry
  mbar_fence_init();
  __syncthreads();
  pdl_launch_dependents();

  if (warp == NC) {
    // ================= producer: the weight stream does not depend on x
    if (lane == 0) {
      const uint32_t so_bytes = nrows ? (row_block(r_end - 1) - rb_first + 1) * G.G2s * 4u : 0u;
      if (so_bytes) {
        mbar_expect_tx(s_sobar, so_bytes);
        bulk_load_nohint(smem + a.so_off, g_sorder + (size_t)rb_first * G.G2s, so_bytes, s_sobar);
      } else {
        mbar_arrive(s_sobar);
      }
      if (a.csr_stage) {  // the CTA's outlier entries (x-independent): one bulk copy
        const uint32_t e_lo = a.cta_e0[blockIdx.x], e_hi = a.cta_e1[blockIdx.x];
        const uint32_t shift = e_lo & 3u, bytes = ((e_hi - e_lo + shift) * 4u + 15u) & ~15u;
        if (e_hi > e_lo) {
          mbar_expect_tx(s_cbar, bytes);
          bulk_load_nohint(smem + a.ent_off, g_csr + (e_lo - shift), bytes, s_cbar);
        } else {
          mbar_arrive(s_cbar);
        }
      }
      const uint8_t* src = g_quads + (size_t)q0 * dense;
      // L2 prefetch of this CTA's slice of the next launch's weights, issued
      // in step with the own units so the ring refills never queue behind it
      uint32_t pf_r = 0, pf_pos = 0, pf_end = 0;
      uint64_t pf_total = 0, pf_done = 0;
      for (uint32_t r = 0; r < a.pf_n; ++r) pf_total += a.pf_bytes[r] / a.grid / 16u * 16u;
      auto pf_region = [&](uint32_t r) {  // this CTA's 16-byte aligned slice of region r
        const uint32_t per = a.pf_bytes[r] / a.grid / 16u * 16u;
        pf_pos = per * blockIdx.x;
        pf_end = blockIdx.x + 1 == a.grid ? a.pf_bytes[r] / 16u * 16u : pf_pos + per;
      };
      if (a.pf_n) pf_region(0);
      auto prefetch_upto = [&](uint64_t target) {
        while (pf_done < target && pf_r < a.pf_n) {
          if (pf_pos >= pf_end) {
            if (++pf_r < a.pf_n) pf_region(pf_r);
            continue;
          }
          const uint32_t n = min(pf_end - pf_pos, 32768u);
          bulk_prefetch_l2(a.pf_ptr[pf_r] + pf_pos, n);
          pf_pos += n, pf_done += n;
        }
      };
      // never gate below the units the consumers precompute before x (deadlock)
      const uint32_t x_gate = max(a.x_gate, (!TM && a.pre) ? min(min(nunit, S), a.npre_max) : 0u);
      uint32_t slot = 0, phase = 0;
      for (uint32_t u = 0; u < nunit; ++u) {
        const uint32_t bytes = min((uint32_t)NQ, nq - NQ * u) * dense;
        // after the first units, hold the stream until x is staged: x then
        // is not queued behind this SM's whole weight range
        if (XSM && u == x_gate) mbar_wait(s_xbar, 0);
        if (u >= S) mbar_wait(&s_empty[slot], phase ^ 1u);
        mbar_expect_tx(&s_full[slot], bytes);
        bulk_load_nohint(smem + (size_t)slot * NQ * dense, src, bytes, &s_full[slot]);
        src += bytes;
        if (++slot == S) slot = 0, phase ^= 1u;
        if (!a.pf_late) prefetch_upto(pf_total * (u + 1) / nunit);
      }
      prefetch_upto(~0ull);
    }
    return;
  }

  if (warp == NC + 1) {
    // ================= outliers: exact fp32 x, CSR order within a row
    const uint32_t e_lo = a.cta_e0[blockIdx.x], e_hi = a.cta_e1[blockIdx.x];
    for (uint32_t t = lane; t <= nrows; t += 32) s_rp[t] = g_row_ptr[r_begin + t] - e_lo;
    for (uint32_t t = lane; t < nrows; t += 32) s_csr[t] = 0.0f;
    const uint32_t n = e_hi - e_lo;
    constexpr int kPer = 8;
    uint32_t ent[kPer], src[kPer];
    const uint32_t* s_ent = reinterpret_cast<const uint32_t*>(smem + a.ent_off) + (e_lo & 3u);
    if (a.csr_stage) {
      // entries staged by the producer: one row per lane, entries in CSR
      // order, product then sum (outliers.cpp:131-141), no chunk barriers
      __syncwarp();  // s_rp
      if (n) {
        mbar_wait(s_cbar, 0);
        if (XSM) mbar_wait(s_xbar, 0);
        else if (a.wait_x) pdl_wait();
      }
      for (uint32_t t = lane; t < nrows; t += 32) {
        const uint32_t lo = s_rp[t], hi = s_rp[t + 1];
        float acc = 0.0f;
        uint32_t e = lo;
        for (; e + 4 <= hi; e += 4) {  // loads of 4 entries in flight, sums in order
          uint32_t w[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) w[j] = s_ent[e + j];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float xv = XSM ? s_x[w[j] & 0xFFFFu] : __ldg(a.x + (w[j] & 0xFFFFu));
            acc = __fadd_rn(acc, __fmul_rn(half_bits_to_float(w[j] >> 16), xv));  // no contraction
          }
        }
        for (; e < hi; ++e) {
          const uint32_t w = s_ent[e];
          acc = __fadd_rn(acc, __fmul_rn(half_bits_to_float(w >> 16), XSM ? s_x[w & 0xFFFFu] : __ldg(a.x + (w & 0xFFFFu))));
        }
        s_csr[t] = acc;
      }
      if (lane == 0) stamp(a.dbg, 6);  // outliers done
      named_sync(2, (NC + 1) * 32);    // meet the consumers for the y store
      return;
    }
    auto fetch = [&](uint32_t c0) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint32_t e = c0 + lane + 32u * j;
        ent[j] = e < n ? (a.csr_stage ? s_ent[e] : __ldg(g_csr + e_lo + e)) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kPer; ++j) src[j] = ent[j] & 0xFFFFu;  // original channel (repack)
    };
    if (n) fetch(0);
    __syncwarp();
    // x: the shared-memory copy once it lands (XSM), else global after the
    // dependency wait (x is the previous kernel's output)
    if (n) {
      if (XSM)
        mbar_wait(s_xbar, 0);
      else if (a.wait_x)
        pdl_wait();
    }
    uint32_t t0 = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += 32u * kPer) {
      const uint32_t c1 = min(c0 + 32u * kPer, n);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint32_t e = c0 + lane + 32u * j;
        if (e < c1) s_prod[e - c0] = half_bits_to_float(ent[j] >> 16) * (XSM ? s_x[src[j]] : __ldg(a.x + src[j]));
      }
      __syncwarp();
      if (c1 < n) fetch(c1);
      // rows the chunk touches: [t0, ...) with rp[t0 + 1] > c0 (warp ballot advance)
      for (;;) {
        const uint32_t t = t0 + lane;
        const uint32_t done = __ballot_sync(0xFFFFFFFFu, t < nrows && s_rp[t + 1] <= c0);
        t0 += __popc(done);
        if (done != 0xFFFFFFFFu) break;
      }
      for (uint32_t t = t0 + lane; t < nrows && s_rp[t] < c1; t += 32) {
        const uint32_t lo = max(s_rp[t], c0), hi = min(s_rp[t + 1], c1);
        float s = s_csr[t];
        for (uint32_t e = lo; e < hi; ++e) s += s_prod[e - c0];  // CSR order within the row
        s_csr[t] = s;
      }
      __syncwarp();
    }
    if (lane == 0) stamp(a.dbg, 6);  // outliers done
    named_sync(2, (NC + 1) * 32);    // meet the consumers for the y store
    return;
  }

  // ================= consumers.  Warps [0, W2) own 2-bit chunks, [W2, W) own
  // 4-bit chunks, so the group type is warp-uniform; lane l of a 2-bit warp
  // owns groups (w + k W2) * 32 + l, of a 4-bit warp blocks (w - W2 + k W4) * 32 + l.
  // A dead lane (past the last group of its type) decodes a real group with
  // X = 0, so it contributes exact zeros without a branch in the loop.
  const uint32_t W2 = a.W2, W4 = W - W2;
  const uint32_t team = warp / W, wt = warp - team * W;  // warp within its team
  const bool two = wt < W2;
  uint32_t gk[KG];
  bool lv[KG];
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    if (two) {
      const uint32_t g = (wt + (uint32_t)k * W2) * 32u + lane;
      lv[k] = g < G.G2;
      gk[k] = lv[k] ? g : G.G2 - 1u;
    } else {
      const uint32_t b = (wt - W2 + (uint32_t)k * W4) * 32u + lane;
      lv[k] = b < G.T4;
      gk[k] = G.G2 + (lv[k] ? b : G.T4 - 1u);
    }
  }
  float* win = reinterpret_cast<float*>(smem + a.win_off) + warp * kWinWords;
  const uint32_t reps = (a.repeat > 1 && nunit <= S) ? a.repeat : 1;
  // units whose scales are precomputed before x (they must have landed first:
  // capped so the main loop can start under the rest of the weight stream)
  const uint32_t npre = (!TM && a.pre) ? min(min(nunit, S), a.npre_max) : 0u;  // team kernels: never (policy)

  // One consumer body per group type (warp-uniform), per-lane constants hoisted.
  auto run = [&](auto two_tag) {
    constexpr bool TWO = decltype(two_tag)::value;
    uint32_t off_c[KG], off_p[KG], off_z[KG], zmask[KG], esh[KG], emask[KG];
    int pe[KG];
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint32_t g = gk[k];
      if (TWO) {
        const uint32_t t = g / 3u, sub = g - 3u * t;
        off_c[k] = 16u * g;
        off_p[k] = G.off_meta + 8u * t;
        off_z[k] = 0;
        zmask[k] = 0x00030003u << (2u * sub);
        // 4/3/3 rule (quantizer.cpp:103-104): eff = scode for sub 0, scode << 1 else;
        // the masked field reads as eff 2^(pe - 24)
        esh[k] = sub == 0 ? 0u : 7u;
        emask[k] = sub == 0 ? 0x03C003C0u : (sub == 1 ? 0x00380038u : 0x01C001C0u);
        pe[k] = sub == 0 ? 6 : (sub == 1 ? 2 : 5);
      } else {
        const uint32_t b = g - G.G2;
        off_c[k] = G.off_c4 + 32u * b;
        off_p[k] = G.off_s4 + 8u * b;
        off_z[k] = G.off_z4 + 2u * b;
        zmask[k] = esh[k] = emask[k] = 0;
        pe[k] = 0;
      }
    }
    // ---- 1st-order scales of the lane's 2-bit groups (the 2-order dequant,
    // engine.cpp:48-63): s1 = (eff - zero2) * scale2, exact in fp32, kept as
    // fp16 (x 2^-P) for the mixed-precision FMA.  x-independent.
    half2 A2[NQ][KG][UNI ? 1 : 2], C2[NQ][KG][UNI ? 1 : 2], P2[KG];
#pragma unroll
    for (int k = 0; k < KG; ++k) P2[k] = __float2half2_rn(pow2f(-pe[k]));
    uint32_t rb_end[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) rb_end[j] = 0;
    auto load_scales = [&](int j, uint32_t r0) {
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        float A[4], Cz[4];
#pragma unroll
        for (int i = 0; i < (UNI ? 1 : 4); ++i) {
          const uint32_t rb = row_block(min(r0 + i, G.rows - 1)) - rb_first;
          const uint32_t e = s_so[rb * G.G2s + gk[k]];
          A[i] = half_bits_to_float(e) * s_scale;  // exact: scale2 * 2^-P
          Cz[i] = -(pow2f(10 - pe[k]) + small_int_to_float(e >> 16));
        }
        if (UNI) {
          A2[j][k][0] = __float2half2_rn(A[0]), C2[j][k][0] = __float2half2_rn(Cz[0]);
        } else {
          A2[j][k][0] = h2_of(A[0], A[1]), C2[j][k][0] = h2_of(Cz[0], Cz[1]);
          A2[j][k][UNI ? 0 : 1] = h2_of(A[2], A[3]), C2[j][k][UNI ? 0 : 1] = h2_of(Cz[2], Cz[3]);
        }
      }
    };
    // s1 of rows {0,1} and {2,3} of quad j of the unit in slot base sb, group k
    auto scales_of = [&](const uint8_t* sb, int j, int k, uint32_t u) -> uint2 {
      const uint32_t r0 = (q0 + u * NQ + j) * kRowsPerQuad;
      if (!UNI || r0 >= rb_end[j]) {
        load_scales(j, r0);
        rb_end[j] = (row_block(r0) + 1) * G.group2;
      }
      const uint2 m = *reinterpret_cast<const uint2*>(sb + j * dense + off_p[k]);
      const int i1 = UNI ? 0 : 1;
      return make_uint2(s1_pair(m.x >> esh[k], emask[k], P2[k], C2[j][k][0], A2[j][k][0]),
                        s1_pair(m.y >> esh[k], emask[k], P2[k], C2[j][k][i1], A2[j][k][i1]));
    };
    auto pre_at = [&](uint32_t slot, int j, int k) -> uint2& {
      return s_pre[((slot * NQ + j) * KG + k) * (W * 32) + wt * 32 + lane];
    };

    // ---- x (the previous kernel's output) -> shared memory: coalesced loads
    // spread over every consumer thread (not queued behind the weight TMAs).
    // x_first (the CTA starts after its predecessor finished, e.g. it cannot
    // co-reside with it): the loads are issued first and land under the
    // scale decode below; else after it (the decode overlaps the predecessor).
    const uint32_t tid = threadIdx.x, nth = NC * 32u;
    const bool xvec = (((uintptr_t)a.x) & 15u) == 0 && (G.cols & 3u) == 0;
    const float4* gx = reinterpret_cast<const float4*>(a.x);
    float4* sx4 = reinterpret_cast<float4*>(s_x);
    const uint32_t n4 = G.cols >> 2;
    constexpr int kXr = 4;
    float4 xr[kXr];
    auto x_issue = [&]() {
      if (a.wait_x) pdl_wait();
      if (threadIdx.x == 0) stamp(a.dbg, 1);  // dependency resolved
      if (xvec) {
#pragma unroll
        for (int j = 0; j < kXr; ++j)
          if (tid + j * nth < n4) xr[j] = __ldg(gx + tid + j * nth);
      }
    };
    auto x_store = [&]() {
      if (xvec) {
#pragma unroll
        for (int j = 0; j < kXr; ++j)
          if (tid + j * nth < n4) sx4[tid + j * nth] = xr[j];
        // the rest (wide layers): 4 loads in flight per batch
        for (uint32_t i = tid + kXr * nth; i < n4; i += 4 * nth) {
          float4 v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (i + j * nth < n4) v[j] = __ldg(gx + i + j * nth);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (i + j * nth < n4) sx4[i + j * nth] = v[j];
        }
      } else {
        for (uint32_t i = tid; i < G.cols; i += nth) s_x[i] = __ldg(a.x + i);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(s_xbar);
    };
    if (XSM && a.x_first) x_issue();

    // ---- asynchronous dequantization: while the previous layer still runs
    // (its output x is not needed yet), decode the 1st-order scales of every
    // resident unit.
    if (TWO) {
      mbar_wait(s_sobar, 0);
      for (uint32_t u = team; u < npre; u += T) {
        mbar_wait(&s_full[u], 0);
        const uint8_t* sb = smem + (size_t)u * NQ * dense;
#pragma unroll
        for (int j = 0; j < NQ; ++j)
#pragma unroll
          for (int k = 0; k < KG; ++k) pre_at(u, j, k) = scales_of(sb, j, k, u);
      }
    }

    // ---- activation prologue: gather the lane's groups in permuted order and
    // scale them by a per-warp power of two (max|x'| in [2^10, 2^11): every
    // fp16 x' keeps 11 bits, the group sums of |x'| stay < 2^15).  The warp's
    // row sums share that scale, undone once per row in the reduction window,
    // so no CTA-wide reduction sits on the critical path.
    uint32_t pw[KG][8];
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint4* pp = reinterpret_cast<const uint4*>(g_perm + 16u * gk[k]);
      const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
      pw[k][0] = p0.x, pw[k][1] = p0.y, pw[k][2] = p0.z, pw[k][3] = p0.w;
      pw[k][4] = p1.x, pw[k][5] = p1.y, pw[k][6] = p1.z, pw[k][7] = p1.w;
    }
    if (threadIdx.x == 0) stamp(a.dbg, 8);  // x-independent work done
    const float* xs;
    if (XSM) {
      if (!a.x_first) x_issue();
      x_store();
      mbar_wait(s_xbar, 0);
      if (threadIdx.x == 0) stamp(a.dbg, 7);  // x landed
      xs = s_x;
    } else {
      if (a.wait_x) pdl_wait();  // x is the previous kernel's output
      xs = a.x;
    }
    // Two teams need the same X: team 0 prepares it and hands it to team 1
    // through team 1's (not yet used) reduction windows.
    half2 X[KG][16], nsxh[KG];
    float yscale;
    const bool share = TM && KG == 1 && T == 2;
    uint32_t* xsh = reinterpret_cast<uint32_t*>(smem + a.win_off) + (W + wt) * kWinWords + lane * 20u;
    if (!share || team == 0) {
    const uint32_t n2 = G.cols - G.n4;
    float xv[KG][16];
    float mx = 0.0f;
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint32_t s0 = 16u * gk[k];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        uint32_t c = (pw[k][jj >> 1] >> (16 * (jj & 1))) & 0xFFFFu;
        float v;
        if (XSM) {
          v = xs[c];  // pads read the zero slot xs[cols]
        } else {
          v = __ldg(xs + min(c, G.cols - 1u));
          if (TWO && s0 + jj >= n2 && s0 + jj < G.n2p) v = 0.0f;  // pads (apply_permutation)
        }
        xv[k][jj] = v;
        mx = fmaxf(mx, fabsf(v));
      }
    }
    // one scale per warp (a single-instruction integer max over the lanes: |x|
    // bits order like the values), no CTA barrier: the row sums of a warp's
    // lanes share it and it is undone once per row
    const uint32_t mxb = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
    if (threadIdx.x == 0) stamp(a.dbg, 9);  // gathered
    const int eb = (int)(mxb >> 23);
    const int sh = (eb == 0 ? -126 : eb - 127) - 10;  // floor(log2 max) - 10
    // x' 2^-b as one power-of-two factor, or two when 2^(-sh-b) leaves the
    // normal range (extreme x); warp-uniform
    const bool split = (-sh > 127) || (-sh - (TWO ? 6 : 12) < -126);
    float f1[4], f2[4];
#pragma unroll
    for (int bi = 0; bi < 4; ++bi) {
      const int e = -sh - (TWO ? 2 * bi : 4 * bi);
      const int e1 = max(-126, min(127, e));
      f1[bi] = pow2f(e1), f2[bi] = pow2f(max(-126, min(127, e - e1)));
    }
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint32_t g = gk[k];
      // a dead lane (past its type's last group) decodes a real group with X = 0
      const float live = lv[k] ? 1.0f : 0.0f;
      float sb[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // sum of x' 2^-b per bit position
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int bi = TWO ? (jj & 3) : (jj & 1);
        float xf = xv[k][jj] * (f1[bi] * live);
        if (split) xf *= f2[bi];
        X[k][jj] = __float2half2_rn(xf);
        sb[bi] += xf;
      }
      const float sx = TWO ? (sb[0] + sb[1] * 4.0f) + (sb[2] * 16.0f + sb[3] * 64.0f)
                           : sb[0] + sb[1] * 16.0f;  // sum x' = sum_b 2^b (sum x' 2^-b)
      // zero point: z lands at 2^(2 sub - 24) (2-bit) or 2^-24 (4-bit): z_h nsxh = -z sum x'
      const int zp = TWO ? 2 * (int)(g - 3u * (g / 3u)) : 0;
      nsxh[k] = __float2half2_rn(-sx * pow2f(-zp));
    }
    // every accumulated term is in units of 2^(sh + 24) (and 2^P for 2-bit s1)
    yscale = pow2f(max(-126, min(127, sh + 24))) * (TWO ? 1.0f / s_scale : 1.0f);
    if (share) {
      uint4* d = reinterpret_cast<uint4*>(xsh);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        d[q] = make_uint4(*reinterpret_cast<uint32_t*>(&X[0][4 * q]), *reinterpret_cast<uint32_t*>(&X[0][4 * q + 1]),
                          *reinterpret_cast<uint32_t*>(&X[0][4 * q + 2]), *reinterpret_cast<uint32_t*>(&X[0][4 * q + 3]));
      d[4] = make_uint4(*reinterpret_cast<uint32_t*>(&nsxh[0]), __float_as_uint(yscale), 0u, 0u);
    }
    }
    if (share) {
      named_sync(3, 2 * W * 32);
      if (team == 1) {
        const uint4* d = reinterpret_cast<const uint4*>(xsh);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = d[q];
          X[0][4 * q] = as_h2(v.x), X[0][4 * q + 1] = as_h2(v.y), X[0][4 * q + 2] = as_h2(v.z),
          X[0][4 * q + 3] = as_h2(v.w);
        }
        const uint4 v = d[4];
        nsxh[0] = as_h2(v.x), yscale = __uint_as_float(v.y);
        __syncwarp();  // every lane has read before the window is reused
      }
    }
    if (threadIdx.x == 0) stamp(a.dbg, 2);  // prologue done
    if (threadIdx.x == 0 && a.dbg && nunit) {  // diagnostics: the first unit is in
      mbar_wait(&s_full[0], 0);
      stamp(a.dbg, 3);
    }

    for (uint32_t rep = 0; rep < reps; ++rep) {
      uint32_t slot = team, phase = 0, wrow = 0, ufirst = 0;
      while (slot >= S) slot -= S, phase ^= 1u;
      for (uint32_t u = team; u < nunit; u += T) {
        mbar_wait(&s_full[slot], phase);
        const uint8_t* sb = smem + (size_t)slot * NQ * dense;
        float acc[NQ][4];
#pragma unroll
        for (int j = 0; j < NQ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          // all NQ quads unconditionally (a short last unit decodes stale slot
          // bytes into rows that are never stored): one basic block, so the
          // quads' independent chains interleave
          if (TWO) {
            uint4 w[NQ];
            uint2 m[NQ], s1[NQ];
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              w[j] = *reinterpret_cast<const uint4*>(sb + j * dense + off_c[k]);
              m[j] = *reinterpret_cast<const uint2*>(sb + j * dense + off_p[k]);
            }
            if (u < npre) {
#pragma unroll
              for (int j = 0; j < NQ; ++j) s1[j] = pre_at(slot, j, k);
            } else {
#pragma unroll
              for (int j = 0; j < NQ; ++j) s1[j] = scales_of(sb, j, k, u);
            }
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              // sum((c - z) x') per row in fp16, then y += s1 * that in fp32
              const half2 T01 = __hfma2(as_h2(m[j].x & zmask[k]), nsxh[k], dot2(w[j].x, w[j].y, X[k]));
              const half2 T23 = __hfma2(as_h2(m[j].y & zmask[k]), nsxh[k], dot2(w[j].z, w[j].w, X[k]));
              acc[j][0] = fhfma_lo(T01, as_h2(s1[j].x), acc[j][0]);
              acc[j][1] = fhfma_hi(T01, as_h2(s1[j].x), acc[j][1]);
              acc[j][2] = fhfma_lo(T23, as_h2(s1[j].y), acc[j][2]);
              acc[j][3] = fhfma_hi(T23, as_h2(s1[j].y), acc[j][3]);
            }
          } else {
            uint4 wa[NQ], wb[NQ];
            uint2 s4[NQ];
            uint32_t z4[NQ];
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              const uint8_t* qb = sb + j * dense;
              wa[j] = *reinterpret_cast<const uint4*>(qb + off_c[k]);
              wb[j] = *reinterpret_cast<const uint4*>(qb + off_c[k] + 16u);
              s4[j] = *reinterpret_cast<const uint2*>(qb + off_p[k]);
              z4[j] = *reinterpret_cast<const uint16_t*>(qb + off_z[k]);
            }
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              // ---- 4-bit block: s4 is fp16 already (fourbit, bitpack.hpp:103-110)
              const uint32_t zz = z4[j] | (z4[j] << 12);
              const half2 T01 = __hfma2(as_h2(zz & 0x000F000Fu), nsxh[k], dot4(wa[j], X[k]));
              const half2 T23 = __hfma2(as_h2((zz >> 8) & 0x000F000Fu), nsxh[k], dot4(wb[j], X[k]));
              acc[j][0] = fhfma_lo(T01, as_h2(s4[j].x), acc[j][0]);
              acc[j][1] = fhfma_hi(T01, as_h2(s4[j].x), acc[j][1]);
              acc[j][2] = fhfma_lo(T23, as_h2(s4[j].y), acc[j][2]);
              acc[j][3] = fhfma_hi(T23, as_h2(s4[j].y), acc[j][3]);
            }
          }
        }
        if (nunit > S) {  // ring: hand the slot back once every warp read it
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[slot]);
        }
#pragma unroll
        for (int j = 0; j < NQ; ++j)
          *reinterpret_cast<float4*>(win + win_base(lane) + wrow + 4 * j) =
              make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
        if (wrow == 0) ufirst = u;
        wrow += 4 * NQ;
        if (wrow == kWinRows || u + T >= nunit) {  // window full: row pairs over lanes
          __syncwarp();
          const uint32_t rp = 2u * (lane & 7u);  // rows rp, rp + 1 of the window
          const float* src = win + win_base(lane & 24u) + rp;
          float2 sum = *reinterpret_cast<const float2*>(src);
#pragma unroll
          for (uint32_t l = 1; l < 8; ++l) sum = fadd2(sum, *reinterpret_cast<const float2*>(src + 20u * l));
          sum = fadd2(sum, make_float2(__shfl_xor_sync(0xFFFFFFFFu, sum.x, 8), __shfl_xor_sync(0xFFFFFFFFu, sum.y, 8)));
          sum = fadd2(sum, make_float2(__shfl_xor_sync(0xFFFFFFFFu, sum.x, 16), __shfl_xor_sync(0xFFFFFFFFu, sum.y, 16)));
          // window row rp of unit ufirst + (rp / 4 NQ) T (a team's units are T apart)
          const uint32_t r = (ufirst + (rp / (4 * NQ)) * T) * NQ * kRowsPerQuad + rp % (4 * NQ);
          if (lane < 8 && rp < wrow) {
            if (r < nrows) s_part[r * W + wt] = sum.x * yscale;
            if (r + 1 < nrows) s_part[(r + 1) * W + wt] = sum.y * yscale;
          }
          __syncwarp();
          wrow = 0;
        }
        for (slot += T; slot >= S;) slot -= S, phase ^= 1u;
      }
    }
  };
  if (two)
    run(std::true_type{});
  else
    run(std::false_type{});
  if (threadIdx.x == 0) stamp(a.dbg, 4);  // consumers done
  named_sync(2, (NC + 1) * 32);          // partials and outlier sums complete
  // the dense sum first (fixed warp order), then the outliers, as row_fma (engine.cpp:111-122)
  for (uint32_t t = threadIdx.x; t < nrows; t += NC * 32) {
    const float* p = s_part + t * W;
    float s = p[0];
    for (uint32_t w2 = 1; w2 < W; ++w2) s += p[w2];
    g_y[r_begin + t] = s + s_csr[t];
  }
  if (threadIdx.x == 0) stamp(a.dbg, 5);
}

using GemvFn = void (*)(GemvArgs);

uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* e = std::getenv(name);
  return e ? (uint32_t)std::atoi(e) : dflt;
}
template <bool UNI, bool XSM>
GemvFn pick2(uint32_t kg) {
  switch (kg) {
    case 1:
      if (UNI && env_u32("QW_NQ1", 2) == 2) return gemv_kernel<1, 2, UNI, XSM>;
      return gemv_kernel<1, UNI ? 4 : 1, UNI, XSM>;
    case 2: return gemv_kernel<2, UNI ? 2 : 1, UNI, XSM>;
    case 3: return gemv_kernel<3, 1, UNI, XSM>;
    default: return gemv_kernel<4, 1, UNI, XSM>;
  }
}
GemvFn pick_teams(uint32_t kg) {
  return kg == 1 ? gemv_kernel<1, 2, true, true, true> : gemv_kernel<2, 2, true, true, true>;
}
GemvFn pick_kernel(uint32_t kg, bool uni, bool xsm) {
  return uni ? (xsm ? pick2<true, true>(kg) : pick2<true, false>(kg))
             : (xsm ? pick2<false, true>(kg) : pick2<false, false>(kg));
}
uint32_t quads_per_slot(uint32_t kg, bool uni) {
  return !uni ? 1u : (kg == 1 ? env_u32("QW_NQ1", 2) : (kg == 2 ? 2u : 1u));
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

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

namespace {
// geometry-dependent part of a plan (warps, groups per lane, quads per slot, ...)
int plan_geometry(GemvPlan& p, const Geometry& G) {
  // chunks of 32 groups, kept apart per type so each warp is all 2-bit or all 4-bit
  const uint32_t c2 = (G.G2 + 31u) / 32u, c4 = (G.T4 + 31u) / 32u;
  p.nchunks = c2 + c4;
  // lanes own KG groups of every quad, W warps cover a row: W <= 8 for KG <= 2
  // (two CTAs per SM), else the fewest KG <= 4 with W <= 15
  auto warps_for = [&](uint32_t kg) { return (c2 + kg - 1) / kg + (c4 + kg - 1) / kg; };
  p.kmax = 1;
  while (p.kmax < 4 && warps_for(p.kmax) > (p.kmax <= 2 ? 8u : 15u)) ++p.kmax;
  if (warps_for(p.kmax) > 15) return (int)cudaErrorInvalidConfiguration;
  p.uniform_rb = (G.group2 % kRowsPerQuad) == 0;
  p.xsm = G.cols <= 16384;  // x staged in shared memory (64 KB at most)
  // wide layers (down_proj): KG = 2 over up to 16 warps in one CTA per SM
  // rather than KG >= 3 (register spills) in two
  p.wide = p.kmax > 2 && warps_for(2) <= 16 && p.uniform_rb && p.xsm && env_u32("QW_WIDE", 1);
  if (p.wide) p.kmax = 2;
  p.warps = warps_for(p.kmax);
  p.warps2 = (c2 + p.kmax - 1) / p.kmax;
  p.teams = 1;
  p.uq = quads_per_slot(p.kmax, p.uniform_rb);
  p.rb_one = G.group2 == 1;
  p.rb_magic = p.rb_one ? 0u : (uint32_t)((0x100000000ull + G.group2 - 1) / G.group2);
  return 0;
}

// CTA ranges (one layer each) + shared-memory layout for the largest range
int plan_ctas(GemvPlan& p, const Geometry& G, const uint32_t* const* host_row_ptrs, uint32_t n, int num_sms) {
  uint32_t per_sm = 1;
  if (const char* e = std::getenv("QW_CTAS_PER_SM")) per_sm = std::max(1, std::atoi(e));
  const uint64_t total = (uint64_t)n * G.quads;
  uint32_t grid = (uint32_t)std::min<uint64_t>(std::min<uint32_t>((uint32_t)num_sms * per_sm, kMaxGrid), total);
  grid = std::max(grid, n);
  p.grid = grid;
  p.nq_max = 0;
  uint32_t so_rows_max = 0, cta = 0, ent_max = 0;
  for (uint32_t l = 0; l < n; ++l) {
    const uint32_t g_l = grid * (l + 1) / n - grid * l / n;  // CTAs of layer l
    for (uint32_t b = 0; b < g_l; ++b, ++cta) {
      const uint32_t q0 = (uint32_t)((uint64_t)b * G.quads / g_l), q1 = (uint32_t)((uint64_t)(b + 1) * G.quads / g_l);
      p.cta_seg[cta] = (uint8_t)l;
      p.cta_q0[cta] = q0, p.cta_q1[cta] = q1;
      const uint32_t r0 = q0 * kRowsPerQuad, r1 = std::min(q1 * kRowsPerQuad, G.rows);
      p.cta_e0[cta] = host_row_ptrs[l][std::min(r0, G.rows)];
      p.cta_e1[cta] = host_row_ptrs[l][std::min(r1, G.rows)];
      p.nq_max = std::max(p.nq_max, q1 - q0);
      ent_max = std::max(ent_max, p.cta_e1[cta] - p.cta_e0[cta]);
      if (r1 > r0) so_rows_max = std::max(so_rows_max, (r1 - 1) / G.group2 - r0 / G.group2 + 1);
    }
  }
  const size_t so_bytes = (size_t)so_rows_max * G.G2s * 4;
  const size_t part_bytes = (size_t)p.nq_max * p.warps * 16;  // [row][warp of a team]
  const size_t misc_bytes = (size_t)p.nq_max * 4 * 4 + ((size_t)p.nq_max * 4 + 4) * 4 + 256 * 4 + 64 * 4;
  const size_t x_bytes = p.xsm ? align_up((size_t)G.cols * 4 + 4, 16) : 0;  // + the pads' zero slot
  const uint32_t tmax = (!p.wide && p.kmax <= 2 && p.uniform_rb && p.xsm && p.uq == 2) ? 2u : 1u;
  const size_t win_bytes = (size_t)p.warps * tmax * kWinWords * 4;
  // long ranges (group launches, big layers): two teams, the whole SM
  p.teams = (!p.wide && p.nq_max >= env_u32("QW_TEAMS_MIN_NQ", 4) && p.kmax <= 2 && p.uniform_rb && p.xsm &&
             p.uq == 2) ? 2 : 1;
  // the CTA's outlier entries staged by one bulk copy when they fit and do
  // not cost a ring slot (decided below)
  const size_t ent_bytes = align_up(((size_t)ent_max + 3) * 4, 16);
  size_t stage_bytes = 0;
  const size_t fixed = align_up(so_bytes, 16) + part_bytes + align_up(misc_bytes, 16) + x_bytes +
                       win_bytes + 64 + 8;
  // precomputed 1st-order scales: one uint2 per (slot, quad, k, lane)
  auto pre_bytes = [&](size_t s) { return p.teams == 2 ? (size_t)0 : s * p.uq * p.kmax * p.warps * 32 * 8; };
  // ring: the CTA's whole quad range when it fits in ~half an SM (so the next
  // layer's CTA fits beside it under PDL), else as many slots as fit
  const size_t unit_bytes = (size_t)p.uq * G.dense_bytes;
  const size_t units = (p.nq_max + p.uq - 1) / p.uq;
  const size_t half_sm = (p.teams == 2 || p.wide ? 200 : env_u32("QW_SMEM_KB", 112)) * 1024, full_sm = 220 * 1024;
  auto total_b = [&](size_t s) {
    return align_up(s * unit_bytes, 128) + fixed + stage_bytes + pre_bytes(s) + (2 * s + 2) * 8;
  };
  auto slots = [&]() {
    size_t s = units;
    while (s > 3 && total_b(s) > half_sm) --s;
    while (s > 2 && total_b(s) > full_sm) --s;
    return s;
  };
  size_t S = slots();
  // (x staged in shared memory only: the per-row sums gather x; a CTA that
  // owns its SM trades ring slots for it, a co-resident one must keep its fit)
  p.csr_stage = 0;
  if (p.xsm && ent_max > 0 && ent_bytes <= (size_t)env_u32("QW_CSR_STAGE_KB", 32) * 1024) {
    stage_bytes = ent_bytes + 16;
    const size_t S1 = slots();
    const bool alone = p.teams == 2 || p.wide;
    const bool ok = alone ? (S1 >= 2 && total_b(S1) <= full_sm)
                          : (S1 == S && (total_b(S1) <= half_sm || total_b(S) > half_sm));
    if (ok)
      p.csr_stage = 1, S = S1;
    else
      stage_bytes = 0;
  }
  // two teams share a ring: with an even slot count slot s only ever holds
  // team (s % 2)'s units, so a team's successive units in a slot are
  // successive barrier phases.  (With an odd count a fast team could wait for
  // phase p + 2 of a slot while the other team's phase p + 1 is still in
  // flight, and the parity wait would alias with the completed phase p.)
  if (p.teams == 2 && S < units && (S & 1)) --S;
  if (total_b(S) > full_sm || (p.teams == 2 && S < 2)) return (int)cudaErrorInvalidConfiguration;
  p.nslot = (uint32_t)S;
  p.so_off = (uint32_t)align_up(S * unit_bytes, 128);
  p.part_off = p.so_off + (uint32_t)align_up(so_bytes, 16);
  p.misc_off = p.part_off + (uint32_t)part_bytes;
  p.xg_off = p.misc_off + (uint32_t)align_up(misc_bytes, 16);
  p.win_off = p.xg_off + (uint32_t)x_bytes;
  p.pre_off = p.win_off + (uint32_t)win_bytes;
  p.ent_off = (uint32_t)align_up(p.pre_off + pre_bytes(S), 16);
  p.bar_off = (uint32_t)align_up(p.ent_off + (p.csr_stage ? ent_bytes : 0), 8);
  p.smem = (uint32_t)(p.bar_off + (2 * S + 3) * 8);
  // launch policy (fixed at plan time; the env knobs are diagnostics).  A CTA
  // that owns its SM (teams / wide) starts after its predecessor: no scale
  // precompute (the main loop must run under the weight stream), x first, and
  // the producer holds the stream after 4 units until x is staged.  Otherwise
  // (two CTAs per SM under PDL) the resident units' scales are precomputed
  // while the predecessor still runs.
  if (env_u32("QW_PLAN_DEBUG", 0))
    std::fprintf(stderr,
                 "qw plan: rows %u cols %u kmax %u warps %u teams %u wide %d xsm %u nq_max %u slots %u unit %zu B "
                 "smem %u csr_stage %u (entries %u)\n",
                 G.rows, G.cols, p.kmax, p.warps, p.teams, (int)p.wide, p.xsm, p.nq_max, p.nslot, unit_bytes, p.smem,
                 p.csr_stage, ent_max);
  const bool alone = p.teams == 2 || p.wide;
  p.pre = env_u32("QW_NO_PRE", 0) ? 0u : 1u;
  p.npre_max = env_u32("QW_NPRE_MAX", alone ? 0u : 1000000u);
  p.x_first = env_u32("QW_XFIRST", alone ? 1u : 0u);
  p.x_gate = env_u32("QW_XGATE", alone ? 1u : 1000000u);
  p.pf_late = env_u32("QW_PF_LATE", 1);
  static bool attr_set = false;  // raise the opt-in limit once per process
  if (!attr_set) {
    for (bool uni : {false, true})
      for (bool xsm : {false, true})
        for (uint32_t k : {1u, 2u, 3u, 4u}) {
          cudaError_t err = cudaFuncSetAttribute(pick_kernel(k, uni, xsm),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(227 * 1024));
          if (err != cudaSuccess) return (int)err;
        }
    for (bool xsm : {false, true}) {
      cudaError_t err = cudaFuncSetAttribute(xsm ? gemv_kernel<1, 2, true, true> : gemv_kernel<1, 2, true, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
      if (err != cudaSuccess) return (int)err;
    }
    for (uint32_t k : {1u, 2u}) {
      cudaError_t err = cudaFuncSetAttribute(pick_teams(k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(227 * 1024));
      if (err != cudaSuccess) return (int)err;
    }
    attr_set = true;
  }
  return 0;
}
}  // namespace

int plan_gemv(DeviceLayer& L, int num_sms, const uint32_t* host_row_ptr) {
  GemvPlan& p = L.plan;
  if (int e = plan_geometry(p, L.g)) return e;
  const uint32_t* rp[1] = {host_row_ptr};
  return plan_ctas(p, L.g, rp, 1, num_sms);
}

int plan_gemv_group(GemvPlan& p, const DeviceLayer* const* layers, const uint32_t* const* host_row_ptrs,
                    uint32_t n, int num_sms) {
  if (n == 0 || n > kMaxSeg) return (int)cudaErrorInvalidValue;
  const Geometry& G = layers[0]->g;
  for (uint32_t l = 1; l < n; ++l) {
    const Geometry& H = layers[l]->g;
    if (H.rows != G.rows || H.cols != G.cols || H.n4 != G.n4 || H.n2p != G.n2p || H.group2 != G.group2 ||
        H.dense_bytes != G.dense_bytes)
      return (int)cudaErrorInvalidValue;
  }
  p = layers[0]->plan;  // geometry part is identical
  return plan_ctas(p, G, host_row_ptrs, n, num_sms);
}

int launch_gemv_group(const GemvPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* x,
                      float* const* ys, void* stream, bool pdl, uint32_t flags, unsigned long long* dbg,
                      uint32_t repeat, bool global_clock) {
  const Geometry& G = layers[0]->g;
  GemvArgs a;
  for (uint32_t l = 0; l < kMaxSeg; ++l) {
    const DeviceLayer& L = *layers[std::min(l, n - 1)];
    a.quads[l] = L.quads, a.sorder[l] = L.sorder, a.row_ptr[l] = L.row_ptr;
    a.csr[l] = L.csr, a.perm[l] = L.perm16, a.s_scale[l] = L.plan.s_scale;
    a.y[l] = ys[std::min(l, n - 1)];
  }
  a.x = x;
  a.g = G;
  a.W = p.warps, a.W2 = p.warps2, a.T = p.teams, a.S = p.nslot;
  a.grid = p.grid, a.nq_max = p.nq_max, a.rb_magic = p.rb_magic, a.rb_one = p.rb_one;
  a.so_off = p.so_off, a.part_off = p.part_off, a.csr_off = p.misc_off, a.x_off = p.xg_off, a.win_off = p.win_off, a.pre_off = p.pre_off;
  a.bar_off = p.bar_off;
  a.ent_off = p.ent_off, a.csr_stage = p.csr_stage;
  a.pf_n = p.pf_n;
  a.pf_late = p.pf_late;
  for (uint32_t r = 0; r < GemvPlan::kMaxPf; ++r) a.pf_ptr[r] = p.pf_ptr[r], a.pf_bytes[r] = p.pf_bytes[r];
  a.dbg = dbg;
  a.dbg_global = global_clock;
  a.wait_x = (flags & kXIndependent) ? 0u : 1u;
  a.pre = p.pre, a.npre_max = p.npre_max, a.x_first = p.x_first, a.x_gate = p.x_gate;
  a.repeat = repeat;
  std::copy(p.cta_seg, p.cta_seg + p.grid, a.cta_seg);
  std::copy(p.cta_q0, p.cta_q0 + p.grid, a.cta_q0);
  std::copy(p.cta_q1, p.cta_q1 + p.grid, a.cta_q1);
  std::copy(p.cta_e0, p.cta_e0 + p.grid, a.cta_e0);
  std::copy(p.cta_e1, p.cta_e1 + p.grid, a.cta_e1);
  const GemvFn fn = (p.teams == 2 || p.wide) ? pick_teams(p.kmax) : pick_kernel(p.kmax, p.uniform_rb, p.xsm);
  const uint32_t threads = (p.warps * p.teams + 2) * 32;
  void* params[] = {&a};
  return (int)launch_ex((const void*)fn, dim3(p.grid), dim3(threads), p.smem, (cudaStream_t)stream, pdl, params);
}

int launch_gemv_group(const GemvPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* x,
                      float* const* ys, void* stream, bool pdl, uint32_t flags) {
  return launch_gemv_group(p, layers, n, x, ys, stream, pdl, flags, nullptr, 1, false);
}

int launch_gemv(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream,
                bool pdl, unsigned long long* dbg, uint32_t repeat, bool global_clock,
                uint32_t flags) {
  const DeviceLayer* layers[1] = {&L};
  for (uint32_t col = 0; col < batch; ++col) {
    float* ys[1] = {y + (size_t)col * L.g.rows};
    const int e = launch_gemv_group(L.plan, layers, 1, x + (size_t)col * L.g.cols, ys, stream, pdl, flags,
                                    dbg, repeat, global_clock);
    if (e) return e;
  }
  return 0;
}


// ============================================================ decode chain
// One persistent kernel runs a whole sequence of batch-1 launch steps (a
// decode step: q/k/v, o, gate/up, down per decoder layer).  One CTA per SM,
// 16 consumer warps + producer + CSR warp.  The producer streams every
// step's quad records through ONE ring that spans the steps, so the weights
// of step s+1 land in shared memory while step s computes -- HBM never waits
// for a kernel boundary or for a CTA slot.  A step whose activation is its
// predecessor's output waits on a grid-wide completion counter (released by
// each CTA after its y stores), then stages x, exactly the dependency a
// kernel boundary would impose.  Per step the 16 consumer warps form T teams
// of W warps (KG = 1, NQ = 2: 4096-wide; KG = 2, NQ = 1: wide layers); the
// per-quad arithmetic is the K2 kernel's (dot2/dot4, s1 from the 2-order
// rows, FHFMA, window reduction), so the results equal the K2 launches'.
namespace {
constexpr uint32_t kChainCons = 16, kChainThreads = (kChainCons + 2) * 32;
constexpr uint32_t kChainEmpty = kChainCons;  // every consumer warp hands every unit back
// team 0 hands its prepared X to team 1 (saves the duplicate prologue); off:
// with both KG bodies in one kernel ptxas spills heavily at the 96-register cap
constexpr bool kChainShareX = false;

struct ChainStep {
  const uint8_t* quads[kMaxSeg];
  const uint32_t* sorder[kMaxSeg];
  const uint32_t* row_ptr[kMaxSeg];
  const uint32_t* csr[kMaxSeg];
  const uint16_t* perm[kMaxSeg];
  float* y[kMaxSeg];
  float s_scale[kMaxSeg];
  const float* x;
  Geometry g;
  uint32_t W, W2, T, KG, NQ, rb_magic, rb_one, depends;
};
struct ChainCta {
  uint32_t seg, q0, q1, e0, e1;
};
struct ChainArgs {
  const ChainStep* steps;
  const ChainCta* ctas;  // [step][grid]
  unsigned* done;        // [step] CTAs that stored their y of the step
  uint32_t nsteps, grid, S, slot_bytes, so_stride, nq_max;
  uint32_t so_off, part_off, misc_off, x_off, win_off, bar_off;
};
// per-step consumer context
struct ChainCtx {
  const uint8_t* ring;
  const uint32_t* s_so;
  float* s_part;
  const float* s_x;
  float* win;
  float* win_all;
  uint64_t* full;
  uint64_t* empty;
  const uint16_t* perm;
  float s_scale;
  uint32_t gu, nunit, nrows, q0, rb_first, team, wt, S, slot_bytes;
};


__device__ __forceinline__ uint32_t ld_acquire_gpu(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Chain diagnostics: with a watch buffer, a wait that spins for ~seconds
// records (code, step, unit/parity, CTA, warp) and traps instead of hanging.
__device__ unsigned* g_chain_watch = nullptr;
__device__ __forceinline__ void chain_wait(uint64_t* bar, uint32_t parity, uint32_t code, uint32_t arg) {
  if (!g_chain_watch) {
    mbar_wait(bar, parity);
    return;
  }
  for (uint32_t i = 0; !mbar_try_wait(bar, parity); ++i) {
    if (i == (1u << 22)) {
      unsigned* w = g_chain_watch + 8 * (blockIdx.x * 32 + (threadIdx.x >> 5));
      w[0] = 1u + code, w[1] = arg, w[2] = parity, w[3] = blockIdx.x, w[4] = threadIdx.x;
      __threadfence_system();
      __trap();
    }
  }
}

template <int KG, int NQ>
__device__ __forceinline__ void chain_consume(const ChainStep& st, const ChainCtx& c) {
  const Geometry G = st.g;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t W = st.W, W2 = st.W2, W4 = W - W2, T = st.T, team = c.team, wt = c.wt;
  const uint32_t dense = G.dense_bytes, nunit = c.nunit;
  // ring position of the step's first unit.  EVERY consumer warp waits for
  // and hands back EVERY unit (the owning team after decoding it): a slot is
  // refilled only when all 16 warps are done with it, so no warp can fall two
  // phases behind a slot and misread a parity.
  uint32_t slot = c.gu % c.S, phase = (c.gu / c.S) & 1u;
  auto pass = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&c.empty[slot]);
    if (++slot == c.S) slot = 0, phase ^= 1u;
  };
  if (team >= T) {  // idle warp this step (W does not divide 16)
    for (uint32_t u = 0; u < nunit; ++u) {
      chain_wait(&c.full[slot], phase, 1, c.gu + u);
      pass();
    }
    return;
  }
  const uint32_t rb_magic = st.rb_magic, rb_one = st.rb_one;
  auto row_block = [&](uint32_t r) { return rb_one ? r : __umulhi(r, rb_magic); };
  const bool two = wt < W2;
  uint32_t gk[KG];
  bool lv[KG];
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    if (two) {
      const uint32_t g = (wt + (uint32_t)k * W2) * 32u + lane;
      lv[k] = g < G.G2;
      gk[k] = lv[k] ? g : G.G2 - 1u;
    } else {
      const uint32_t b = (wt - W2 + (uint32_t)k * W4) * 32u + lane;
      lv[k] = b < G.T4;
      gk[k] = G.G2 + (lv[k] ? b : G.T4 - 1u);
    }
  }
  float* win = c.win;

  auto run = [&](auto two_tag) {
    constexpr bool TWO = decltype(two_tag)::value;
    uint32_t off_c[KG], off_p[KG], off_z[KG], zmask[KG], esh[KG], emask[KG];
    int pe[KG];
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint32_t g = gk[k];
      if (TWO) {
        const uint32_t t = g / 3u, sub = g - 3u * t;
        off_c[k] = 16u * g;
        off_p[k] = G.off_meta + 8u * t;
        off_z[k] = 0;
        zmask[k] = 0x00030003u << (2u * sub);
        esh[k] = sub == 0 ? 0u : 7u;  // 4/3/3 rule (quantizer.cpp:103-104)
        emask[k] = sub == 0 ? 0x03C003C0u : (sub == 1 ? 0x00380038u : 0x01C001C0u);
        pe[k] = sub == 0 ? 6 : (sub == 1 ? 2 : 5);
      } else {
        const uint32_t b = g - G.G2;
        off_c[k] = G.off_c4 + 32u * b;
        off_p[k] = G.off_s4 + 8u * b;
        off_z[k] = G.off_z4 + 2u * b;
        zmask[k] = esh[k] = emask[k] = 0;
        pe[k] = 0;
      }
    }
    // the 2-order dequant of the lane's groups (engine.cpp:48-63), as in K2
    // one 2-order row block at a time: the team visits its rows in increasing
    // order (quads j of a unit, then the next unit), so one set is live
    half2 A2[KG], C2[KG], P2[KG];
#pragma unroll
    for (int k = 0; k < KG; ++k) P2[k] = __float2half2_rn(pow2f(-pe[k]));
    uint32_t rb_end = 0;
    auto scales_of = [&](const uint8_t* sb, int j, int k, uint32_t u) -> uint2 {
      const uint32_t r0 = (c.q0 + u * NQ + j) * kRowsPerQuad;
      if (r0 >= rb_end) {
#pragma unroll
        for (int kk = 0; kk < KG; ++kk) {
          const uint32_t rb = row_block(min(r0, G.rows - 1)) - c.rb_first;
          const uint32_t e = c.s_so[rb * G.G2s + gk[kk]];
          A2[kk] = __float2half2_rn(half_bits_to_float(e) * c.s_scale);
          C2[kk] = __float2half2_rn(-(pow2f(10 - pe[kk]) + small_int_to_float(e >> 16)));
        }
        rb_end = (row_block(r0) + 1) * G.group2;
      }
      const uint2 m = *reinterpret_cast<const uint2*>(sb + j * dense + off_p[k]);
      return make_uint2(s1_pair(m.x >> esh[k], emask[k], P2[k], C2[k], A2[k]),
                        s1_pair(m.y >> esh[k], emask[k], P2[k], C2[k], A2[k]));
    };

    // ---- activation prologue (as K2): permuted gather, per-warp power of two.
    // Two teams of one geometry need the same X: team 0 prepares it and hands
    // it to team 1 through team 1's (not yet used) reduction windows.
    half2 X[KG][16], nsxh[KG];
    float yscale;
    const bool share = KG == 1 && T == 2 && kChainShareX;
    uint32_t* xsh = reinterpret_cast<uint32_t*>(c.win_all + (W + wt) * kWinWords) + lane * 20u;
    if (!share || team == 0) {
    uint32_t pw[KG][8];
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint4* pp = reinterpret_cast<const uint4*>(c.perm + 16u * gk[k]);
      const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
      pw[k][0] = p0.x, pw[k][1] = p0.y, pw[k][2] = p0.z, pw[k][3] = p0.w;
      pw[k][4] = p1.x, pw[k][5] = p1.y, pw[k][6] = p1.z, pw[k][7] = p1.w;
    }
    float xv[KG][16];
    float mx = 0.0f;
#pragma unroll
    for (int k = 0; k < KG; ++k) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const float v = c.s_x[(pw[k][jj >> 1] >> (16 * (jj & 1))) & 0xFFFFu];  // pads: zero slot
        xv[k][jj] = v;
        mx = fmaxf(mx, fabsf(v));
      }
    }
    const uint32_t mxb = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
    const int eb = (int)(mxb >> 23);
    const int sh = (eb == 0 ? -126 : eb - 127) - 10;
    const bool split = (-sh > 127) || (-sh - (TWO ? 6 : 12) < -126);
    float f1[4], f2[4];
#pragma unroll
    for (int bi = 0; bi < 4; ++bi) {
      const int e = -sh - (TWO ? 2 * bi : 4 * bi);
      const int e1 = max(-126, min(127, e));
      f1[bi] = pow2f(e1), f2[bi] = pow2f(max(-126, min(127, e - e1)));
    }
    auto prep = [&](auto split_tag) {
      constexpr bool SPLIT = decltype(split_tag)::value;
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const uint32_t g = gk[k];
      const float live = lv[k] ? 1.0f : 0.0f;
      float sb[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int bi = TWO ? (jj & 3) : (jj & 1);
        float xf = xv[k][jj] * (f1[bi] * live);
        if (SPLIT) xf *= f2[bi];
        X[k][jj] = __float2half2_rn(xf);
        sb[bi] += xf;
      }
      const float sx = TWO ? (sb[0] + sb[1] * 4.0f) + (sb[2] * 16.0f + sb[3] * 64.0f) : sb[0] + sb[1] * 16.0f;
      const int zp = TWO ? 2 * (int)(g - 3u * (g / 3u)) : 0;
      nsxh[k] = __float2half2_rn(-sx * pow2f(-zp));
    }
    };
    if (split)
      prep(std::true_type{});
    else
      prep(std::false_type{});
    yscale = pow2f(max(-126, min(127, sh + 24))) * (TWO ? 1.0f / c.s_scale : 1.0f);
    if (share) {
      uint4* d = reinterpret_cast<uint4*>(xsh);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        d[q] = make_uint4(*reinterpret_cast<uint32_t*>(&X[0][4 * q]), *reinterpret_cast<uint32_t*>(&X[0][4 * q + 1]),
                          *reinterpret_cast<uint32_t*>(&X[0][4 * q + 2]), *reinterpret_cast<uint32_t*>(&X[0][4 * q + 3]));
      d[4] = make_uint4(*reinterpret_cast<uint32_t*>(&nsxh[0]), __float_as_uint(yscale), 0u, 0u);
    }
    }
    if (share) {
      named_sync(3, 2 * W * 32);
      if (team == 1) {
        const uint4* d = reinterpret_cast<const uint4*>(xsh);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = d[q];
          X[0][4 * q] = as_h2(v.x), X[0][4 * q + 1] = as_h2(v.y), X[0][4 * q + 2] = as_h2(v.z), X[0][4 * q + 3] = as_h2(v.w);
        }
        const uint4 v = d[4];
        nsxh[0] = as_h2(v.x), yscale = __uint_as_float(v.y);
        __syncwarp();  // every lane has read before the window is reused
      }
    }

    uint32_t wrow = 0, ufirst = 0, owner = 0;
    for (uint32_t u = 0; u < nunit; ++u, owner = owner + 1 == T ? 0 : owner + 1) {
      // every unit's phase is observed in order (a parity wait that skipped a
      // phase could alias with an older completed one); only the team's own
      // units (u = team mod T) are decoded
      if (g_chain_watch && lane == 0) {  // diagnostics: progress (unit being waited for)
        volatile unsigned* w = g_chain_watch + 8 * (blockIdx.x * 32 + (threadIdx.x >> 5));
        w[5] = c.gu + u + 1, w[6] = slot, w[7] = phase;
      }
      chain_wait(&c.full[slot], phase, 1, c.gu + u);
      if (owner != team) {
        pass();
        continue;
      }
      const uint8_t* sb = c.ring + (size_t)slot * c.slot_bytes;
      float acc[NQ][4];
#pragma unroll
      for (int j = 0; j < NQ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        if (TWO) {
          uint4 w[NQ];
          uint2 m[NQ], s1[NQ];
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            w[j] = *reinterpret_cast<const uint4*>(sb + j * dense + off_c[k]);
            m[j] = *reinterpret_cast<const uint2*>(sb + j * dense + off_p[k]);
          }
#pragma unroll
          for (int j = 0; j < NQ; ++j) s1[j] = scales_of(sb, j, k, u);
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            const half2 T01 = __hfma2(as_h2(m[j].x & zmask[k]), nsxh[k], dot2(w[j].x, w[j].y, X[k]));
            const half2 T23 = __hfma2(as_h2(m[j].y & zmask[k]), nsxh[k], dot2(w[j].z, w[j].w, X[k]));
            acc[j][0] = fhfma_lo(T01, as_h2(s1[j].x), acc[j][0]);
            acc[j][1] = fhfma_hi(T01, as_h2(s1[j].x), acc[j][1]);
            acc[j][2] = fhfma_lo(T23, as_h2(s1[j].y), acc[j][2]);
            acc[j][3] = fhfma_hi(T23, as_h2(s1[j].y), acc[j][3]);
          }
        } else {
          uint4 wa[NQ], wb[NQ];
          uint2 s4[NQ];
          uint32_t z4[NQ];
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            const uint8_t* qb = sb + j * dense;
            wa[j] = *reinterpret_cast<const uint4*>(qb + off_c[k]);
            wb[j] = *reinterpret_cast<const uint4*>(qb + off_c[k] + 16u);
            s4[j] = *reinterpret_cast<const uint2*>(qb + off_p[k]);
            z4[j] = *reinterpret_cast<const uint16_t*>(qb + off_z[k]);
          }
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            const uint32_t zz = z4[j] | (z4[j] << 12);
            const half2 T01 = __hfma2(as_h2(zz & 0x000F000Fu), nsxh[k], dot4(wa[j], X[k]));
            const half2 T23 = __hfma2(as_h2((zz >> 8) & 0x000F000Fu), nsxh[k], dot4(wb[j], X[k]));
            acc[j][0] = fhfma_lo(T01, as_h2(s4[j].x), acc[j][0]);
            acc[j][1] = fhfma_hi(T01, as_h2(s4[j].x), acc[j][1]);
            acc[j][2] = fhfma_lo(T23, as_h2(s4[j].y), acc[j][2]);
            acc[j][3] = fhfma_hi(T23, as_h2(s4[j].y), acc[j][3]);
          }
        }
      }
      pass();
#pragma unroll
      for (int j = 0; j < NQ; ++j)
        *reinterpret_cast<float4*>(win + win_base(lane) + wrow + 4 * j) =
            make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
      if (wrow == 0) ufirst = u;
      wrow += 4 * NQ;
      if (wrow == kWinRows || u + T >= nunit) {  // window full or the team's last unit
        __syncwarp();
        const uint32_t rp = 2u * (lane & 7u);
        const float* src = win + win_base(lane & 24u) + rp;
        float2 sum = *reinterpret_cast<const float2*>(src);
#pragma unroll
        for (uint32_t l = 1; l < 8; ++l) sum = fadd2(sum, *reinterpret_cast<const float2*>(src + 20u * l));
        sum = fadd2(sum, make_float2(__shfl_xor_sync(0xFFFFFFFFu, sum.x, 8), __shfl_xor_sync(0xFFFFFFFFu, sum.y, 8)));
        sum = fadd2(sum, make_float2(__shfl_xor_sync(0xFFFFFFFFu, sum.x, 16), __shfl_xor_sync(0xFFFFFFFFu, sum.y, 16)));
        const uint32_t r = (ufirst + (rp / (4 * NQ)) * T) * NQ * kRowsPerQuad + rp % (4 * NQ);
        if (lane < 8 && rp < wrow) {
          if (r < c.nrows) c.s_part[r * W + wt] = sum.x * yscale;
          if (r + 1 < c.nrows) c.s_part[(r + 1) * W + wt] = sum.y * yscale;
        }
        __syncwarp();
        wrow = 0;
      }
    }
  };
  if (two)
    run(std::true_type{});
  else
    run(std::false_type{});
}

__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(const __grid_constant__ ChainArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint8_t* ring = smem;
  uint32_t* s_so = reinterpret_cast<uint32_t*>(smem + a.so_off);  // 2 buffers (steps alternate)
  float* s_part = reinterpret_cast<float*>(smem + a.part_off);
  float* s_csr = reinterpret_cast<float*>(smem + a.misc_off);
  uint32_t* s_rp = reinterpret_cast<uint32_t*>(s_csr + a.nq_max * 4);
  float* s_prod = reinterpret_cast<float*>(s_rp + a.nq_max * 4 + 4);
  float* s_x = reinterpret_cast<float*>(smem + a.x_off);
  float* s_win = reinterpret_cast<float*>(smem + a.win_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* empty = full + a.S;
  uint64_t* so_full = empty + a.S;
  uint64_t* so_empty = so_full + 2;
  uint64_t* xbar = so_empty + 2;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, b = blockIdx.x;

  if (threadIdx.x < a.S) {
    mbar_init(&full[threadIdx.x], 1);
    mbar_init(&empty[threadIdx.x], kChainEmpty);
  }
  if (threadIdx.x == 32) {
    mbar_init(&so_full[0], 1), mbar_init(&so_full[1], 1);
    mbar_init(&so_empty[0], kChainCons), mbar_init(&so_empty[1], kChainCons);
    mbar_init(xbar, 1);
  }
  mbar_fence_init();
  __syncthreads();

  if (warp == kChainCons) {
    // ================= producer: every step's 2-order rows and quad records,
    // one ring across the steps (never waits for x or for a dependency)
    if (lane == 0) {
      uint32_t slot = 0, phase = 0, gu = 0;
      for (uint32_t s = 0; s < a.nsteps; ++s) {
        const ChainStep& st = a.steps[s];
        const ChainCta cc = a.ctas[s * a.grid + b];
        const Geometry& G = st.g;
        auto row_block = [&](uint32_t r) { return st.rb_one ? r : __umulhi(r, st.rb_magic); };
        const uint32_t nq = cc.q1 - cc.q0, NQ = st.NQ, dense = G.dense_bytes;
        const uint32_t r_begin = cc.q0 * kRowsPerQuad, r_end = min(cc.q1 * kRowsPerQuad, G.rows);
        const uint32_t sb = s & 1u;
        if (s >= 2) chain_wait(&so_empty[sb], ((s >> 1) - 1u) & 1u, 2, s);  // step s-2 done with the buffer
        const uint32_t so_bytes =
            r_end > r_begin ? (row_block(r_end - 1) - row_block(r_begin) + 1) * G.G2s * 4u : 0u;
        if (so_bytes) {
          mbar_expect_tx(&so_full[sb], so_bytes);
          bulk_load_nohint(reinterpret_cast<uint8_t*>(s_so) + sb * a.so_stride,
                           st.sorder[cc.seg] + (size_t)row_block(r_begin) * G.G2s, so_bytes, &so_full[sb]);
        } else {
          mbar_arrive(&so_full[sb]);
        }
        const uint8_t* src = st.quads[cc.seg] + (size_t)cc.q0 * dense;
        const uint32_t nunit = (nq + NQ - 1) / NQ;
        for (uint32_t u = 0; u < nunit; ++u, ++gu) {
          const uint32_t bytes = min(NQ, nq - NQ * u) * dense;
          if (g_chain_watch) {
            volatile unsigned* w = g_chain_watch + 8 * (blockIdx.x * 32 + 16);
            w[5] = gu + 1, w[6] = slot, w[7] = phase;
          }
          if (gu >= a.S) chain_wait(&empty[slot], phase ^ 1u, 3, gu);
          mbar_expect_tx(&full[slot], bytes);
          bulk_load_nohint(smem + (size_t)slot * a.slot_bytes, src, bytes, &full[slot]);
          src += bytes;
          if (++slot == a.S) slot = 0, phase ^= 1u;
        }
      }
    }
    return;
  }

  if (warp == kChainCons + 1) {
    // ================= outliers of every step: exact fp32 x, CSR order
    for (uint32_t s = 0; s < a.nsteps; ++s) {
      const ChainStep& st = a.steps[s];
      const ChainCta cc = a.ctas[s * a.grid + b];
      const uint32_t r_begin = cc.q0 * kRowsPerQuad, r_end = min(cc.q1 * kRowsPerQuad, st.g.rows);
      const uint32_t nrows = r_end > r_begin ? r_end - r_begin : 0u;
      const uint32_t* g_row_ptr = st.row_ptr[cc.seg];
      const uint32_t* g_csr = st.csr[cc.seg];
      const uint16_t* g_perm = st.perm[cc.seg];
      const uint32_t e_lo = cc.e0, n = cc.e1 - cc.e0;
      for (uint32_t t = lane; t <= nrows; t += 32) s_rp[t] = g_row_ptr[r_begin + t] - e_lo;
      for (uint32_t t = lane; t < nrows; t += 32) s_csr[t] = 0.0f;
      constexpr int kPer = 8;
      uint32_t ent[kPer], src[kPer];
      auto fetch = [&](uint32_t c0) {
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const uint32_t e = c0 + lane + 32u * j;
          ent[j] = e < n ? __ldg(g_csr + e_lo + e) : 0u;
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) src[j] = ent[j] & 0xFFFFu;  // original channel (repack)
      };
      if (n) fetch(0);
      __syncwarp();
      chain_wait(xbar, s & 1u, 4, s);  // x of step s staged
      uint32_t t0 = 0;
      for (uint32_t c0 = 0; c0 < n; c0 += 32u * kPer) {
        const uint32_t c1 = min(c0 + 32u * kPer, n);
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const uint32_t e = c0 + lane + 32u * j;
          if (e < c1) s_prod[e - c0] = half_bits_to_float(ent[j] >> 16) * s_x[src[j]];
        }
        __syncwarp();
        if (c1 < n) fetch(c1);
        for (;;) {  // rows the chunk touches: [t0, ...)
          const uint32_t t = t0 + lane;
          const uint32_t done = __ballot_sync(0xFFFFFFFFu, t < nrows && s_rp[t + 1] <= c0);
          t0 += __popc(done);
          if (done != 0xFFFFFFFFu) break;
        }
        for (uint32_t t = t0 + lane; t < nrows && s_rp[t] < c1; t += 32) {
          const uint32_t lo = max(s_rp[t], c0), hi = min(s_rp[t + 1], c1);
          float acc = s_csr[t];
          for (uint32_t e = lo; e < hi; ++e) acc += s_prod[e - c0];
          s_csr[t] = acc;
        }
        __syncwarp();
      }
      named_sync(2, (kChainCons + 1) * 32);  // outlier sums ready
      named_sync(2, (kChainCons + 1) * 32);  // the step's y stored
    }
    return;
  }

  // ================= consumers
  uint32_t gu = 0;  // units of the previous steps (ring position)
  for (uint32_t s = 0; s < a.nsteps; ++s) {
    const ChainStep& st = a.steps[s];
    const ChainCta cc = a.ctas[s * a.grid + b];
    const uint32_t rows = st.g.rows, cols = st.g.cols, NQ = st.NQ, W = st.W;
    const uint32_t nq = cc.q1 - cc.q0, nunit = (nq + NQ - 1) / NQ;
    const uint32_t r_begin = cc.q0 * kRowsPerQuad, r_end = min(cc.q1 * kRowsPerQuad, rows);
    const uint32_t nrows = r_end > r_begin ? r_end - r_begin : 0u;
    // dependency: every CTA stored its y of step s-1 (the activation of step s)
    if (st.depends && s > 0) {
      if (threadIdx.x == 0)
        while (ld_acquire_gpu(&a.done[s - 1]) < a.grid) __nanosleep(32);
      named_sync(1, kChainCons * 32);
    }
    // stage x (L2 reads: it may have been written by this kernel)
    {
      const uint32_t nth = kChainCons * 32;
      if ((((uintptr_t)st.x) & 15u) == 0 && (cols & 3u) == 0) {
        const float4* gx = reinterpret_cast<const float4*>(st.x);
        float4* sx4 = reinterpret_cast<float4*>(s_x);
        for (uint32_t i = threadIdx.x; i < (cols >> 2); i += nth) sx4[i] = __ldcg(gx + i);
      } else {
        for (uint32_t i = threadIdx.x; i < cols; i += nth) s_x[i] = __ldcg(st.x + i);
      }
      if (threadIdx.x == 0) s_x[cols] = 0.0f;  // the pads' zero slot
      named_sync(1, kChainCons * 32);
      if (threadIdx.x == 0) mbar_arrive(xbar);
    }
    chain_wait(&so_full[s & 1u], (s >> 1) & 1u, 5, s);
    ChainCtx c;
    c.ring = ring;
    c.s_so = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(s_so) + (s & 1u) * a.so_stride);
    c.s_part = s_part;
    c.s_x = s_x;
    c.full = full, c.empty = empty;
    c.perm = st.perm[cc.seg];
    c.s_scale = st.s_scale[cc.seg];
    c.gu = gu;
    c.nunit = nunit, c.nrows = nrows, c.q0 = cc.q0;
    c.rb_first = st.rb_one ? r_begin : __umulhi(r_begin, st.rb_magic);
    c.team = warp / W, c.wt = warp - c.team * W;
    c.S = a.S, c.slot_bytes = a.slot_bytes;
    c.win = s_win + warp * kWinWords;
    c.win_all = s_win;
    if (st.KG == 1)
      chain_consume<1, 2>(st, c);
    else
      chain_consume<2, 1>(st, c);
    __syncwarp();
    if (lane == 0) mbar_arrive(&so_empty[s & 1u]);
    named_sync(2, (kChainCons + 1) * 32);  // partials and outlier sums complete
    float* g_y = st.y[cc.seg];
    for (uint32_t t = threadIdx.x; t < nrows; t += kChainCons * 32) {
      const float* p = s_part + t * W;
      float acc = p[0];
      for (uint32_t w2 = 1; w2 < W; ++w2) acc += p[w2];
      g_y[r_begin + t] = acc + s_csr[t];
    }
    __threadfence();
    named_sync(2, (kChainCons + 1) * 32);
    if (threadIdx.x == 0) red_release_gpu(&a.done[s], 1u);
    gu += nunit;
  }
}
}  // namespace

unsigned*& chain_watch_host() {
  static unsigned* p = nullptr;
  return p;
}
const unsigned* chain_watch() { return chain_watch_host(); }

struct ChainPlan {
  ChainArgs args{};
  void* dmem = nullptr;
  uint32_t smem = 0, grid = 0, nsteps = 0;
};

int plan_chain(ChainPlan** out, const ChainStepDesc* steps, uint32_t n, int num_sms) {
  if (!out || !steps || n == 0) return (int)cudaErrorInvalidValue;
  const uint32_t grid = (uint32_t)num_sms;
  std::vector<ChainStep> hs(n);
  std::vector<ChainCta> hc((size_t)n * grid);
  uint32_t nq_max = 0, max_cols = 0;
  size_t so_stride = 16, part_max = 16, slot_bytes = 0;
  for (uint32_t s = 0; s < n; ++s) {
    const ChainStepDesc& d = steps[s];
    if (d.n == 0 || d.n > kMaxSeg || !d.layers || !d.ys || !d.x) return (int)cudaErrorInvalidValue;
    const Geometry& G = d.layers[0]->g;
    for (uint32_t l = 1; l < d.n; ++l) {
      const Geometry& H = d.layers[l]->g;
      if (H.rows != G.rows || H.cols != G.cols || H.n4 != G.n4 || H.n2p != G.n2p || H.group2 != G.group2 ||
          H.dense_bytes != G.dense_bytes)
        return (int)cudaErrorInvalidValue;
    }
    GemvPlan gp;
    if (plan_geometry(gp, G)) return (int)cudaErrorNotSupported;
    if (!gp.uniform_rb || !gp.xsm || gp.kmax > 2 || gp.warps > kChainCons) return (int)cudaErrorNotSupported;
    ChainStep& st = hs[s];
    for (uint32_t l = 0; l < kMaxSeg; ++l) {
      const DeviceLayer& L = *d.layers[std::min(l, d.n - 1)];
      st.quads[l] = L.quads, st.sorder[l] = L.sorder, st.row_ptr[l] = L.row_ptr;
      st.csr[l] = L.csr, st.perm[l] = L.perm16, st.s_scale[l] = L.plan.s_scale;
      st.y[l] = d.ys[std::min(l, d.n - 1)];
    }
    st.x = d.x;
    st.g = G;
    st.KG = gp.kmax;
    st.NQ = gp.kmax == 1 ? 2u : 1u;
    st.W = gp.warps, st.W2 = gp.warps2, st.T = kChainCons / gp.warps;
    st.rb_magic = gp.rb_magic, st.rb_one = gp.rb_one;
    st.depends = d.depends;
    max_cols = std::max(max_cols, G.cols);
    slot_bytes = std::max(slot_bytes, (size_t)st.NQ * G.dense_bytes);
    // CTA ranges: the grid split evenly over the step's layers, quads evenly
    for (uint32_t l = 0, cta = 0; l < d.n; ++l) {
      const uint32_t g_l = grid * (l + 1) / d.n - grid * l / d.n;
      for (uint32_t bb = 0; bb < g_l; ++bb, ++cta) {
        ChainCta& cc = hc[(size_t)s * grid + cta];
        cc.seg = l;
        cc.q0 = (uint32_t)((uint64_t)bb * G.quads / g_l), cc.q1 = (uint32_t)((uint64_t)(bb + 1) * G.quads / g_l);
        const uint32_t r0 = std::min(cc.q0 * kRowsPerQuad, G.rows), r1 = std::min(cc.q1 * kRowsPerQuad, G.rows);
        cc.e0 = d.host_row_ptrs[l][r0], cc.e1 = d.host_row_ptrs[l][r1];
        nq_max = std::max(nq_max, cc.q1 - cc.q0);
        part_max = std::max(part_max, (size_t)(cc.q1 - cc.q0) * kRowsPerQuad * st.W * 4);
        if (r1 > r0) {
          const size_t rows_so = (r1 - 1) / G.group2 - r0 / G.group2 + 1;
          so_stride = std::max(so_stride, align_up(rows_so * G.G2s * 4, 16));
        }
      }
    }
  }
  slot_bytes = align_up(slot_bytes, 128);
  ChainPlan* p = new ChainPlan;
  ChainArgs& a = p->args;
  a.nsteps = n, a.grid = grid, a.nq_max = nq_max;
  a.so_stride = (uint32_t)so_stride;
  const size_t misc = (size_t)nq_max * 4 * 4 + ((size_t)nq_max * 4 + 4) * 4 + 256 * 4;
  const size_t fixed = 2 * so_stride + align_up(part_max, 16) + align_up(misc, 16) +
                       align_up(((size_t)max_cols + 1) * 4, 16) + (size_t)kChainCons * kWinWords * 4;
  const size_t budget = 227 * 1024;
  size_t S = 2;
  while ((S + 1) * slot_bytes + fixed + (2 * (S + 1) + 5) * 8 + 128 <= budget) ++S;
  if (S * slot_bytes + fixed + (2 * S + 5) * 8 + 128 > budget) {
    delete p;
    return (int)cudaErrorNotSupported;
  }
  a.S = (uint32_t)S, a.slot_bytes = (uint32_t)slot_bytes;
  a.so_off = (uint32_t)(S * slot_bytes);
  a.part_off = a.so_off + (uint32_t)(2 * so_stride);
  a.misc_off = a.part_off + (uint32_t)align_up(part_max, 16);
  a.x_off = a.misc_off + (uint32_t)align_up(misc, 16);
  a.win_off = a.x_off + (uint32_t)align_up(((size_t)max_cols + 1) * 4, 16);
  a.bar_off = (uint32_t)align_up(a.win_off + (size_t)kChainCons * kWinWords * 4, 8);
  p->smem = a.bar_off + (uint32_t)(2 * S + 5) * 8;
  p->grid = grid, p->nsteps = n;
  const size_t bytes_steps = align_up(sizeof(ChainStep) * n, 256), bytes_ctas = align_up(sizeof(ChainCta) * hc.size(), 256);
  cudaError_t e = cudaMalloc(&p->dmem, bytes_steps + bytes_ctas + 4 * (size_t)n);
  if (e == cudaSuccess) e = cudaMemcpy(p->dmem, hs.data(), sizeof(ChainStep) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy((uint8_t*)p->dmem + bytes_steps, hc.data(), sizeof(ChainCta) * hc.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem);
  if (e == cudaSuccess && std::getenv("QW_CHAIN_WATCH")) {  // diagnostics: hang -> record + trap
    static unsigned* host_watch = nullptr;
    if (!host_watch) {
      e = cudaHostAlloc((void**)&host_watch, 148 * 32 * 8 * 4 * 4, cudaHostAllocMapped);
      if (e == cudaSuccess) std::memset(host_watch, 0, 148 * 32 * 8 * 4 * 4);
    }
    unsigned* dptr = nullptr;
    if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&dptr, host_watch, 0);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_chain_watch, &dptr, sizeof(dptr));
    chain_watch_host() = host_watch;
  }
  if (e != cudaSuccess) {
    free_chain(p);
    return (int)e;
  }
  a.steps = reinterpret_cast<const ChainStep*>(p->dmem);
  a.ctas = reinterpret_cast<const ChainCta*>((uint8_t*)p->dmem + bytes_steps);
  a.done = reinterpret_cast<unsigned*>((uint8_t*)p->dmem + bytes_steps + bytes_ctas);
  *out = p;
  return 0;
}

int launch_chain(const ChainPlan* p, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(p->args.done, 0, 4 * (size_t)p->nsteps, st);
  if (e != cudaSuccess) return (int)e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->grid);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = p->smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the step counters are grid-wide
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {const_cast<ChainArgs*>(&p->args)};
  return (int)cudaLaunchKernelExC(&cfg, (const void*)chain_kernel, params);
}

void free_chain(ChainPlan* p) {
  if (!p) return;
  if (p->dmem) cudaFree(p->dmem);
  delete p;
}
}  // namespace qwdev
