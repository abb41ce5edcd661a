// qw_gemv.cu -- the hot path: y = W_q x for the mixed 2/4-bit layer, one
// fused kernel per activation column.
//
// Reference semantics: matvec_oracle (engine.cpp:169-183) over the stages
// row_fetch_params / row_compute_scales / row_decode / row_fma
// (engine.cpp:40-122), the activation gather of checked_permute /
// apply_permutation (engine.cpp:124-132, plan.cpp:107-116) and the CSR
// outliers of sparse_matvec (outliers.cpp:131-141).
//
// CTA roles (warp-specialised, persistent over a contiguous range of 4-row
// quad records; small enough that the next kernel's CTA fits beside it):
//   producer   TMA bulk copies: the CTA's 2-order rows once, then one quad
//              record per mbarrier (a ring when the range exceeds smem).
//              Never waits on the previous kernel, so under programmatic
//              dependent launch the weights stream while it still runs.
//   consumers  W warps; lane <-> 16-channel group(s).  Prologue: gather the
//              group's 16 activations (permutation prefetched before
//              griddepcontrol.wait), scale to fp16.  Then per quad: decode
//              its groups for the quad's two row pairs and store 4 row
//              partials; every `win` quads the warps sum the partials in a
//              fixed order (deterministic) into per-row dense sums.
//   csr        the CTA's outliers: exact fp32 products with x, summed per row
//              in CSR order; joins the consumers for the final y store.
//
// Code unpack: a code masked into the mantissa of an fp16 whose exponent
// field is zero reads as c * 2^(bitpos-24) exactly (a subnormal: no implicit
// one to remove).  Rows 2p and 2p+1 share each 32-bit word (qw_layout.hpp),
// so one AND + one HFMA2 multiplies one channel of two rows by x'_k
// pre-scaled by 2^-bitpos; every product is c * x0 * 2^-24 in a common
// scale and the accumulator's two halves are the two rows.  Zero points are
// applied per group as sum((c - z) x) = sum(c x) - z * sum(x); scales and
// zeros of the two rows go through packed fp32x2 instructions.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

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
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
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
// two small non-negative integers -> exact floats (2^23 magic, one FADD2)
__device__ __forceinline__ float2 small_ints_to_float2(uint32_t lo, uint32_t hi) {
  return fadd2(make_float2(__uint_as_float(0x4B000000u | lo), __uint_as_float(0x4B000000u | hi)),
               make_float2(-8388608.0f, -8388608.0f));
}
__device__ __forceinline__ float pow2f(int e) {  // 2^e for -126 <= e <= 127
  return __uint_as_float((uint32_t)(e + 127) << 23);
}

// ------------------------------------------------------------ unpack + dot
// 2-bit row pair: w0 = channels 0-7 of rows A|B, w1 = channels 8-15; channel
// j of a half at bits 2j.  X[k] = {x'_k, x'_k} pre-scaled by 2^-2(k%4).
// Returns {sum over the group for row A, for row B}.  Four independent
// 4-long HFMA2 chains keep the issue slots busy (fixed-latency stalls
// dominated with one 8-long chain per word).
__device__ __forceinline__ float2 dot_pair_2bit(uint32_t w0, uint32_t w1, const half2* X) {
  const uint32_t h0 = w0 >> 8, h1 = w1 >> 8;
  half2 a = __hmul2(as_h2(w0 & 0x00030003u), X[0]);
  half2 b = __hmul2(as_h2(h0 & 0x00030003u), X[4]);
  half2 c = __hmul2(as_h2(w1 & 0x00030003u), X[8]);
  half2 d = __hmul2(as_h2(h1 & 0x00030003u), X[12]);
  a = __hfma2(as_h2(w0 & 0x000C000Cu), X[1], a);
  b = __hfma2(as_h2(h0 & 0x000C000Cu), X[5], b);
  c = __hfma2(as_h2(w1 & 0x000C000Cu), X[9], c);
  d = __hfma2(as_h2(h1 & 0x000C000Cu), X[13], d);
  a = __hfma2(as_h2(w0 & 0x00300030u), X[2], a);
  b = __hfma2(as_h2(h0 & 0x00300030u), X[6], b);
  c = __hfma2(as_h2(w1 & 0x00300030u), X[10], c);
  d = __hfma2(as_h2(h1 & 0x00300030u), X[14], d);
  a = __hfma2(as_h2(w0 & 0x00C000C0u), X[3], a);
  b = __hfma2(as_h2(h0 & 0x00C000C0u), X[7], b);
  c = __hfma2(as_h2(w1 & 0x00C000C0u), X[11], c);
  d = __hfma2(as_h2(h1 & 0x00C000C0u), X[15], d);
  return __half22float2(__hadd2(__hadd2(a, b), __hadd2(c, d)));
}
// 4-bit row pair: word j = channels 4j..4j+3 of rows A|B, nibble i of a half
// at bits 4i.  X[k] pre-scaled by 2^-4(k%2).
__device__ __forceinline__ float2 dot_pair_4bit(const uint32_t* w, const half2* X) {
  half2 acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc[j] = __hmul2(as_h2(w[j] & 0x000F000Fu), X[4 * j + 0]);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = __hfma2(as_h2(w[j] & 0x00F000F0u), X[4 * j + 1], acc[j]);
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = __hfma2(as_h2((w[j] >> 8) & 0x000F000Fu), X[4 * j + 2], acc[j]);
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = __hfma2(as_h2((w[j] >> 8) & 0x00F000F0u), X[4 * j + 3], acc[j]);
  return __half22float2(__hadd2(__hadd2(acc[0], acc[1]), __hadd2(acc[2], acc[3])));
}

// ------------------------------------------------------------ prologue
// A lane's view of one 16-channel group: x'_k duplicated into both fp16
// halves and pre-scaled by 2^-bitpos(k), with max|x0| in [2^14, 2^15) (full
// fp16 precision, partial sums below 1, any finite fp32 x); minus their sum
// in product units; and the power-of-two factor back to x.
struct XGroup {
  half2 X[16];
  float nsx, ex;
};
// compact form kept in shared memory for layers too wide for registers
struct XGroupSm {
  __half h[16];
  float nsx, ex;
};

// pw: the group's 16 permuted->original channel indices (u16, two per word);
// pads (2-bit slots n2 <= s < n2p) read 0 as in apply_permutation.
__device__ __forceinline__ void prepare_group(__half* hx, float& nsx, float& ex, uint32_t g,
                                              bool two, const uint32_t* pw,
                                              const float* __restrict__ x, uint32_t n2,
                                              uint32_t n2p) {
  float v[16];
  const uint32_t s0 = 16u * g;
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __ldg(x + ((pw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu));
  if (s0 + 16u > n2 && s0 < n2p) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (s0 + k >= n2 && s0 + k < n2p) v[k] = 0.0f;
  }
  float m = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; ++k) m = fmaxf(m, fabsf(v[k]));
  // sh = floor(log2 max) - 14 from the exponent bits; tiny, huge and zero
  // groups take the exact slow path
  const uint32_t eb = (__float_as_uint(m) >> 23) & 0xFFu;
  int sh = (int)eb - 127 - 14;
  const bool fast = eb >= 20 && eb <= 220;
  if (!fast) sh = (m > 0.0f && m <= 3.4e38f) ? ilogbf(m) - 14 : 0;
  float2 sx = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const int b0 = two ? 2 * (k & 3) : 4 * (k & 1);
    const int b1 = two ? 2 * ((k + 1) & 3) : 4 * ((k + 1) & 1);
    float2 vv;
    if (fast) {
      vv = fmul2(make_float2(v[k], v[k + 1]), make_float2(pow2f(-sh - b0), pow2f(-sh - b1)));
    } else {
      vv = make_float2(ldexpf(v[k], -sh - b0), ldexpf(v[k + 1], -sh - b1));
    }
    const half2 h = __floats2half2_rn(vv.x, vv.y);
    hx[k] = __low2half(h), hx[k + 1] = __high2half(h);
    sx = ffma2(__half22float2(h), make_float2(pow2f(b0 - 24), pow2f(b1 - 24)), sx);
  }
  nsx = -(sx.x + sx.y);
  ex = (sh + 24 <= 127 && sh + 24 >= -126) ? pow2f(sh + 24) : ldexpf(1.0f, sh + 24);
}

// ------------------------------------------------------------ K2+K3 GEMV
struct GemvArgs {
  const uint8_t* quads;
  const uint32_t* sorder;
  const uint32_t* row_ptr;
  const uint32_t* csr;
  const uint16_t* perm;
  const float* x;
  float* y;
  Geometry g;
  uint32_t W, K, nslot, uq, win, nchunks, grid, nq_max;
  uint32_t repeat;  // diagnostics: consumers re-run the resident quads this many times
  uint32_t so_off, part_off, xg_off, misc_off, bar_off;
  unsigned long long* dbg;  // optional timeline: kTimelineEvents clock64 stamps per CTA
  uint32_t csr_lo[kMaxGrid + 1];
};

// timeline probe (diagnostics only; dbg == nullptr in production launches)
__device__ __forceinline__ void stamp(unsigned long long* dbg, uint32_t ev) {
  if (dbg) dbg[blockIdx.x * kTimelineEvents + ev] = clock64();
}

// 2-order rows of the quad: A = scale2 * ex, B = -zero2 * A per row
template <bool UNI>
__device__ __forceinline__ void quad_scales(float2& A01, float2& B01, float2& A23, float2& B23,
                                            const uint32_t* so, uint32_t rbq, uint32_t rbpat,
                                            uint32_t G2s, uint32_t g, float ex) {
  if (UNI) {
    const uint32_t e = so[rbq * G2s + g];
    const float A = half_bits_to_float(e) * ex;  // exact: scale2 * 2^k
    const float B = -small_int_to_float(e >> 16) * A;
    A01 = A23 = make_float2(A, A);
    B01 = B23 = make_float2(B, B);
  } else {
    float A[4], B[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t e = so[(rbq + ((rbpat >> (8 * i)) & 0xFFu)) * G2s + g];
      A[i] = half_bits_to_float(e) * ex;
      B[i] = -small_int_to_float(e >> 16) * A[i];
    }
    A01 = make_float2(A[0], A[1]), A23 = make_float2(A[2], A[3]);
    B01 = make_float2(B[0], B[1]), B23 = make_float2(B[2], B[3]);
  }
}

struct LaneGroup {
  uint32_t g, code_off, par_off, z_off, esh, emask, zsh;
  bool live, two;
};

template <int KMAX, bool XREG, bool UNI>
__global__ void __launch_bounds__(576, 1) gemv_kernel(const __grid_constant__ GemvArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Geometry& G = a.g;
  const uint32_t W = a.W, nslot = a.nslot, dense = G.dense_bytes;
  uint8_t* s_dense = smem;
  const uint32_t* s_so = reinterpret_cast<const uint32_t*>(smem + a.so_off);
  float* s_part = reinterpret_cast<float*>(smem + a.part_off);
  XGroupSm* s_xg = reinterpret_cast<XGroupSm*>(smem + a.xg_off);
  float* s_dsum = reinterpret_cast<float*>(smem + a.misc_off);
  float* s_csr = s_dsum + a.nq_max * 4;
  uint32_t* s_rp = reinterpret_cast<uint32_t*>(s_csr + a.nq_max * 4);
  float* s_prod = reinterpret_cast<float*>(s_rp + a.nq_max * 4 + 4);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* s_empty = s_full + nslot;
  uint64_t* s_sobar = s_empty + nslot;

  const uint32_t q0 = (uint32_t)((uint64_t)blockIdx.x * G.quads / a.grid);
  const uint32_t q1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * G.quads / a.grid);
  const uint32_t nq = q1 - q0;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t r_begin = q0 * kRowsPerQuad;
  const uint32_t r_end = min(q1 * kRowsPerQuad, G.rows);
  const uint32_t nrows = r_end - r_begin;
  const uint32_t rb_first = r_begin / G.group2;

  if (threadIdx.x < nslot) {
    mbar_init(&s_full[threadIdx.x], 1);
    mbar_init(&s_empty[threadIdx.x], W);
  }
  if (threadIdx.x == 32) mbar_init(s_sobar, 1);
  if (threadIdx.x == 0) stamp(a.dbg, 0);  // entry
  mbar_fence_init();
  __syncthreads();
  pdl_launch_dependents();

  if (warp == W) {
    // ================= producer: the weight stream does not depend on x
    if (lane == 0) {
      const uint32_t so_bytes = ((r_end - 1) / G.group2 - rb_first + 1) * G.G2s * 4u;
      if (so_bytes) {
        mbar_expect_tx(s_sobar, so_bytes);
        bulk_load_nohint(smem + a.so_off, a.sorder + (size_t)rb_first * G.G2s, so_bytes, s_sobar);
      } else {
        mbar_arrive(s_sobar);
      }
      const uint8_t* src = a.quads + (size_t)q0 * dense;
      const uint32_t uq = a.uq, nunit = (nq + uq - 1) / uq;
      uint32_t slot = 0, phase = 0;
      for (uint32_t u = 0; u < nunit; ++u) {
        const uint32_t bytes = min(uq, nq - uq * u) * dense;
        if (u >= nslot) mbar_wait(&s_empty[slot], phase ^ 1u);
        mbar_expect_tx(&s_full[slot], bytes);
        bulk_load_nohint(s_dense + (size_t)slot * uq * dense, src, bytes, &s_full[slot]);
        if (u < 8) stamp(a.dbg, 26 + u);  // unit u copy issued
        src += bytes;
        if (++slot == nslot) slot = 0, phase ^= 1u;
        if (u + 1 == min(nunit, nslot)) stamp(a.dbg, 1);  // first ring of copies issued
      }
      stamp(a.dbg, 2);  // all copies issued
      if (a.dbg && nunit <= nslot)  // diagnostics: when each unit landed
        for (uint32_t u = 0; u < nunit && u < 8; ++u) {
          mbar_wait(&s_full[u], 0);
          stamp(a.dbg, 34 + u);
        }
    }
    return;
  }

  if (warp == W + 1) {
    // ================= outliers: exact fp32 x, CSR order within a row
    const uint32_t e_lo = a.csr_lo[blockIdx.x], e_hi = a.csr_lo[blockIdx.x + 1];
    for (uint32_t t = lane; t <= nrows; t += 32) s_rp[t] = a.row_ptr[r_begin + t] - e_lo;
    for (uint32_t t = lane; t < nrows; t += 32) s_csr[t] = 0.0f;
    const uint32_t n = e_hi - e_lo;
    constexpr int kPer = 8;
    uint32_t ent[kPer], src[kPer];
    auto fetch = [&](uint32_t c0) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint32_t e = c0 + lane + 32u * j;
        ent[j] = e < n ? __ldg(a.csr + e_lo + e) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kPer; ++j) src[j] = __ldg(a.perm + (ent[j] & 0xFFFFu));
    };
    if (n) fetch(0);
    __syncwarp();
    if (n) pdl_wait();  // x is the previous kernel's output
    for (uint32_t c0 = 0; c0 < n; c0 += 32u * kPer) {
      const uint32_t c1 = min(c0 + 32u * kPer, n);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint32_t e = c0 + lane + 32u * j;
        if (e < c1) s_prod[e - c0] = half_bits_to_float(ent[j] >> 16) * __ldg(a.x + src[j]);
      }
      __syncwarp();
      if (c1 < n) fetch(c1);
      for (uint32_t t = lane; t < nrows; t += 32) {
        const uint32_t lo = max(s_rp[t], c0), hi = min(s_rp[t + 1], c1);
        float s = s_csr[t];
        for (uint32_t e = lo; e < hi; ++e) s += s_prod[e - c0];
        s_csr[t] = s;
      }
      __syncwarp();
    }
    if (lane == 0) stamp(a.dbg, 3);  // outliers done
    named_sync(2, (W + 1) * 32);     // meet the consumers for the y store
    return;
  }

  // ================= consumers
  LaneGroup lg[KMAX];
  XGroup xr[XREG ? KMAX : 1];
  uint32_t pw[XREG ? KMAX : 1][8];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    LaneGroup& L = lg[k];
    const uint32_t c = warp + (uint32_t)k * W;
    L.g = c * 32u + lane;
    L.live = k < (int)a.K && c < a.nchunks && L.g < G.G;
    L.two = L.g < G.G2;
    if (L.two) {
      const uint32_t t = L.g / 3u, sub = L.g - 3u * t;
      L.code_off = 16u * L.g;
      L.par_off = G.off_meta + 8u * t;
      L.z_off = 0;
      L.zsh = 2u * sub;
      L.esh = sub == 0 ? 6u : (sub == 1 ? 9u : 12u);  // 4/3/3 rule: eff = scode << 1
      L.emask = sub == 0 ? 15u : 14u;
    } else {
      const uint32_t b = L.g - G.G2;
      L.code_off = G.off_c4 + 32u * b;
      L.par_off = G.off_s4 + 8u * b;
      L.z_off = G.off_z4 + 2u * b;
      L.zsh = L.esh = L.emask = 0;
    }
    if (XREG && L.live) {  // prologue, part 1: permutation (layer data)
      const uint4* pp = reinterpret_cast<const uint4*>(a.perm + 16u * L.g);
      const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
      uint32_t* d = pw[XREG ? k : 0];
      d[0] = p0.x, d[1] = p0.y, d[2] = p0.z, d[3] = p0.w;
      d[4] = p1.x, d[5] = p1.y, d[6] = p1.z, d[7] = p1.w;
    }
  }
  pdl_wait();  // x is the previous kernel's output
  if (threadIdx.x == 0) stamp(a.dbg, 6);
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const LaneGroup& L = lg[k];
    if (!L.live) continue;
    if (XREG) {
      __half hx[16];
      XGroup& o = xr[XREG ? k : 0];
      prepare_group(hx, o.nsx, o.ex, L.g, L.two, pw[XREG ? k : 0], a.x, G.cols - G.n4, G.n2p);
#pragma unroll
      for (int j = 0; j < 16; ++j) o.X[j] = __half2half2(hx[j]);
    } else {
      const uint4* pp = reinterpret_cast<const uint4*>(a.perm + 16u * L.g);
      const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
      const uint32_t pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
      XGroupSm& o = s_xg[L.g];  // lane-private entry
      prepare_group(o.h, o.nsx, o.ex, L.g, L.two, pv, a.x, G.cols - G.n4, G.n2p);
    }
  }
  if (threadIdx.x == 0) stamp(a.dbg, 7);
  mbar_wait(s_sobar, 0);

  // 2-order row block of the current quad, tracked without divisions
  uint32_t rbq = 0, rb_left = 0, rbpat = 0, rel3 = 0, row_left = 0;
  if (UNI) {
    const uint32_t g2q = G.group2 / kRowsPerQuad;
    rb_left = g2q - (r_begin / kRowsPerQuad) % g2q;
  } else {
    row_left = G.group2 - r_begin % G.group2;  // rows left in rb_first
  }
  const uint32_t win = a.win;
  // 2-order block of the next quad (rbq, rbpat) and advance past it
  auto quad_rb = [&](uint32_t& q_rb, uint32_t& q_pat) {
    if (UNI) {
      q_rb = rbq, q_pat = 0;
      if (--rb_left == 0) ++rbq, rb_left = G.group2 / kRowsPerQuad;
    } else {
      uint32_t rel[4];
      uint32_t cur = rel3;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (row_left == 0) ++cur, row_left = G.group2;
        rel[i] = cur;
        --row_left;
      }
      rel3 = cur;
      q_rb = rel[0];
      q_pat = (rel[1] - rel[0]) << 8 | (rel[2] - rel[0]) << 16 | (rel[3] - rel[0]) << 24;
    }
  };
  // one unit = up to two quads in one slot; NQ quads are decoded together so
  // their independent dot-product chains interleave
  auto unit = [&](auto nq_tag, const uint8_t* sb, const uint32_t* q_rb, const uint32_t* q_pat,
                  float2* acc01, float2* acc23) {
    constexpr int NQ = decltype(nq_tag)::value;
#pragma unroll
    for (int j = 0; j < NQ; ++j) acc01[j] = acc23[j] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      const LaneGroup& L = lg[k];
      if (!L.live) continue;
      half2 xs[XREG ? 1 : 16];
      const half2* X;
      float ex, nsx;
      if (XREG) {
        X = xr[XREG ? k : 0].X, ex = xr[XREG ? k : 0].ex, nsx = xr[XREG ? k : 0].nsx;
      } else {
        const XGroupSm& o = s_xg[L.g];
#pragma unroll
        for (int j = 0; j < 16; ++j) xs[XREG ? 0 : j] = __half2half2(o.h[j]);
        X = xs, ex = o.ex, nsx = o.nsx;
      }
      const float2 nsx2 = make_float2(nsx, nsx);
      if (L.two) {
        // ---- 2-bit group: meta, 2-order -> 1-order scale, decode, FMA
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const uint8_t* qb = sb + (size_t)j * dense;
          const uint4 w = *reinterpret_cast<const uint4*>(qb + L.code_off);
          const uint2 m = *reinterpret_cast<const uint2*>(qb + L.par_off);
          float2 A01, B01, A23, B23;
          quad_scales<UNI>(A01, B01, A23, B23, s_so, q_rb[j], q_pat[j], G.G2s, L.g, ex);
          const float2 P01 = dot_pair_2bit(w.x, w.y, X);
          const float2 P23 = dot_pair_2bit(w.z, w.w, X);
          const float2 e01 = small_ints_to_float2((m.x >> L.esh) & L.emask, (m.x >> (L.esh + 16)) & L.emask);
          const float2 e23 = small_ints_to_float2((m.y >> L.esh) & L.emask, (m.y >> (L.esh + 16)) & L.emask);
          const float2 z01 = small_ints_to_float2((m.x >> L.zsh) & 3u, (m.x >> (L.zsh + 16)) & 3u);
          const float2 z23 = small_ints_to_float2((m.y >> L.zsh) & 3u, (m.y >> (L.zsh + 16)) & 3u);
          // s1 = (eff - zero2) * scale2 (engine.cpp:48-63); acc += s1 * sum((c - z) x)
          acc01[j] = ffma2(ffma2(e01, A01, B01), ffma2(z01, nsx2, P01), acc01[j]);
          acc23[j] = ffma2(ffma2(e23, A23, B23), ffma2(z23, nsx2, P23), acc23[j]);
        }
      } else {
        // ---- 4-bit block
        const float2 ex2 = make_float2(ex, ex);
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const uint8_t* qb = sb + (size_t)j * dense;
          const uint4 wa = *reinterpret_cast<const uint4*>(qb + L.code_off);
          const uint4 wb = *reinterpret_cast<const uint4*>(qb + L.code_off + 16u);
          const uint2 s4 = *reinterpret_cast<const uint2*>(qb + L.par_off);
          const uint32_t z4 = *reinterpret_cast<const uint16_t*>(qb + L.z_off);
          const uint32_t pa[4] = {wa.x, wa.y, wa.z, wa.w}, pb[4] = {wb.x, wb.y, wb.z, wb.w};
          const float2 P01 = dot_pair_4bit(pa, X);
          const float2 P23 = dot_pair_4bit(pb, X);
          const float2 s01 = fmul2(make_float2(half_bits_to_float(s4.x), half_bits_to_float(s4.x >> 16)), ex2);
          const float2 s23 = fmul2(make_float2(half_bits_to_float(s4.y), half_bits_to_float(s4.y >> 16)), ex2);
          const float2 z01 = small_ints_to_float2(z4 & 15u, (z4 >> 4) & 15u);
          const float2 z23 = small_ints_to_float2((z4 >> 8) & 15u, z4 >> 12);
          acc01[j] = ffma2(s01, ffma2(z01, nsx2, P01), acc01[j]);
          acc23[j] = ffma2(s23, ffma2(z23, nsx2, P23), acc23[j]);
        }
      }
    }
  };
  const uint32_t uq = a.uq, nunit = (nq + uq - 1) / uq;
  const uint32_t reps = (a.repeat > 1 && nunit <= nslot) ? a.repeat : 1;
  uint32_t slot = 0, phase = 0, wq = 0, wbase = 0;
  for (uint32_t it = 0; it < reps * nunit; ++it) {
    const uint32_t u = it % nunit;
    if (u == 0 && it) {  // diagnostics re-run: same quads, fresh sums
      slot = 0, phase = 0, wq = 0, wbase = 0, rbq = 0, rel3 = 0;
      if (UNI) rb_left = G.group2 / kRowsPerQuad - (r_begin / kRowsPerQuad) % (G.group2 / kRowsPerQuad);
      else row_left = G.group2 - r_begin % G.group2;
    }
    const uint32_t nu = min(uq, nq - uq * u);
    uint32_t q_rb[2], q_pat[2];
    quad_rb(q_rb[0], q_pat[0]);
    if (nu == 2) quad_rb(q_rb[1], q_pat[1]);
    mbar_wait(&s_full[slot], phase);
    if (threadIdx.x == 0 && it == 0) stamp(a.dbg, 8);
    if (threadIdx.x == 0 && it < 8) stamp(a.dbg, 10 + 2 * it);
    const uint8_t* sb = s_dense + (size_t)slot * uq * dense;
    float2 acc01[2], acc23[2];
    if (nu == 2)
      unit(std::integral_constant<int, 2>{}, sb, q_rb, q_pat, acc01, acc23);
    else
      unit(std::integral_constant<int, 1>{}, sb, q_rb, q_pat, acc01, acc23);
    if (threadIdx.x == 0 && it < 8) stamp(a.dbg, 11 + 2 * it);
    if (nunit > nslot) {  // ring: hand the slot back once every warp read it
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[slot]);
    }
    // row partials: [window quad][row][warp][lane] -- conflict-free stores
    for (uint32_t j = 0; j < nu; ++j) {
      float* pq = s_part + ((size_t)(wq + j) * 4 * W + warp) * 32 + lane;
      pq[0] = acc01[j].x, pq[W * 32] = acc01[j].y, pq[2 * W * 32] = acc23[j].x, pq[3 * W * 32] = acc23[j].y;
    }
    wq += nu;
    if (++slot == nslot) slot = 0, phase ^= 1u;
    if (wq >= win || u + 1 == nunit) {
      if (u + 1 == nunit && it + 1 < reps * nunit) {  // not the last re-run: skip the sums
        wq = 0;
        continue;
      }
      // window complete: fixed-order sums of its rows, one row per warp pass
      named_sync(1, W * 32);
      const uint32_t wrows = wq * 4;
      for (uint32_t r = warp; r < wrows; r += W) {
        const float* pr = s_part + (size_t)r * W * 32 + lane;
        float s = pr[0];
        for (uint32_t w2 = 1; w2 < W; ++w2) s += pr[w2 * 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        if (lane == 0) s_dsum[wbase + r] = s;
      }
      named_sync(1, W * 32);
      wbase += wrows, wq = 0;
    }
  }
  if (threadIdx.x == 0) stamp(a.dbg, 9);
  named_sync(2, (W + 1) * 32);  // outlier sums are complete
  // the dense sum first, then the outliers, as row_fma (engine.cpp:111-122)
  for (uint32_t t = threadIdx.x; t < nrows; t += W * 32) a.y[r_begin + t] = s_dsum[t] + s_csr[t];
  if (threadIdx.x == 0) stamp(a.dbg, 5);
}

using GemvFn = void (*)(GemvArgs);

template <bool UNI>
GemvFn pick_uni(uint32_t kmax) {
  if (kmax <= 1) return gemv_kernel<1, true, UNI>;
  if (kmax <= 2) return gemv_kernel<2, true, UNI>;
  if (kmax <= 4) return gemv_kernel<4, false, UNI>;
  return gemv_kernel<8, false, UNI>;
}
GemvFn pick_kernel(uint32_t kmax, bool uni) { return uni ? pick_uni<true>(kmax) : pick_uni<false>(kmax); }

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

int plan_gemv(DeviceLayer& L, int num_sms, const uint32_t* host_row_ptr) {
  const Geometry& G = L.g;
  GemvPlan& p = L.plan;
  p.nchunks = (G.G + 31u) / 32u;
  // consumers: W warps, kmax chunks (of 32 groups) per warp; <= 16 warps keeps
  // a CTA small enough that the next kernel's CTA can sit beside it
  p.kmax = (p.nchunks + 15) / 16;
  if (p.kmax > 8) return (int)cudaErrorInvalidConfiguration;
  if (p.kmax == 1 && p.nchunks > 8) p.kmax = 2;  // fewer, fuller warps (registers hold 2)
  p.warps = (p.nchunks + p.kmax - 1) / p.kmax;
  p.teams = 1;
  p.grid = std::min<uint32_t>(std::min<uint32_t>((uint32_t)num_sms, kMaxGrid), G.quads);
  p.nq_max = (G.quads + p.grid - 1) / p.grid;
  p.uniform_rb = (G.group2 % kRowsPerQuad) == 0;
  // the largest 2-order block range of any CTA
  uint32_t so_rows_max = 0;
  for (uint32_t b = 0; b <= p.grid; ++b) {
    const uint32_t q = (uint32_t)((uint64_t)b * G.quads / p.grid);
    p.csr_lo[b] = host_row_ptr[std::min(q * (uint32_t)kRowsPerQuad, G.rows)];
    if (b < p.grid) {
      const uint32_t qn = (uint32_t)((uint64_t)(b + 1) * G.quads / p.grid);
      const uint32_t r0 = q * kRowsPerQuad, r1 = std::min(qn * kRowsPerQuad, G.rows);
      so_rows_max = std::max(so_rows_max, (r1 - 1) / G.group2 - r0 / G.group2 + 1);
    }
  }
  const size_t so_bytes = (size_t)so_rows_max * G.G2s * 4;
  const bool xreg = p.kmax <= 2;
  const size_t xg_bytes = xreg ? 0 : (size_t)G.G * sizeof(XGroupSm);
  auto layout = [&](size_t nslot, size_t uq, size_t win, size_t* bar_off) {
    size_t off = align_up(nslot * uq * G.dense_bytes, 128);
    off += align_up(so_bytes, 16);
    off += win * 4 * p.warps * 32 * 4;
    off += align_up(xg_bytes, 16);
    off += (size_t)p.nq_max * 4 * 4 * 2 + ((size_t)p.nq_max * 4 + 4) * 4 + 256 * 4;
    off = align_up(off, 8);
    *bar_off = off;
    return off + (2 * nslot + 1) * 8;
  };
  // slots hold `uq` quads (2: two interleaved quads per consumer step); the
  // whole quad range resident when it fits in ~half an SM (so a PDL
  // successor fits too), else a ring in the whole SM
  const size_t half_sm = 112 * 1024, full_sm = 220 * 1024;
  size_t uq = 2, nslot = 0, win = 0, bar = 0;
  for (; uq >= 1; --uq) {
    const size_t units = (p.nq_max + uq - 1) / uq;
    nslot = units, win = std::min<size_t>(8, uq * units);
    if (layout(nslot, uq, win, &bar) > half_sm) {
      nslot = std::min<size_t>(units, 4);
      while (nslot > 2 && layout(nslot, uq, win, &bar) > full_sm) --nslot;
      while (win > 2 * uq && layout(nslot, uq, win, &bar) > full_sm) win -= uq;
    }
    if (layout(nslot, uq, win, &bar) <= full_sm) break;
  }
  if (uq == 0) return (int)cudaErrorInvalidConfiguration;
  p.uq = (uint32_t)uq;
  p.smem = (uint32_t)layout(nslot, uq, win, &bar);
  p.nslot = (uint32_t)nslot;
  p.win = (uint32_t)win;
  p.so_off = (uint32_t)align_up(nslot * uq * G.dense_bytes, 128);
  p.part_off = p.so_off + (uint32_t)align_up(so_bytes, 16);
  p.xg_off = p.part_off + (uint32_t)(win * 4 * p.warps * 32 * 4);
  p.misc_off = p.xg_off + (uint32_t)align_up(xg_bytes, 16);
  p.bar_off = (uint32_t)bar;
  static bool attr_set = false;  // raise the opt-in limit once per process
  if (!attr_set) {
    for (bool uni : {false, true})
      for (uint32_t k : {1u, 2u, 4u, 8u}) {
        cudaError_t err = cudaFuncSetAttribute(pick_kernel(k, uni),
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(227 * 1024));
        if (err != cudaSuccess) return (int)err;
      }
    attr_set = true;
  }
  return 0;
}

int launch_gemv(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream,
                bool pdl, unsigned long long* dbg, uint32_t repeat) {
  const Geometry& G = L.g;
  const GemvPlan& p = L.plan;
  GemvArgs a;
  a.quads = L.quads;
  a.sorder = L.sorder;
  a.row_ptr = L.row_ptr;
  a.csr = L.csr;
  a.perm = L.perm16;
  a.g = G;
  a.W = p.warps, a.K = p.kmax, a.nslot = p.nslot, a.uq = p.uq, a.win = p.win;
  a.nchunks = p.nchunks, a.grid = p.grid, a.nq_max = p.nq_max;
  a.so_off = p.so_off, a.part_off = p.part_off, a.xg_off = p.xg_off, a.misc_off = p.misc_off;
  a.bar_off = p.bar_off;
  a.dbg = dbg;
  a.repeat = repeat;
  std::copy(p.csr_lo, p.csr_lo + p.grid + 1, a.csr_lo);
  const GemvFn fn = pick_kernel(p.kmax, p.uniform_rb);
  const uint32_t threads = (p.warps + 2) * 32;
  for (uint32_t col = 0; col < batch; ++col) {
    a.x = x + (size_t)col * G.cols;
    a.y = y + (size_t)col * G.rows;
    void* params[] = {&a};
    cudaError_t err = launch_ex((const void*)fn, dim3(p.grid), dim3(threads), p.smem,
                                (cudaStream_t)stream, pdl, params);
    if (err != cudaSuccess) return (int)err;
  }
  return 0;
}

}  // namespace qwdev
