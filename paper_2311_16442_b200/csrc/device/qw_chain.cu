// qw_chain.cu -- the persistent decode-chain kernel (batch 1): a fixed
// sequence of launch steps run by ONE kernel (see the comment below and
// DESIGN.md "Decode chain kernel").
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "qw_device.hpp"
#include "qw_gemv_common.cuh"
#include "qw_ptx.cuh"

namespace qwdev {

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
  if (e == cudaSuccess && qwdev::knob_str("QW_CHAIN_WATCH")) {  // diagnostics: hang -> record + trap
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
