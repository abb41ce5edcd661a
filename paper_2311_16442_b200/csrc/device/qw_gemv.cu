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
#include <mutex>
#include <cstdint>
#include <type_traits>
#include <vector>

#include "qw_device.hpp"
#include "qw_gemv_common.cuh"
#include "qw_ptx.cuh"

namespace qwdev {
namespace {

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
  uint32_t seg_rows[kMaxSeg];  // output rows of each layer (a group may mix row counts: GQA q/k/v)
  const float* xs[kMaxSeg];    // the segment's input: one x for a layer group, one column each for a batch
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
  PeerOut peers;            // fused exchange: y rows also to peer buffers, then arrival counters
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


// The fused tensor-parallel exchange (GemvArgs::peers): the CTA's rows, summed
// exactly as for y, into every peer's buffer; once every consumer's stores
// are issued, thread 0 makes one cumulative system-scope release and adds
// the CTA's arrival to every peer's counter (qw_peer.cu waits for them).
__device__ __forceinline__ void push_peers(const PeerOut& po, const float* s_part, const float* s_csr, uint32_t W,
                                        uint32_t nrows, uint32_t r_begin, uint32_t nthreads) {
  for (uint32_t t = threadIdx.x; t < nrows; t += nthreads) {
    const float* p = s_part + t * W;
    float s = p[0];
    for (uint32_t w2 = 1; w2 < W; ++w2) s += p[w2];
    const float v = s + s_csr[t];
    for (uint32_t q = 0; q < po.n; ++q) po.y[q][r_begin + t] = v;
  }
  named_sync(4, nthreads);
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (uint32_t q = 0; q < po.n; ++q)
      asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(po.flag[q]) : "memory");
  }
}

// KG groups per lane, NQ quads per ring slot (decoded together for ILP),
// UNI: group2 % 4 == 0 (a quad never straddles 2-order blocks), XSM: x is
// staged in shared memory (TMA) before the gather.
// TM: two teams of consumer warps take alternate units (long quad ranges:
// group launches, wide layers); then the CTA owns the SM (no PDL co-residency).
template <int KG, int NQ, bool UNI, bool XSM, bool TM = false, bool PEER = false>
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
  const float* __restrict__ g_x = a.xs[seg];
  const float s_scale = a.s_scale[seg];
  const uint32_t nunit = (nq + NQ - 1) / NQ;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t r_begin = q0 * kRowsPerQuad;
  const uint32_t seg_rows = a.seg_rows[seg];
  const uint32_t r_end = min(q1 * kRowsPerQuad, seg_rows);
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
            const float xv = XSM ? s_x[w[j] & 0xFFFFu] : __ldg(g_x + (w[j] & 0xFFFFu));
            acc = __fadd_rn(acc, __fmul_rn(half_bits_to_float(w[j] >> 16), xv));  // no contraction
          }
        }
        for (; e < hi; ++e) {
          const uint32_t w = s_ent[e];
          acc = __fadd_rn(acc, __fmul_rn(half_bits_to_float(w >> 16), XSM ? s_x[w & 0xFFFFu] : __ldg(g_x + (w & 0xFFFFu))));
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
        if (e < c1) s_prod[e - c0] = half_bits_to_float(ent[j] >> 16) * (XSM ? s_x[src[j]] : __ldg(g_x + src[j]));
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
          const uint32_t rb = row_block(min(r0 + i, r_end - 1)) - rb_first;  // the staged row blocks only
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
        if (UNI && j > 0 && r0 < rb_end[j > 0 ? j - 1 : 0]) {
          // the unit's previous quad is in the same 2-order row block (loaded
          // just now): its scales, no second decode
#pragma unroll
          for (int kk = 0; kk < KG; ++kk) A2[j][kk][0] = A2[j - 1][kk][0], C2[j][kk][0] = C2[j - 1][kk][0];
          rb_end[j] = rb_end[j - 1];
        } else {
          load_scales(j, r0);
          rb_end[j] = (row_block(r0) + 1) * G.group2;
        }
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
    const bool xvec = (((uintptr_t)g_x) & 15u) == 0 && (G.cols & 3u) == 0;
    const float4* gx = reinterpret_cast<const float4*>(g_x);
    float4* sx4 = reinterpret_cast<float4*>(s_x);
    const uint32_t n4 = G.cols >> 2;
    constexpr int kXr = KG >= 2 ? 5 : 4;  // 5 x 16 B x 576 threads: 11008 channels in one round trip
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
        for (uint32_t i = tid; i < G.cols; i += nth) s_x[i] = __ldg(g_x + i);
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
      xs = g_x;
    }
    // Each team gathers and scales its own X (the same values: handing team
    // 0's X to team 1 through shared memory put a barrier over both teams in
    // front of the main loop, 2 % slower on the bench step).
    half2 X[KG][16], nsxh[KG];
    float yscale;
    {
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
  // fused TP exchange: a separate instantiation (PEER), so the kernels that
  // never push keep their code generation
  if constexpr (PEER) push_peers(a.peers, s_part, s_csr, W, nrows, r_begin, NC * 32);
  if (threadIdx.x == 0) stamp(a.dbg, 5);
}

using GemvFn = void (*)(GemvArgs);

// quads per ring slot of a one-group-per-lane kernel: 2, or 4 (diagnostics);
// the plan (quads_per_slot) and the instantiation (pick2) both read it here
uint32_t nq1() { return env_u32("QW_NQ1", 2) == 4 ? 4u : 2u; }

template <bool UNI, bool XSM, bool PEER = false>
GemvFn pick2(uint32_t kg) {
  switch (kg) {
    case 1:
      if (!UNI) return gemv_kernel<1, 1, UNI, XSM, false, PEER>;
      return nq1() == 2 ? gemv_kernel<1, 2, UNI, XSM, false, PEER> : gemv_kernel<1, UNI ? 4 : 1, UNI, XSM, false, PEER>;
    case 2: return gemv_kernel<2, UNI ? 2 : 1, UNI, XSM, false, PEER>;
    case 3: return gemv_kernel<3, 1, UNI, XSM, false, PEER>;
    default: return gemv_kernel<4, 1, UNI, XSM, false, PEER>;
  }
}
template <bool PEER = false>
GemvFn pick_teams(uint32_t kg) {
  return kg == 1 ? gemv_kernel<1, 2, true, true, true, PEER> : gemv_kernel<2, 2, true, true, true, PEER>;
}
GemvFn pick_kernel(uint32_t kg, bool uni, bool xsm) {
  return uni ? (xsm ? pick2<true, true>(kg) : pick2<true, false>(kg))
             : (xsm ? pick2<false, true>(kg) : pick2<false, false>(kg));
}
// the exchange variants: group2 % 4 == 0 layers only (every Llama config)
GemvFn pick_peer(uint32_t kg, bool xsm, bool teams) {
  return teams ? pick_teams<true>(kg) : (xsm ? pick2<true, true, true>(kg) : pick2<true, false, true>(kg));
}
uint32_t quads_per_slot(uint32_t kg, bool uni) {
  return !uni ? 1u : (kg == 1 ? nq1() : (kg == 2 ? 2u : 1u));
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

namespace {

// CTA ranges (one layer each) + shared-memory layout for the largest range
int plan_ctas(GemvPlan& p, const Geometry& G, const uint32_t* const* host_row_ptrs, const uint32_t* seg_rows,
              uint32_t n, int num_sms, uint32_t min_per_sm = 1) {
  uint32_t per_sm = min_per_sm;
  if (const char* e = qwdev::knob_str("QW_CTAS_PER_SM")) per_sm = std::max<uint32_t>(per_sm, std::atoi(e));
  uint64_t total = 0;
  uint32_t lq[kMaxSeg];
  for (uint32_t l = 0; l < n; ++l) lq[l] = (seg_rows[l] + kRowsPerQuad - 1) / kRowsPerQuad, total += lq[l];
  uint32_t grid = (uint32_t)std::min<uint64_t>(std::min<uint32_t>((uint32_t)num_sms * per_sm, kMaxGrid), total);
  grid = std::max(grid, n);
  p.grid = grid;
  p.nq_max = 0;
  // CTAs per layer in proportion to its quads (equal layers: an equal split)
  uint32_t gl[kMaxSeg], given = 0;
  uint64_t acc = 0;
  for (uint32_t l = 0; l < n; ++l) {
    acc += lq[l];
    const uint32_t upto = (uint32_t)(grid * acc / total);
    gl[l] = std::max<uint32_t>(1, std::min<uint32_t>(lq[l], upto > given ? upto - given : 1));
    given += gl[l];
  }
  while (given > grid) {  // rounding with the >= 1 floor: take CTAs back from the largest share
    uint32_t m = 0;
    for (uint32_t l = 1; l < n; ++l) m = gl[l] > gl[m] ? l : m;
    --gl[m], --given;
  }
  p.grid = grid = given;
  uint32_t so_rows_max = 0, cta = 0, ent_max = 0;
  for (uint32_t l = 0; l < n; ++l) {
    const uint32_t g_l = gl[l], quads = lq[l], rows = seg_rows[l];  // CTAs / quads / rows of layer l
    for (uint32_t b = 0; b < g_l; ++b, ++cta) {
      const uint32_t q0 = (uint32_t)((uint64_t)b * quads / g_l), q1 = (uint32_t)((uint64_t)(b + 1) * quads / g_l);
      p.cta_seg[cta] = (uint8_t)l;
      p.cta_q0[cta] = q0, p.cta_q1[cta] = q1;
      const uint32_t r0 = q0 * kRowsPerQuad, r1 = std::min(q1 * kRowsPerQuad, rows);
      p.cta_e0[cta] = host_row_ptrs[l][std::min(r0, rows)];
      p.cta_e1[cta] = host_row_ptrs[l][std::min(r1, rows)];
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
  // raise the opt-in limit once per device (the attribute is per device)
  static std::mutex attr_mu;
  static uint64_t attr_dev = 0;
  int cur = 0;
  cudaGetDevice(&cur);
  std::lock_guard<std::mutex> lk(attr_mu);
  if (cur >= 64 || !(attr_dev & (1ull << cur))) {
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
    for (bool teams : {false, true})
      for (bool xsm : {false, true})
        for (uint32_t k : {1u, 2u, 3u, 4u}) {
          if (teams && (!xsm || k > 2)) continue;
          cudaError_t err = cudaFuncSetAttribute(pick_peer(k, xsm, teams), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(227 * 1024));
          if (err != cudaSuccess) return (int)err;
        }
    if (cur < 64) attr_dev |= 1ull << cur;
  }
  return 0;
}
}  // namespace

// one CTA per SM first; when the CTA's share does not fit in shared memory
// (x, its 2-order rows -- one per row at group2 = 1 -- and a ring of at least
// two slots) up to three CTAs per SM, each with a third of the rows, run in
// waves
int plan_ctas_fit(GemvPlan& p, const Geometry& G, const uint32_t* const* host_row_ptrs, const uint32_t* seg_rows,
                  uint32_t n, int num_sms) {
  int e = 0;
  for (uint32_t f = 1; f <= 3; ++f)
    if ((e = plan_ctas(p, G, host_row_ptrs, seg_rows, n, num_sms, f)) != (int)cudaErrorInvalidConfiguration) break;
  return e;
}

int plan_gemv(DeviceLayer& L, int num_sms, const uint32_t* host_row_ptr) {
  GemvPlan& p = L.plan;
  if (int e = plan_geometry(p, L.g)) return e;
  const uint32_t* rp[1] = {host_row_ptr};
  const uint32_t rows[1] = {L.g.rows};
  return plan_ctas_fit(p, L.g, rp, rows, 1, num_sms);
}

int plan_gemv_group(GemvPlan& p, const DeviceLayer* const* layers, const uint32_t* const* host_row_ptrs,
                    uint32_t n, int num_sms) {
  if (n == 0 || n > kMaxSeg) return (int)cudaErrorInvalidValue;
  const Geometry& G = layers[0]->g;
  for (uint32_t l = 1; l < n; ++l) {
    const Geometry& H = layers[l]->g;
    // one decode body for all: same columns, channel split and 2-order group;
    // the row counts may differ (GQA q/k/v)
    if (H.cols != G.cols || H.n4 != G.n4 || H.n2p != G.n2p || H.group2 != G.group2 || H.dense_bytes != G.dense_bytes ||
        H.G2s != G.G2s)
      return (int)cudaErrorInvalidValue;
  }
  p = layers[0]->plan;  // geometry part is identical
  uint32_t rows[kMaxSeg];
  for (uint32_t l = 0; l < n; ++l) rows[l] = layers[l]->g.rows;
  return plan_ctas_fit(p, G, host_row_ptrs, rows, n, num_sms);
}

int launch_gemv_group(const GemvPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* const* xs,
                      float* const* ys, void* stream, bool pdl, uint32_t flags, unsigned long long* dbg,
                      uint32_t repeat, bool global_clock, const PeerOut* peers) {
  const Geometry& G = layers[0]->g;
  GemvArgs a;
  for (uint32_t l = 0; l < kMaxSeg; ++l) {
    const DeviceLayer& L = *layers[std::min(l, n - 1)];
    a.quads[l] = L.quads, a.sorder[l] = L.sorder, a.row_ptr[l] = L.row_ptr;
    a.csr[l] = L.csr, a.perm[l] = L.perm16, a.s_scale[l] = L.plan.s_scale;
    a.y[l] = ys[std::min(l, n - 1)];
    a.xs[l] = xs[std::min(l, n - 1)];
    a.seg_rows[l] = L.g.rows;
  }
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
  a.peers = PeerOut{};
  if (peers) a.peers = *peers;
  a.wait_x = (flags & kXIndependent) ? 0u : 1u;
  a.pre = p.pre, a.npre_max = p.npre_max, a.x_first = p.x_first, a.x_gate = p.x_gate;
  a.repeat = repeat;
  std::copy(p.cta_seg, p.cta_seg + p.grid, a.cta_seg);
  std::copy(p.cta_q0, p.cta_q0 + p.grid, a.cta_q0);
  std::copy(p.cta_q1, p.cta_q1 + p.grid, a.cta_q1);
  std::copy(p.cta_e0, p.cta_e0 + p.grid, a.cta_e0);
  std::copy(p.cta_e1, p.cta_e1 + p.grid, a.cta_e1);
  if (a.peers.n && !p.uniform_rb) return (int)cudaErrorNotSupported;  // (exchange variants: group2 % 4 == 0)
  const GemvFn fn = a.peers.n ? pick_peer(p.kmax, p.xsm, p.teams == 2 || p.wide)
                              : (p.teams == 2 || p.wide) ? pick_teams(p.kmax) : pick_kernel(p.kmax, p.uniform_rb, p.xsm);
  const uint32_t threads = (p.warps * p.teams + 2) * 32;
  void* params[] = {&a};
  return (int)launch_ex((const void*)fn, dim3(p.grid), dim3(threads), p.smem, (cudaStream_t)stream, pdl, params);
}

int launch_gemv_group(const GemvPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* x,
                      float* const* ys, void* stream, bool pdl, uint32_t flags) {
  const float* xs[kMaxSeg];
  std::fill(xs, xs + kMaxSeg, x);
  return launch_gemv_group(p, layers, n, xs, ys, stream, pdl, flags, nullptr, 1, false);
}

int launch_gemv(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream,
                bool pdl, unsigned long long* dbg, uint32_t repeat, bool global_clock,
                uint32_t flags) {
  const DeviceLayer* layers[1] = {&L};
  for (uint32_t col = 0; col < batch; ++col) {
    float* ys[1] = {y + (size_t)col * L.g.rows};
    const float* xs[1] = {x + (size_t)col * L.g.cols};
    const int e = launch_gemv_group(L.plan, layers, 1, xs, ys, stream, pdl, flags, dbg, repeat, global_clock);
    if (e) return e;
  }
  return 0;
}


}  // namespace qwdev
