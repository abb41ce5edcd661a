// qw_mma.cu -- K2m: the batch-1 quantized GEMV y = W_q x on the warp-level
// tensor cores (mma.sync m16n8k16, fp16 in, fp32 accumulate).
//
// Reference semantics: matvec_oracle (engine.cpp:169-183): per row the
// 1st-order scales from the 2-order pair (row_compute_scales,
// engine.cpp:48-63, 4/3/3 rule quantizer.cpp:103-104), the 2/4-bit codes
// (row_decode, engine.cpp:66-108), w = (c - z) s, y = sum w x' over the
// permuted channels (apply_permutation, plan.cpp:107-116) plus the fp16 CSR
// outliers (sparse_matvec, outliers.cpp:131-141).
//
// Why tensor cores at batch 1.  The SIMT kernel (qw_gemv.cu) spends one
// LOP3 + one HFMA2 per two weights plus the per-(row, group) scale work and
// is issue-bound (~2 instructions per weight in its main loop, ncu r01_v15).
// Here a 16-row x 16-channel group tile is ONE MMA operand: the masked codes
// (LOP3, no conversion: a code masked into an fp16 with a zero exponent
// field reads as c 2^(p-24), exactly) are the A operand, and B is x made
// block-diagonal -- N column n holds the 16 activations of group n and zeros
// elsewhere -- so one m16n8k16 accumulates 8 separate group dot products for
// 16 rows (D[row][group]) and the per-(row, group) 1st-order scales are
// applied once per group in the epilogue.  The zero point rides in a 9th MMA
// (A = z, B = -sum x' split hi + lo over the two K halves).  ~1 instruction
// per weight instead of ~2.
//
// Precision: every product c x' is exact, D is fp32 (the group dot product
// is no longer an fp16 partial sum), s1 = (eff - zero2) scale2 2^-P is
// rounded once to fp16 (as in the SIMT kernel), the scaled terms accumulate
// in fp32.
//
// CTA: 16 consumer warps (warp w owns blocks 2w, 2w+1 of the current chunk:
// their B fragments live in registers), one TMA producer warp streaming
// (tile, chunk) records through a ring of shared-memory slots, one CSR warp.
// A CTA owns a contiguous range of (chunk-major) items; layers wider than one
// chunk combine their chunk partial sums in a fixed order (last arrival).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "qw_device.hpp"
#include "qw_ptx.cuh"

namespace qwdev {

// ------------------------------------------------------------ geometry (host)
void mma_geometry(MmaGeometry& m, const Geometry& g) {
  m = MmaGeometry{};
  if (g.group2 % 16 != 0 || g.rows == 0) return;
  m.RT = (g.rows + 15) / 16;
  m.SB = (g.T2 + 7) / 8;
  m.B4 = (g.T4 + 7) / 8;
  const uint32_t nb2 = 3 * m.SB, nb4 = m.B4, nb = nb2 + nb4;
  if (nb == 0) return;
  // chunks of at most 32 blocks, each an even share of the 2-bit and of the
  // 4-bit blocks (records of similar size and work)
  auto span = [](uint32_t n, uint32_t c, uint32_t k) { return (c + 1) * n / k - c * n / k; };
  uint32_t nc = (nb + kMmaChunkBlk - 1) / kMmaChunkBlk;
  for (;; ++nc) {
    uint32_t mx = 0;
    for (uint32_t c = 0; c < nc; ++c) mx = std::max(mx, span(nb2, c, nc) + span(nb4, c, nc));
    if (mx <= kMmaChunkBlk) break;
  }
  if (nc > kMmaMaxChunks) return;
  m.nchunks = nc;
  uint32_t stride = 0;
  for (uint32_t c = 0; c < nc; ++c) {
    MmaChunk& C = m.chunk[c];
    uint32_t off = 0, k = 0;
    const uint32_t a0 = c * nb2 / nc, a1 = (c + 1) * nb2 / nc;
    for (uint32_t i = a0; i < a1; ++i, ++k) {
      const uint32_t sb = i / 3, b = i % 3;
      if (b == 0 || i == a0) {  // the super-block's header, once per chunk
        C.hdr_off[k] = off;
        off += kMmaHdr2;
      } else {
        C.hdr_off[k] = C.hdr_off[k - 1];
      }
      C.kind[k] = (uint8_t)b, C.grp[k] = (uint16_t)sb;
      C.code_off[k] = off;
      off += kMmaCode2;
    }
    const uint32_t f0 = c * nb4 / nc, f1 = (c + 1) * nb4 / nc;
    for (uint32_t i = f0; i < f1; ++i, ++k) {
      C.kind[k] = 3, C.grp[k] = (uint16_t)i;
      C.code_off[k] = off;
      C.hdr_off[k] = off + kMmaCode4;
      off += kMmaCode4 + kMmaS4 + kMmaZ4;
    }
    C.nblk = k;
    C.rec_bytes = off;
    stride = std::max(stride, off);
  }
  m.rec_stride = (stride + 127) / 128 * 128;
  m.ok = 1;
}

namespace {

constexpr uint32_t kNW = QW_MMA_NW;             // consumer warps
constexpr uint32_t kThreads = (kNW + 2) * 32;   // + producer + CSR warp
constexpr uint32_t kCsrSlotsMax = 16;            // CSR ring: a power of two <= this many tile spans in flight

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ float pow2f(int e) { return __uint_as_float((uint32_t)(e + 127) << 23); }
__device__ __forceinline__ uint32_t h_bits(float v) { return (uint32_t)__half_as_ushort(__float2half_rn(v)); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 h2f2(uint32_t h) { return __half22float2(as_h2(h)); }

// 1st-order scales of rows (g, g+8) for one column: v = the two rows' meta
// fields (row g low half), ac = (a = scale2 2^-P | c = -(2^(10-pe) + zero2)).
// (v & mask) | 0x6400 reads 1024 + eff 2^pe; one HFMA2 leaves eff - zero2
// exactly, one HMUL2 rounds the exact product once (= the fp32 s1 rounded).
__device__ __forceinline__ uint32_t magic6400() {  // in a register: (v & imm) | reg is ONE LOP3
  uint32_t m;
  asm volatile("mov.b32 %0, 0x64006400;" : "=r"(m));
  return m;
}
__device__ __forceinline__ float2 s1_rows(uint32_t v, uint32_t mask, uint32_t p2, uint32_t ac) {
  const half2 e = as_h2((v & mask) | magic6400());
  const half2 d = __hfma2(e, as_h2(p2), __high2half2(as_h2(ac)));
  return __half22float2(__hmul2(d, __low2half2(as_h2(ac))));
}

// One 2-bit block (b = position in its super-block) of one 16-row tile.
template <int B>
__device__ __forceinline__ void body2(const uint8_t* rec, uint32_t code_off, uint32_t hdr_off, uint32_t lane,
                                      const uint32_t (&bf)[8][2], const uint32_t (&bz)[2], float2& acc) {
  const uint4 w = *reinterpret_cast<const uint4*>(rec + code_off + 16u * lane);
  const uint2 M = *reinterpret_cast<const uint2*>(rec + hdr_off + 8u * lane);
  const uint2 AC = *reinterpret_cast<const uint2*>(rec + hdr_off + 256u + 8u * (4u * B + (lane & 3u)));
  const uint4 ws = make_uint4(w.x >> 6, w.y >> 6, w.z >> 6, w.w >> 6);
  // two accumulator chains (even / odd s) halve the dependent HMMA latency
  float d[4] = {0.0f, 0.0f, 0.0f, 0.0f}, e[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint32_t m = 0x00030003u << (s < 5 ? 2 * s : 2 * s - 6);
    const uint4& q = s < 5 ? w : ws;
    mma16816(s & 1 ? e : d, q.x & m, q.y & m, q.z & m, q.w & m, bf[s][0], bf[s][1]);
  }
  // zero points of (row, column 2t) | (row, column 2t+1): z 2^(q-24)
  uint32_t vg, vg8, zm;
  if (B == 0) vg = prmt(M.x, M.x, 0x1010u), vg8 = prmt(M.y, M.y, 0x1010u), zm = 0x000C0003u;
  if (B == 1) vg = M.x, vg8 = M.y, zm = 0x00030030u;
  if (B == 2) vg = prmt(M.x, M.x, 0x3232u), vg8 = prmt(M.y, M.y, 0x3232u), zm = 0x0030000Cu;
  mma16816(e, vg & zm, vg8 & zm, vg & zm, vg8 & zm, bz[0], bz[1]);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] += e[i];
  // 1st-order scales, rows (g, g+8) per column
  const uint32_t m7x = M.x >> 7, m7y = M.y >> 7;
  float2 s0, s1;
  if (B == 0) {
    s0 = s1_rows(prmt(M.x, M.y, 0x5410u), 0x03C003C0u, 0x24002400u, AC.x);  // sub 0: 2^-6
    s1 = s1_rows(prmt(m7x, m7y, 0x5410u), 0x00380038u, 0x34003400u, AC.y);  // sub 1: 2^-2
  } else if (B == 1) {
    s0 = s1_rows(prmt(m7x, m7y, 0x5410u), 0x01C001C0u, 0x28002800u, AC.x);  // sub 2: 2^-5
    s1 = s1_rows(prmt(M.x, M.y, 0x7632u), 0x03C003C0u, 0x24002400u, AC.y);  // sub 0 (next triple)
  } else {
    s0 = s1_rows(prmt(m7x, m7y, 0x7632u), 0x00380038u, 0x34003400u, AC.x);  // sub 1
    s1 = s1_rows(prmt(m7x, m7y, 0x7632u), 0x01C001C0u, 0x28002800u, AC.y);  // sub 2
  }
  acc = ffma2(s0, make_float2(d[0], d[2]), acc);
  acc = ffma2(s1, make_float2(d[1], d[3]), acc);
}

// One 4-bit block of one 16-row tile.
__device__ __forceinline__ void body4(const uint8_t* rec, uint32_t code_off, uint32_t hdr_off, uint32_t lane,
                                      const uint32_t (&bf)[8][2], const uint32_t (&bz)[2], float2& ag,
                                      float2& ag8) {
  const uint4 w0 = *reinterpret_cast<const uint4*>(rec + code_off + 32u * lane);
  const uint4 w1 = *reinterpret_cast<const uint4*>(rec + code_off + 32u * lane + 16u);
  const uint2 S = *reinterpret_cast<const uint2*>(rec + hdr_off + 8u * lane);
  const uint32_t z16 = *reinterpret_cast<const uint16_t*>(rec + hdr_off + kMmaS4 + 2u * lane);
  float d[4] = {0.0f, 0.0f, 0.0f, 0.0f}, e[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint4& q = h ? w1 : w0;
    const uint4 qs = make_uint4(q.x >> 8, q.y >> 8, q.z >> 8, q.w >> 8);
    mma16816(d, q.x & 0x000F000Fu, q.y & 0x000F000Fu, q.z & 0x000F000Fu, q.w & 0x000F000Fu, bf[4 * h][0],
             bf[4 * h][1]);
    mma16816(e, q.x & 0x00F000F0u, q.y & 0x00F000F0u, q.z & 0x00F000F0u, q.w & 0x00F000F0u, bf[4 * h + 1][0],
             bf[4 * h + 1][1]);
    mma16816(d, qs.x & 0x000F000Fu, qs.y & 0x000F000Fu, qs.z & 0x000F000Fu, qs.w & 0x000F000Fu,
             bf[4 * h + 2][0], bf[4 * h + 2][1]);
    mma16816(e, qs.x & 0x00F000F0u, qs.y & 0x00F000F0u, qs.z & 0x00F000F0u, qs.w & 0x00F000F0u,
             bf[4 * h + 3][0], bf[4 * h + 3][1]);
  }
  const uint32_t Z = prmt(z16, 0u, 0x4140u);
  const uint32_t zg = Z & 0x000F000Fu, zg8 = (Z >> 4) & 0x000F000Fu;
  mma16816(e, zg, zg8, zg, zg8, bz[0], bz[1]);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] += e[i];
  ag = ffma2(h2f2(S.x), make_float2(d[0], d[1]), ag);
  ag8 = ffma2(h2f2(S.y), make_float2(d[2], d[3]), ag8);
}

struct MmaRing {
  const uint8_t* smem;
  uint64_t* full;
  uint64_t* empty;
  float* part;  // [item][16 rows][kNW]
  uint32_t stride, S, slot, phase;
};

template <int K>
__device__ __forceinline__ void body(const uint8_t* rec, uint32_t coff, uint32_t hoff, uint32_t lane,
                                     const uint32_t (&bf)[8][2], const uint32_t (&bz)[2], float2& acc2, float2& ag,
                                     float2& ag8) {
  if constexpr (K < 3) body2<K>(rec, coff, hoff, lane, bf, bz, acc2);
  else if constexpr (K == 3) body4(rec, coff, hoff, lane, bf, bz, ag, ag8);
}

// Items [k, kend) of one chunk for a warp whose two blocks have kinds K0, K1
// (4 = no block): decode + MMA + epilogue, hand the slot back, row sums of
// the warp into the item's partial slots.
// NI consecutive items (1 or 2: two items' bodies interleave, twice the
// independent MMA chains per warp) for a warp whose blocks have kinds K0, K1.
template <int K0, int K1, int NI>
__device__ __forceinline__ void step_items(MmaRing& r, uint32_t k, uint32_t lane, uint32_t warp,
                                           const uint32_t (&coff)[2], const uint32_t (&hoff)[2],
                                           const uint32_t (&bf)[2][8][2], const uint32_t (&bz)[2][2], float2 ys,
                                           uint32_t diag) {
  const uint32_t g = lane >> 2, t = lane & 3u;
  uint32_t slot[NI];
  const uint8_t* rec[NI];
  float2 acc2[NI], ag[NI], ag8[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    slot[i] = r.slot;
    const uint32_t ph = r.phase;
    if (++r.slot == r.S) r.slot = 0, r.phase ^= 1u;
    if (!(diag & 1) || k + i < r.S) mbar_wait(&r.full[slot[i]], (diag & 1) ? 0u : ph);
    rec[i] = r.smem + (size_t)slot[i] * r.stride;
    acc2[i] = ag[i] = ag8[i] = make_float2(0.0f, 0.0f);
  }
  if (!(diag & 2)) {
#pragma unroll
    for (int i = 0; i < NI; ++i) body<K0>(rec[i], coff[0], hoff[0], lane, bf[0], bz[0], acc2[i], ag[i], ag8[i]);
#pragma unroll
    for (int i = 0; i < NI; ++i) body<K1>(rec[i], coff[1], hoff[1], lane, bf[1], bz[1], acc2[i], ag[i], ag8[i]);
  }
  __syncwarp();
  if (lane == 0 && !(diag & 1))
#pragma unroll
    for (int i = 0; i < NI; ++i) mbar_arrive(&r.empty[slot[i]]);
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    float yg = acc2[i].x * ys.x, yg8 = acc2[i].y * ys.x;
    if constexpr (K0 == 3 || K1 == 3) yg += (ag[i].x + ag[i].y) * ys.y, yg8 += (ag8[i].x + ag8[i].y) * ys.y;
    yg += __shfl_xor_sync(0xFFFFFFFFu, yg, 1);
    yg8 += __shfl_xor_sync(0xFFFFFFFFu, yg8, 1);
    yg += __shfl_xor_sync(0xFFFFFFFFu, yg, 2);
    yg8 += __shfl_xor_sync(0xFFFFFFFFu, yg8, 2);
    if (t == 0) {
      r.part[((k + i) * 16 + g) * kNW + warp] = yg;
      r.part[((k + i) * 16 + g + 8) * kNW + warp] = yg8;
    }
  }
}

template <int K0, int K1>
__device__ __forceinline__ void run_items(MmaRing& r, uint32_t k, uint32_t kend, uint32_t lane, uint32_t warp,
                                          const uint32_t (&coff)[2], const uint32_t (&hoff)[2],
                                          const uint32_t (&bf)[2][8][2], const uint32_t (&bz)[2][2], float2 ys,
                                          uint32_t diag) {
  // (two items interleaved per step were measured slower: 96-register cap of 18 warps, spills)
  for (; k < kend; ++k) step_items<K0, K1, 1>(r, k, lane, warp, coff, hoff, bf, bz, ys, diag);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Shared-memory layout of a K2m CTA (fixed per plan; a chain plan takes the
// maximum over its steps).
struct MmaLayout {
  uint32_t S, rec_stride, x_off, part_off, csr_off, ent_off, csr_slot, csr_nslot, rp_off, bst_off, bar_off,
      items_cap, diag, x_gate;
};

// One step (a layer group sharing x) as one CTA sees it.
struct StepView {
  const uint8_t* recs;
  const uint16_t* perm16;
  const uint32_t* row_ptr;
  const uint32_t* csr;
  float* y;
  float* part;
  uint32_t* cnt;
  uint32_t rows, RT;
  float inv_s_scale;  // 2^P: 2-bit s1 carries 2^-P
  const float* x;
  uint32_t cols, n2p, G2, T4, nchunks;
  const MmaChunk* chunk;
  uint32_t i0, i1;
  uint32_t hbm_stride;  // the layer's record stride in HBM (the ring slot stride may be larger)
};

// Per-launch kernel arguments (a single layer or a group launch).
struct MmaArgs {
  const uint8_t* recs[kMaxSeg];
  const uint16_t* perm16[kMaxSeg];
  const uint32_t* row_ptr[kMaxSeg];
  const uint32_t* csr[kMaxSeg];
  float* y[kMaxSeg];
  float* part[kMaxSeg];
  uint32_t* cnt[kMaxSeg];
  uint32_t rows[kMaxSeg], RT[kMaxSeg];
  float inv_s_scale[kMaxSeg];
  const float* xs[kMaxSeg];
  uint32_t cols, n2p, G2, T4, nchunks, wait_x;
  MmaLayout lay;
  MmaChunk chunk[kMmaMaxChunks];
  uint8_t cta_seg[kMaxGrid];
  uint32_t cta_i0[kMaxGrid], cta_i1[kMaxGrid];
  unsigned long long* dbg;  // diagnostics: [grid][kTimelineEvents] %globaltimer stamps (or null)
};

// Persistent decode chain: per step (global memory) ...
struct MmaStepDesc {
  const uint8_t* recs[kMaxSeg];
  const uint16_t* perm16[kMaxSeg];
  const uint32_t* row_ptr[kMaxSeg];
  const uint32_t* csr[kMaxSeg];
  float* y[kMaxSeg];
  float* part[kMaxSeg];
  uint32_t* cnt[kMaxSeg];
  uint32_t rows[kMaxSeg], RT[kMaxSeg];
  float inv_s_scale[kMaxSeg];
  const float* x;
  uint32_t cols, n2p, G2, T4, nchunks, depends, hbm_stride, pad;
  MmaChunk chunk[kMmaMaxChunks];
};
struct MmaCtaRange {  // ... and per (step, CTA)
  uint32_t seg, i0, i1, pad;
};
struct MmaProdStep {  // the producer's view of (step, CTA)
  uint64_t recs;
  uint32_t i0, i1, RT, hbm_stride;
  uint32_t rec_bytes[kMmaMaxChunks];
  uint32_t pad[2];
};
struct MmaChainArgs {
  const MmaStepDesc* steps;
  const MmaCtaRange* ranges;  // [step][grid]
  const MmaProdStep* prod;    // [step][grid]
  uint32_t* done;             // [step] CTAs that finished the step (zeroed before each run)
  unsigned long long* tl;     // diagnostics (QW_DEBUG_MMA_TL): [step][cta][8] %globaltimer stamps
  uint32_t nsteps, grid;
  MmaLayout lay;
};

// Role code of one step.  Ring (producer / consumers) and CSR-ring counters
// persist across steps in the chain kernel.
struct MmaState {
  uint32_t slot, phase;  // weight ring position (producer and consumers each keep their own copy)
  uint32_t q;            // CSR ring position (CSR warp)
};

__device__ __forceinline__ void producer_step(const StepView& v, const MmaLayout& L, uint8_t* smem, uint64_t* full,
                                              uint64_t* empty, MmaState& st, uint32_t& issued,
                                              uint64_t* xbar = nullptr, uint32_t x_gate = 0) {
  const uint32_t nitems = v.i1 - v.i0;
  if (!nitems) return;
  const uint32_t RT = v.RT;
  uint32_t ch = v.i0 / RT, left = RT - (v.i0 - ch * RT);
  const uint32_t n = (L.diag & 1) ? min(nitems, L.S) : nitems;
  for (uint32_t k = 0; k < n; ++k) {
    const uint32_t bytes = v.chunk[ch].rec_bytes;
    // hold the stream after x_gate records until x is staged: the x loads
    // then meet a quieter memory system (they sit on the critical path)
    if (xbar && k == x_gate) mbar_wait(xbar, 0);
    if (issued >= L.S) mbar_wait_spin(&empty[st.slot], st.phase ^ 1u);  // no suspend: refill at once
    mbar_expect_tx(&full[st.slot], bytes);
    bulk_load_nohint(smem + (size_t)st.slot * L.rec_stride, v.recs + (size_t)(v.i0 + k) * v.hbm_stride, bytes,
                     &full[st.slot]);
    ++issued;
    if (++st.slot == L.S) st.slot = 0, st.phase ^= 1u;
    if (--left == 0) ++ch, left = RT;
  }
}

// Outliers: exact fp32 products (outliers.cpp:131-141).  Tile t's outliers are
// summed by the CTA that holds item (chunk t % nch, t) -- spread over the
// CTAs.  The warp stages the row_ptr words of its tiles, streams each tile's
// entry span into a ring of its own (bulk copies of 16-byte aligned spans; a
// span beyond the slot reads the rest from global memory), and sums a row in
// two halves (lanes l and l + 16), 4 entries in flight per step, halves
// joined in a fixed order.
// CSR item q of a step (ring position q0 + q): the tile's entry span -> its slot
__device__ __forceinline__ void csr_issue(const StepView& v, const MmaLayout& L, uint8_t* smem, uint64_t* cbar,
                                          uint32_t q0, uint32_t q) {
  const uint32_t* s_rp = reinterpret_cast<const uint32_t*>(smem + L.rp_off);
  const uint32_t sl = (q0 + q) & (L.csr_nslot - 1);
  const uint32_t lo = s_rp[q * 17] & ~3u, hi = s_rp[q * 17 + 16];
  const uint32_t bytes = min(((hi - lo) * 4u + 15u) & ~15u, L.csr_slot);
  if (bytes) {
    mbar_expect_tx(&cbar[sl], bytes);
    bulk_load_nohint(smem + L.ent_off + (size_t)sl * L.csr_slot, v.csr + lo, bytes, &cbar[sl]);
  } else {
    mbar_arrive(&cbar[sl]);
  }
}

__device__ __forceinline__ void csr_prepare(const StepView& v, const MmaLayout& L, uint8_t* smem, uint64_t* cbar,
                                            const MmaState& st, uint32_t lane, uint32_t& nq) {
  const uint32_t nitems = v.i1 - v.i0, RT = v.RT, rows = v.rows, nch = v.nchunks;
  const uint32_t* __restrict__ rp = v.row_ptr;
  uint32_t* s_rp = reinterpret_cast<uint32_t*>(smem + L.rp_off);      // [q][17]
  uint16_t* s_qk = reinterpret_cast<uint16_t*>(s_rp + L.items_cap * 17);  // item of CSR item q
  nq = 0;
  if (!(L.diag & 4) && nitems) {
    // the CSR items (tiles this CTA sums) first, then their row_ptr words
    // with 8 loads in flight per lane (one load per item in a dependent
    // sequence cost a memory latency per item: 7 us for 9 items)
    uint32_t ch = v.i0 / RT, tile = v.i0 - ch * RT;
    for (uint32_t k = 0; k < nitems; ++k) {
      if (tile % nch == ch) {
        if (lane == 0) s_qk[nq] = (uint16_t)k;
        ++nq;
      }
      if (++tile == RT) tile = 0, ++ch;
    }
    __syncwarp();
    const uint32_t nw = nq * 17;
    for (uint32_t base = 0; base < nw; base += 8 * 32) {
      uint32_t w[8];
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) {
        const uint32_t f = base + u * 32 + lane;
        if (f < nw) {
          const uint32_t q = f / 17, j = f - q * 17, t = (v.i0 + s_qk[q]) % RT;
          w[u] = __ldg(rp + min(t * 16 + j, rows));
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u)
        if (base + u * 32 + lane < nw) s_rp[base + u * 32 + lane] = w[u];
    }
  }
  __syncwarp();
  if (lane == 0)
    for (uint32_t q = 0; q < min(nq, L.csr_nslot); ++q) csr_issue(v, L, smem, cbar, st.q, q);
}

// Outliers: exact fp32 products (outliers.cpp:131-141).  Tile t's outliers are
// summed by the CTA that holds item (chunk t % nch, t) -- spread over the
// CTAs.  csr_prepare stages the row_ptr words of the warp's tiles and starts
// streaming each tile's entry span into a ring of its own (bulk copies of
// 16-byte aligned spans; a span beyond the slot reads the rest from global
// memory); here a row is summed in two halves (lanes l and l + 16), 4
// entries in flight per step, halves joined in a fixed order.
__device__ __forceinline__ void csr_compute(const StepView& v, const MmaLayout& L, uint8_t* smem, uint64_t* xbar,
                                            uint32_t xphase, uint64_t* cbar, float* s_x, float* s_csr,
                                            MmaState& st, uint32_t lane, uint32_t nq) {
  const uint32_t* __restrict__ ent = v.csr;
  const uint32_t* s_rp = reinterpret_cast<const uint32_t*>(smem + L.rp_off);
  const uint16_t* s_qk = reinterpret_cast<const uint16_t*>(s_rp + L.items_cap * 17);
  const uint32_t CS = L.csr_nslot, cmask = CS - 1, csh = __ffs(CS) - 1, q0 = st.q;
  mbar_wait(xbar, xphase);
  const uint32_t r = lane & 15u, half = lane >> 4, nst = L.csr_slot / 4;
  for (uint32_t q = 0; q < nq; ++q) {
    const uint32_t qq = q0 + q, sl = qq & cmask;
    mbar_wait(&cbar[sl], (qq >> csh) & 1u);
    const uint32_t* s_ent = reinterpret_cast<const uint32_t*>(smem + L.ent_off + (size_t)sl * L.csr_slot);
    const uint32_t e_base = s_rp[q * 17] & ~3u;
    const uint32_t lo0 = s_rp[q * 17 + r] - e_base, hi0 = s_rp[q * 17 + r + 1] - e_base;
    const uint32_t mid = lo0 + (hi0 - lo0) / 2;
    uint32_t e = half ? mid : lo0;
    const uint32_t end = half ? hi0 : mid;
    float acc = 0.0f;
    for (; e + 4 <= end; e += 4) {
      uint32_t w[4];
      float xv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = e + j < nst ? s_ent[e + j] : __ldg(ent + e_base + e + j);
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = s_x[w[j] & 0xFFFFu];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc = __fadd_rn(acc, __fmul_rn(half_bits_to_float(w[j] >> 16), xv[j]));
    }
    for (; e < end; ++e) {
      const uint32_t w = e < nst ? s_ent[e] : __ldg(ent + e_base + e);
      acc = __fadd_rn(acc, __fmul_rn(half_bits_to_float(w >> 16), s_x[w & 0xFFFFu]));
    }
    const float other = __shfl_down_sync(0xFFFFFFFFu, acc, 16);
    if (lane < 16) s_csr[(uint32_t)s_qk[q] * 16 + r] = acc + other;  // first half, then second
    __syncwarp();
    if (lane == 0 && q + CS < nq) csr_issue(v, L, smem, cbar, q0, q + CS);
  }
  st.q = q0 + nq;
}

// A consumer warp's two blocks of one chunk and the lane's perm entries.
struct WarpBlocks {
  uint32_t kind[2], coff[2], hoff[2];
  uint2 pq[2];  // perm16 of the lane's 4 channels of each block
};
// the chunk's block descriptors + the lane's perm entries (x-independent)
__device__ __forceinline__ void fetch_blocks(WarpBlocks& wb, const StepView& v, uint32_t ch, uint32_t warp,
                                             uint32_t lane) {
  const uint32_t bn = lane >> 2, bq = lane & 3u;
  const MmaChunk& C = v.chunk[ch];
  const uint32_t nblk = C.nblk;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint32_t blk = 2 * warp + j;
    wb.kind[j] = blk < nblk ? C.kind[blk] : 4u;  // 4: no block
    wb.coff[j] = blk < nblk ? C.code_off[blk] : 0u;
    wb.hoff[j] = blk < nblk ? C.hdr_off[blk] : 0u;
    const uint32_t grp = blk < nblk ? C.grp[blk] : 0u;
    bool valid = wb.kind[j] < 4;
    uint32_t base = 0;
    if (wb.kind[j] < 3) {
      const uint32_t jg = 24u * grp + 6u * (bn >> 1) + 2u * wb.kind[j] + (bn & 1u);
      valid = valid && jg < v.G2;
      base = 16u * jg;
    } else {
      const uint32_t b4 = 8u * grp + bn;
      valid = valid && b4 < v.T4;
      base = v.n2p + 16u * b4;
    }
    // invalid columns gather the zero slot x[cols]
    wb.pq[j] = valid ? __ldg(reinterpret_cast<const uint2*>(v.perm16 + base + 4 * bq))
                     : make_uint2(v.cols | (v.cols << 16), v.cols | (v.cols << 16));
  }
}

// Consumers of one step: x staging (after the caller resolved the
// dependency), per chunk the B fragments of the warp's two blocks and the
// item loop, then (after meeting the CSR warp) the fixed-order row sums ->
// y, or chunk partials + last-arrival combine.  `prefetched`: wb already
// holds the first chunk's blocks (fetched during the previous step); `next`:
// fetch the next step's first chunk under this step's tail.
__device__ __forceinline__ void consumer_step(const StepView& v, const MmaLayout& L, uint8_t* smem, uint64_t* full,
                                              uint64_t* empty, uint64_t* xbar, uint32_t xphase, float* s_x,
                                              float* s_part, float* s_csr, MmaState& st, uint32_t warp,
                                              uint32_t lane, bool wait_pdl, WarpBlocks& wb, bool prefetched,
                                              const StepView* next, unsigned long long* tl = nullptr,
                                              bool per_launch = false) {
  const uint32_t g = lane >> 2, t = lane & 3u;
  const bool nz = t == (g >> 1);  // this lane holds column g of the block-diagonal B
  // B staging (cooperative build): lane (n = lane / 4, quarter c = lane % 4)
  // prepares channels 4c .. 4c+3 of column n of each of the warp's blocks
  const uint32_t bn = lane >> 2, bq = lane & 3u;
  uint32_t* s_bst = reinterpret_cast<uint32_t*>(smem + L.bst_off) + warp * (2 * 8 * 20);
  const uint32_t* s_bzero = reinterpret_cast<const uint32_t*>(smem + L.bst_off) + kNW * (2 * 8 * 20);
  const uint32_t nitems = v.i1 - v.i0, RT = v.RT;
  uint32_t* kind = wb.kind;
  uint2* pq = wb.pq;
  auto fetch_perm = [&](uint32_t ch) { fetch_blocks(wb, v, ch, warp, lane); };
  if (nitems && !prefetched) fetch_perm(v.i0 / RT);
  // x -> shared memory (coalesced), the pads' zero slot at cols
  if (wait_pdl) pdl_wait();
  if (per_launch && tl && threadIdx.x == 0) tl[10] = gtimer();  // dependency resolved
  {
    const uint32_t tid = threadIdx.x, nth = kNW * 32, cols = v.cols;
    if ((((uintptr_t)v.x) & 15u) == 0 && (cols & 3u) == 0) {
      const float4* gx = reinterpret_cast<const float4*>(v.x);
      float4* sx4 = reinterpret_cast<float4*>(s_x);
      for (uint32_t i = tid; i < cols / 4; i += nth) sx4[i] = __ldcg(gx + i);
    } else {
      for (uint32_t i = tid; i < cols; i += nth) s_x[i] = __ldcg(v.x + i);
    }
    if (tid == 0) s_x[cols] = 0.0f;
    __syncwarp();
    if (lane == 0) mbar_arrive(xbar);
  }
  mbar_wait(xbar, xphase);
  if (tl && threadIdx.x == 0) tl[1] = gtimer();  // x staged

  uint32_t bf[2][8][2], bz[2][2];
  float ys2 = 0.0f, ys4 = 0.0f;
  // B fragments of the warp's two blocks (block-diagonal x): every lane
  // scales 4 channels, the 8 lanes that hold a column read its 18 words back
  auto build_b = [&]() {
    float xv[2][4];
    float mx = 0.0f;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t w = c < 2 ? pq[j].x : pq[j].y;
        xv[j][c] = s_x[(w >> (16 * (c & 1))) & 0xFFFFu];
        mx = fmaxf(mx, fabsf(xv[j][c]));
      }
    // one power-of-two scale per warp: max|x'| in [2^10, 2^11)
    const uint32_t mxb = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
    const int eb = (int)(mxb >> 23);
    const int sh = (eb == 0 ? -126 : eb - 127) - 10;
    const int e = -sh, e1 = max(-126, min(127, e));
    const float f1 = pow2f(e1), f2 = pow2f(max(-126, min(127, e - e1)));
    const float yb = pow2f(max(-126, min(127, sh + 24)));
    ys2 = yb * v.inv_s_scale, ys4 = yb;
    const uint32_t hs = 16u * (bn & 1u);  // the half of column bn
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const bool two = kind[j] < 3;
      float sx = 0.0f;
      uint32_t w4[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float xs = (xv[j][c] * f1) * f2;
        sx += xs;
        const int s = 2 * (int)bq + (c >> 1);  // channel 4 bq + c = 2 s + (c & 1)
        const int p = two ? (s < 5 ? 2 * s : 2 * s - 6) : 4 * (s & 1);
        w4[c] = h_bits(xs * pow2f(-p)) << hs;
      }
      // fragment words of column bn: [s][e] at 2 s + e, s = 2 bq .. 2 bq + 1
      *reinterpret_cast<uint4*>(s_bst + (j * 8 + bn) * 20 + 4 * bq) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      sx += __shfl_xor_sync(0xFFFFFFFFu, sx, 1);
      sx += __shfl_xor_sync(0xFFFFFFFFu, sx, 2);
      if (bq == 0) {
        // zero point: -sum x' as hi + lo fp16, scaled by 2^-q of the z field
        const float hi = __half2float(__float2half_rn(sx));
        const float lo = sx - hi;
        int q = 0;
        if (kind[j] == 0) q = (bn & 1u) ? 2 : 0;
        if (kind[j] == 1) q = (bn & 1u) ? 0 : 4;
        if (kind[j] == 2) q = (bn & 1u) ? 4 : 2;
        *reinterpret_cast<uint2*>(s_bst + (j * 8 + bn) * 20 + 16) =
            make_uint2(h_bits(-hi * pow2f(-q)) << hs, h_bits(-lo * pow2f(-q)) << hs);
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t* src = nz ? s_bst + (j * 8 + g) * 20 : s_bzero;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const uint4 u = *reinterpret_cast<const uint4*>(src + 4 * q4);
        bf[j][2 * q4][0] = u.x, bf[j][2 * q4][1] = u.y, bf[j][2 * q4 + 1][0] = u.z, bf[j][2 * q4 + 1][1] = u.w;
      }
      const uint2 z = *reinterpret_cast<const uint2*>(src + 16);
      bz[j][0] = z.x, bz[j][1] = z.y;
    }
    __syncwarp();
  };

  MmaRing ring{smem, full, empty, s_part, L.rec_stride, L.S, st.slot, st.phase};
  uint32_t ch = nitems ? v.i0 / RT : 0u, k = 0;
  while (k < nitems) {
    build_b();
    if (per_launch && tl && threadIdx.x == 0 && k == 0) tl[11] = gtimer();  // first B built
    // the items of this chunk, one warp-role specialised loop (no per-item dispatch)
    const uint32_t kend = min(nitems, k + (RT - (v.i0 + k - ch * RT)));
    const float2 ys = make_float2(ys2, ys4);
    switch (kind[0] * 5 + kind[1]) {
#define QW_CASE(K0, K1) \
  case K0 * 5 + K1: run_items<K0, K1>(ring, k, kend, lane, warp, wb.coff, wb.hoff, bf, bz, ys, L.diag); break;
      QW_CASE(0, 1) QW_CASE(1, 2) QW_CASE(2, 0) QW_CASE(0, 3) QW_CASE(1, 3) QW_CASE(2, 3) QW_CASE(3, 3)
      QW_CASE(0, 4) QW_CASE(1, 4) QW_CASE(2, 4) QW_CASE(3, 4) QW_CASE(4, 4)
      QW_CASE(0, 0) QW_CASE(1, 1) QW_CASE(2, 2) QW_CASE(0, 2) QW_CASE(1, 0) QW_CASE(2, 1)
      QW_CASE(3, 0) QW_CASE(3, 1) QW_CASE(3, 2) QW_CASE(4, 0) QW_CASE(4, 1) QW_CASE(4, 2) QW_CASE(4, 3)
#undef QW_CASE
      default: break;
    }
    k = kend;
    if (k < nitems) fetch_perm(++ch);
  }
  st.slot = ring.slot, st.phase = ring.phase;
  if (tl && threadIdx.x == 0) tl[2] = gtimer();  // items done (warp 0)
  named_sync(1, (kNW + 1) * 32);  // consumers' partials and the CSR sums
  if (tl && threadIdx.x == 0) tl[3] = gtimer();  // every warp + CSR done
  // the next step's first chunk (x-independent): its loads fly under the
  // reduction, the step barrier and the dependency wait
  if (next && next->i1 > next->i0) fetch_blocks(wb, *next, next->i0 / next->RT, warp, lane);
  // dense sum in a fixed warp order, then the outliers (row_fma, engine.cpp:111-122)
  const uint32_t tid = threadIdx.x, nch = v.nchunks, rows = v.rows;
  float* __restrict__ gy = v.y;
  for (uint32_t idx = tid; idx < nitems * 16; idx += kNW * 32) {
    const uint32_t kk = idx >> 4, r = idx & 15u, it = v.i0 + kk, c = it / RT, tile = it - c * RT;
    const float* p = s_part + (size_t)idx * kNW;
    float s = p[0];
#pragma unroll
    for (uint32_t w = 1; w < kNW; ++w) s += p[w];
    const uint32_t row = tile * 16 + r;
    if (nch == 1) {
      if (row < rows) gy[row] = s + s_csr[idx];
    } else {
      if (!wait_pdl) pdl_wait();  // the layer's scratch: never under a still-running predecessor
      v.part[(size_t)c * RT * 16 + row] = s;
      if (c == tile % nch) v.part[(size_t)nch * RT * 16 + row] = s_csr[idx];
    }
  }
  if (per_launch && tl && threadIdx.x == 0) tl[9] = gtimer();  // dense sums stored (thread 0)
  if (nch == 1 || (L.diag & 8)) return;
  // chunk partials meet: the last arriving CTA of a tile sums them in chunk
  // order (CTA barrier, then lane 0's acq_rel atomic: cumulative release of
  // the CTA's partial writes, acquire of the other CTAs')
  named_sync(3, kNW * 32);
  // one warp per item: lane 0 counts the arrival, 16 lanes sum a row each
  for (uint32_t kk = warp; kk < nitems; kk += kNW) {
    const uint32_t it = v.i0 + kk, tile = it % RT;
    uint32_t old = 0;
    if (lane == 0) asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(v.cnt + tile) : "memory");
    old = __shfl_sync(0xFFFFFFFFu, old, 0);
    if (old == nch - 1) {
      __syncwarp();
      const float* __restrict__ part = v.part;
      const uint32_t row = tile * 16 + (lane & 15u);
      if (lane < 16 && row < rows) {
        const float csr = __ldcg(part + (size_t)nch * RT * 16 + row);
        float s = __ldcg(part + row);
        for (uint32_t c = 1; c < nch; ++c) s += __ldcg(part + (size_t)c * RT * 16 + row);
        gy[row] = s + csr;  // chunk order, then the outliers
      }
      if (lane == 0) v.cnt[tile] = 0;
    }
  }
}

__device__ __forceinline__ uint8_t* aligned_smem(uint8_t* raw) {
  return raw + ((128u - (smem_addr(raw) & 127u)) & 127u);
}
__device__ __forceinline__ void init_barriers(uint64_t* bars, uint32_t S) {
  // [0, S) full, [S, 2S) empty, 2S x staged, 2S+1 .. 2S+kCsrSlotsMax CSR ring
  if (threadIdx.x < S) mbar_init(&bars[threadIdx.x], 1), mbar_init(&bars[S + threadIdx.x], kNW);
  if (threadIdx.x == 32) mbar_init(&bars[2 * S], kNW);
  if (threadIdx.x >= 64 && threadIdx.x < 64 + kCsrSlotsMax) mbar_init(&bars[2 * S + 1 + (threadIdx.x - 64)], 1);
}

__global__ void __launch_bounds__(kThreads, kNW <= 8 ? 2 : 1) mma_gemv_kernel(const __grid_constant__ MmaArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  const MmaLayout& L = a.lay;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t seg = a.cta_seg[blockIdx.x];
  StepView v{a.recs[seg], a.perm16[seg], a.row_ptr[seg], a.csr[seg], a.y[seg], a.part[seg], a.cnt[seg],
             a.rows[seg], a.RT[seg], a.inv_s_scale[seg], a.xs[seg], a.cols, a.n2p, a.G2, a.T4, a.nchunks, a.chunk,
             a.cta_i0[blockIdx.x], a.cta_i1[blockIdx.x], L.rec_stride};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  unsigned long long* tl = a.dbg ? a.dbg + (size_t)blockIdx.x * kTimelineEvents : nullptr;
  if (tl && threadIdx.x == 0) tl[0] = gtimer();  // entry
  if (threadIdx.x < 20) reinterpret_cast<uint32_t*>(smem + L.bst_off)[kNW * 2 * 8 * 20 + threadIdx.x] = 0u;
  init_barriers(bars, L.S);
  mbar_fence_init();
  __syncthreads();
  pdl_launch_dependents();
  MmaState st{0u, 0u, 0u};
  float* s_x = reinterpret_cast<float*>(smem + L.x_off);
  float* s_csr = reinterpret_cast<float*>(smem + L.csr_off);
  if (warp == kNW) {  // producer: the weight stream never waits on x
    uint32_t issued = 0;
    if (lane == 0) producer_step(v, L, smem, bars, bars + L.S, st, issued, L.x_gate ? bars + 2 * L.S : nullptr, L.x_gate);
    if (tl && lane == 0) tl[7] = gtimer();  // every copy issued
    return;
  }
  if (warp == kNW + 1) {
    uint32_t nq = 0;
    csr_prepare(v, L, smem, bars + 2 * L.S + 1, st, lane, nq);
    if (tl && lane == 0) tl[8] = gtimer();  // CSR spans requested
    csr_compute(v, L, smem, bars + 2 * L.S, 0u, bars + 2 * L.S + 1, s_x, s_csr, st, lane, nq);
    if (tl && lane == 0) tl[6] = gtimer();  // outlier sums done
    named_sync(1, (kNW + 1) * 32);
    return;
  }
  WarpBlocks wb;
  consumer_step(v, L, smem, bars, bars + L.S, bars + 2 * L.S, 0u, s_x, reinterpret_cast<float*>(smem + L.part_off),
                s_csr, st, warp, lane, a.wait_x != 0, wb, false, nullptr, tl, true);
  if (tl && threadIdx.x == 0) tl[5] = gtimer();  // y / partials stored, fixup done (thread 0)
}

// The whole decode step as ONE persistent kernel (one CTA per SM): the
// producer streams the records of every step through one ring that spans the
// steps (step s+1's weights land while step s computes); a step whose x is
// the previous step's y waits on a grid-wide completion counter.  Every
// x-independent load of step s+1 (its view, the warps' block descriptors and
// perm entries, the CSR row pointers and entry spans) is issued during step
// s, so a step boundary costs the counter wait, the x staging and the B build.
__global__ void __launch_bounds__(kThreads, 1) mma_chain_kernel(const __grid_constant__ MmaChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  const MmaLayout& L = a.lay;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  StepView* s_view = reinterpret_cast<StepView*>(smem + L.bar_off + ((2 * L.S + 1 + kCsrSlotsMax) * 8 + 15) / 16 * 16);
  auto load_view = [&](uint32_t s, StepView& out) {
    const MmaStepDesc& d = a.steps[s];
    const MmaCtaRange r = a.ranges[(size_t)s * a.grid + blockIdx.x];
    const uint32_t seg = r.seg;
    out = StepView{d.recs[seg], d.perm16[seg], d.row_ptr[seg], d.csr[seg], d.y[seg], d.part[seg], d.cnt[seg],
                   d.rows[seg], d.RT[seg], d.inv_s_scale[seg], d.x, d.cols, d.n2p, d.G2, d.T4, d.nchunks,
                   d.chunk, r.i0, r.i1, d.hbm_stride};
  };
  if (threadIdx.x < 20) reinterpret_cast<uint32_t*>(smem + L.bst_off)[kNW * 2 * 8 * 20 + threadIdx.x] = 0u;
  if (threadIdx.x == 0) load_view(0, s_view[0]);
  init_barriers(bars, L.S);
  mbar_fence_init();
  __syncthreads();
  MmaState st{0u, 0u, 0u};
  float* s_x = reinterpret_cast<float*>(smem + L.x_off);
  float* s_csr = reinterpret_cast<float*>(smem + L.csr_off);
  float* s_part = reinterpret_cast<float*>(smem + L.part_off);
  if (warp == kNW) {
    // producer: lane j keeps the records of step base + j in registers
    // (prefetched 32 steps at a time); lane 0 issues every copy
    uint32_t issued = 0, slot = 0, phase = 0;
    for (uint32_t base = 0; base < a.nsteps; base += 32) {
      MmaProdStep mine{};
      if (base + lane < a.nsteps) mine = a.prod[(size_t)(base + lane) * a.grid + blockIdx.x];
      for (uint32_t s = base; s < min(base + 32, a.nsteps); ++s) {
        const uint32_t src = s - base;
        const uint32_t i0 = __shfl_sync(0xFFFFFFFFu, mine.i0, src), i1 = __shfl_sync(0xFFFFFFFFu, mine.i1, src);
        const uint32_t RT = __shfl_sync(0xFFFFFFFFu, mine.RT, src);
        const uint32_t stride = __shfl_sync(0xFFFFFFFFu, mine.hbm_stride, src);
        const uint64_t recs = __shfl_sync(0xFFFFFFFFu, mine.recs, src);
        uint32_t rb[kMmaMaxChunks];
#pragma unroll
        for (uint32_t c = 0; c < kMmaMaxChunks; ++c) rb[c] = __shfl_sync(0xFFFFFFFFu, mine.rec_bytes[c], src);
        if (lane == 0 && i1 > i0) {
          uint32_t ch = i0 / RT, left = RT - (i0 - ch * RT);
          const uint32_t n = (L.diag & 1) ? min(i1 - i0, L.S) : i1 - i0;
          for (uint32_t k = 0; k < n; ++k) {
            uint32_t bytes = rb[0];
#pragma unroll
            for (uint32_t c = 1; c < kMmaMaxChunks; ++c) bytes = ch == c ? rb[c] : bytes;
            if (issued >= L.S) mbar_wait_spin(&bars[L.S + slot], phase ^ 1u);
            mbar_expect_tx(&bars[slot], bytes);
            bulk_load_nohint(smem + (size_t)slot * L.rec_stride,
                             reinterpret_cast<const uint8_t*>(recs) + (size_t)(i0 + k) * stride, bytes, &bars[slot]);
            ++issued;
            if (++slot == L.S) slot = 0, phase ^= 1u;
            if (--left == 0) ++ch, left = RT;
          }
        }
        if (lane == 0 && a.tl) a.tl[((size_t)s * a.grid + blockIdx.x) * 8 + 7] = gtimer();  // step's copies issued
        __syncwarp();
      }
    }
    return;
  }
  if (warp == kNW + 1) {
    uint32_t nq = 0;
    csr_prepare(s_view[0], L, smem, bars + 2 * L.S + 1, st, lane, nq);
    for (uint32_t s = 0; s < a.nsteps; ++s) {
      csr_compute(s_view[s & 1], L, smem, bars + 2 * L.S, s & 1u, bars + 2 * L.S + 1, s_x, s_csr, st, lane, nq);
      named_sync(1, (kNW + 1) * 32);  // meet the consumers: sums complete; s_view[s+1] written
      named_sync(2, (kNW + 1) * 32);  // s_csr read by the reduction: free for the next step
      // the next step's row pointers + first entry spans: under its dependency wait
      if (s + 1 < a.nsteps) csr_prepare(s_view[(s + 1) & 1], L, smem, bars + 2 * L.S + 1, st, lane, nq);
    }
    return;
  }
  WarpBlocks wb;
  for (uint32_t s = 0; s < a.nsteps; ++s) {
    const StepView& v = s_view[s & 1];
    unsigned long long* tl = a.tl ? a.tl + ((size_t)s * a.grid + blockIdx.x) * 8 : nullptr;
    if (tl && threadIdx.x == 0) tl[0] = gtimer();  // step start
    if (threadIdx.x == 0 && s + 1 < a.nsteps) load_view(s + 1, s_view[(s + 1) & 1]);  // read after barrier 1
    // the step's first-chunk block descriptors + perm entries: their loads
    // fly under the dependency wait
    if (v.i1 > v.i0) fetch_blocks(wb, v, v.i0 / v.RT, warp, lane);
    if (s > 0 && a.steps[s].depends) {  // x is step s-1's y: all of it
      if (threadIdx.x == 0) {
        const uint32_t* cnt = a.done + (s - 1);
        uint32_t seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
        } while (seen < a.grid);
      }
      named_sync(3, kNW * 32);
    }
    if (tl && threadIdx.x == 0) tl[4] = gtimer();  // dependency resolved
    consumer_step(v, L, smem, bars, bars + L.S, bars + 2 * L.S, s & 1u, s_x, s_part, s_csr, st, warp, lane, false,
                  wb, true, nullptr, tl);
    if (tl && threadIdx.x == 0) tl[5] = gtimer();  // reduction / fixup done (thread 0)
    // CTA barrier, then one cumulative release: every consumer's y / partial
    // / fixup write is ordered before the step counter
    named_sync(2, (kNW + 1) * 32);
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.done + s) : "memory");
      if (tl) tl[6] = gtimer();
    }
  }
}

cudaError_t launch_ex(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                      void** params) {
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

size_t align16(size_t v) { return (v + 15) / 16 * 16; }

uint32_t diag_flags() {
  static const char* d = qwdev::knob_str("QW_DEBUG_MMA_DIAG");
  return d ? (uint32_t)std::atoi(d) : 0u;
}

// Split a group's items (chunk-major per layer) over `grid` CTAs in
// proportion to the layers' item counts; CTAs past the work get empty ranges.
void split_items(const DeviceLayer* const* layers, uint32_t n, uint32_t grid, uint8_t* seg, uint32_t* i0,
                 uint32_t* i1, uint32_t& items_max) {
  uint64_t total = 0;
  uint32_t items[kMaxSeg];
  for (uint32_t l = 0; l < n; ++l) items[l] = layers[l]->mg.RT * layers[l]->mg.nchunks, total += items[l];
  const uint32_t used = (uint32_t)std::max<uint64_t>(std::min<uint64_t>(grid, total), n);
  uint32_t gl[kMaxSeg], given = 0;
  uint64_t acc = 0;
  for (uint32_t l = 0; l < n; ++l) {
    acc += items[l];
    const uint32_t upto = (uint32_t)(used * acc / total);
    gl[l] = std::max<uint32_t>(1, std::min<uint32_t>(items[l], upto > given ? upto - given : 1));
    given += gl[l];
  }
  while (given > used) {
    uint32_t mi = 0;
    for (uint32_t l = 1; l < n; ++l) mi = gl[l] > gl[mi] ? l : mi;
    --gl[mi], --given;
  }
  uint32_t cta = 0;
  for (uint32_t l = 0; l < n; ++l)
    for (uint32_t b = 0; b < gl[l]; ++b, ++cta) {
      seg[cta] = (uint8_t)l;
      i0[cta] = (uint32_t)((uint64_t)b * items[l] / gl[l]);
      i1[cta] = (uint32_t)((uint64_t)(b + 1) * items[l] / gl[l]);
      items_max = std::max(items_max, i1[cta] - i0[cta]);
    }
  for (; cta < grid; ++cta) seg[cta] = 0, i0[cta] = i1[cta] = 0;
}

// largest 16-byte aligned CSR entry span of one 16-row tile
uint32_t csr_span_max(const DeviceLayer* const* layers, const uint32_t* const* host_row_ptrs, uint32_t n) {
  uint32_t cmax = 0;
  for (uint32_t l = 0; l < n; ++l) {
    const uint32_t rows = layers[l]->g.rows;
    for (uint32_t t = 0; t < layers[l]->mg.RT; ++t) {
      const uint32_t e0 = host_row_ptrs[l][16 * t] & ~3u, e1 = host_row_ptrs[l][std::min(16 * t + 16, rows)];
      cmax = std::max(cmax, ((e1 - e0) * 4u + 15u) & ~15u);
    }
  }
  return cmax;
}

// Shared-memory layout for rec_stride / cols / items_max / CSR span maxima.
int make_layout(MmaLayout& L, uint32_t rec_stride, uint32_t cols, uint32_t items_max, uint32_t csr_max,
                uint32_t& smem, size_t extra = 0) {
  L = MmaLayout{};
  L.rec_stride = rec_stride, L.items_cap = std::max(items_max, 1u), L.diag = diag_flags();
  L.csr_slot = std::min<uint32_t>(csr_max, 12 * 1024);
  const size_t x_bytes = align16(((size_t)cols + 1) * 4);
  const size_t part_bytes = (size_t)L.items_cap * 16 * kNW * 4;
  const size_t csr_bytes = align16((size_t)L.items_cap * 16 * 4);
  const size_t bst_bytes = ((size_t)kNW * 2 * 8 * 20 + 20) * 4;  // B staging + a zero fragment
  const size_t rp_bytes = align16((size_t)L.items_cap * 17 * 4 + (size_t)L.items_cap * 2);
  const size_t fixed = x_bytes + part_bytes + csr_bytes + bst_bytes + rp_bytes + extra + 16 + 128 /* alignment */;
  // 8 consumer warps: half an SM, so the next launch's CTA co-resides (PDL)
  const size_t limit = (kNW <= 8 && !extra ? 112 : 227) * 1024;
  size_t S = std::min<size_t>(L.items_cap, 16);
  // CSR ring: every tile span of the CTA in flight at once when it fits (a
  // span refilled only after an earlier one was summed costs a memory
  // latency on the CSR warp's critical path)
  L.csr_nslot = 2;
  while (L.csr_nslot < kCsrSlotsMax && L.csr_nslot < L.items_cap && L.csr_nslot * 2 * L.csr_slot <= 48 * 1024)
    L.csr_nslot *= 2;
  auto total_b = [&](size_t s) {
    return s * rec_stride + L.csr_nslot * L.csr_slot + fixed + (2 * s + 1 + kCsrSlotsMax) * 8;
  };
  while (S > 2 && total_b(S) > limit) --S;
  while (total_b(S) > limit && L.csr_nslot > 2) L.csr_nslot /= 2;  // shallower CSR ring
  while (total_b(S) > limit && L.csr_slot > 1024) L.csr_slot = L.csr_slot / 2 & ~15u;  // rest from global
  if (total_b(S) > limit) return (int)cudaErrorInvalidConfiguration;
  L.S = (uint32_t)S;
  L.x_off = (uint32_t)(S * rec_stride);
  L.part_off = L.x_off + (uint32_t)x_bytes;
  L.csr_off = L.part_off + (uint32_t)part_bytes;
  L.ent_off = L.csr_off + (uint32_t)csr_bytes;
  L.rp_off = L.ent_off + L.csr_nslot * L.csr_slot;
  L.bst_off = L.rp_off + (uint32_t)rp_bytes;
  L.bar_off = L.bst_off + (uint32_t)bst_bytes;
  smem = L.bar_off + (uint32_t)(((2 * S + 1 + kCsrSlotsMax) * 8 + 15) / 16 * 16 + extra) + 128;
  return 0;
}

int opt_in_smem(const void* fn) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static uint64_t done[2] = {0, 0};  // bit per device: the >48 KB opt-in is per device
  const int which = fn == (const void*)mma_gemv_kernel ? 0 : 1;
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 64 || !(done[which] & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return (int)e;
    if (dev < 64) done[which] |= 1ull << dev;
  }
  return 0;
}

bool same_columns(const DeviceLayer* const* layers, uint32_t n) {
  const Geometry& G = layers[0]->g;
  for (uint32_t l = 0; l < n; ++l) {
    const Geometry& H = layers[l]->g;
    if (!layers[l]->mg.ok || H.cols != G.cols || H.n4 != G.n4 || H.n2p != G.n2p || H.group2 != G.group2)
      return false;
  }
  return true;
}

}  // namespace

int plan_mma(MmaPlan& p, const DeviceLayer* const* layers, const uint32_t* const* host_row_ptrs, uint32_t n,
             int num_sms) {
  if (n == 0 || n > kMaxSeg) return (int)cudaErrorInvalidValue;
  if (!layers[0]->mg.ok) return (int)cudaErrorNotSupported;
  if (!same_columns(layers, n)) return (int)cudaErrorInvalidValue;
  p = MmaPlan{};
  uint64_t total = 0;
  for (uint32_t l = 0; l < n; ++l) total += layers[l]->mg.RT * layers[l]->mg.nchunks;
  const uint32_t grid =
      std::max<uint32_t>((uint32_t)std::min<uint64_t>(std::min<uint32_t>((uint32_t)num_sms, kMaxGrid), total), n);
  split_items(layers, n, grid, p.cta_seg, p.cta_i0, p.cta_i1, p.items_max);
  p.grid = grid;
  MmaLayout L;
  uint32_t smem = 0;
  if (int e = make_layout(L, layers[0]->mg.rec_stride, layers[0]->g.cols, p.items_max,
                          csr_span_max(layers, host_row_ptrs, n), smem))
    return e;
  p.nslot = L.S, p.smem = smem;
  p.x_off = L.x_off, p.part_off = L.part_off, p.csr_off = L.csr_off, p.ent_off = L.ent_off;
  p.csr_slot = L.csr_slot, p.csr_nslot = L.csr_nslot, p.rp_off = L.rp_off, p.bst_off = L.bst_off;
  p.bar_off = L.bar_off;
  return opt_in_smem((const void*)mma_gemv_kernel);
}

int launch_mma(const MmaPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* const* xs,
               float* const* ys, void* stream, bool pdl, uint32_t flags, const uint32_t* slots,
               unsigned long long* dbg) {
  const DeviceLayer& L0 = *layers[0];
  const MmaGeometry& m = L0.mg;
  MmaArgs a;
  std::memset(&a, 0, sizeof a);
  const size_t part_slot = (size_t)(m.nchunks + 1) * m.RT * 16;  // floats per scratch slot
  for (uint32_t l = 0; l < kMaxSeg; ++l) {
    const uint32_t s = std::min(l, n - 1);
    const DeviceLayer& L = *layers[s];
    a.recs[l] = L.mrecs, a.perm16[l] = L.perm16, a.row_ptr[l] = L.row_ptr, a.csr[l] = L.csr;
    a.y[l] = ys[s];
    a.xs[l] = xs[s];
    // the columns of one layer must not share its chunk-partial scratch
    const uint32_t slot = slots ? slots[s] : 0u;
    a.part[l] = L.mpart ? L.mpart + slot * part_slot : nullptr;
    a.cnt[l] = L.mcnt ? L.mcnt + slot * m.RT : nullptr;
    a.rows[l] = L.g.rows, a.RT[l] = L.mg.RT;
    a.inv_s_scale[l] = 1.0f / L.plan.s_scale;
  }
  a.cols = L0.g.cols, a.n2p = L0.g.n2p, a.G2 = L0.g.G2, a.T4 = L0.g.T4, a.nchunks = m.nchunks;
  a.wait_x = (flags & kXIndependent) ? 0u : 1u;
  a.lay = MmaLayout{p.nslot, m.rec_stride, p.x_off, p.part_off, p.csr_off, p.ent_off, p.csr_slot, p.csr_nslot,
                    p.rp_off, p.bst_off, p.bar_off, p.items_max, diag_flags(),
                    (flags & kXIndependent) ? 0u : qwdev::knob("QW_MMA_XGATE", 0)};
  for (uint32_t c = 0; c < kMmaMaxChunks; ++c) a.chunk[c] = m.chunk[c];
  std::copy(p.cta_seg, p.cta_seg + p.grid, a.cta_seg);
  std::copy(p.cta_i0, p.cta_i0 + p.grid, a.cta_i0);
  std::copy(p.cta_i1, p.cta_i1 + p.grid, a.cta_i1);
  a.dbg = dbg;
  void* params[] = {&a};
  return (int)launch_ex((const void*)mma_gemv_kernel, dim3(p.grid), dim3(kThreads), p.smem,
                        (cudaStream_t)stream, pdl, params);
}

int launch_mma(const MmaPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* x,
               float* const* ys, void* stream, bool pdl, uint32_t flags) {
  const float* xs[kMaxSeg];
  std::fill(xs, xs + kMaxSeg, x);
  return launch_mma(p, layers, n, xs, ys, stream, pdl, flags, nullptr, nullptr);
}

// ------------------------------------------------------------ decode chain
struct MmaChainPlan {
  MmaChainArgs args{};
  void* dmem = nullptr;
  uint32_t smem = 0;
  size_t tl_count = 0;
};

int mma_chain_timeline(const MmaChainPlan* p, unsigned long long* out, size_t n) {
  if (!p || !p->args.tl) return (int)cudaErrorInvalidValue;
  return (int)cudaMemcpy(out, p->args.tl, std::min(n, p->tl_count) * 8, cudaMemcpyDeviceToHost);
}

int plan_mma_chain(MmaChainPlan** out, const ChainStepDesc* steps, uint32_t n, int num_sms) {
  *out = nullptr;
  if (n == 0) return (int)cudaErrorInvalidValue;
  const uint32_t grid = std::min<uint32_t>((uint32_t)num_sms, kMaxGrid);
  std::vector<MmaStepDesc> sd(n);
  std::vector<MmaCtaRange> rg((size_t)n * grid);
  uint32_t rec_max = 0, cols_max = 0, items_max = 0, csr_max = 0;
  std::vector<uint8_t> seg(grid);
  std::vector<uint32_t> i0(grid), i1(grid);
  for (uint32_t s = 0; s < n; ++s) {
    const ChainStepDesc& st = steps[s];
    if (st.n == 0 || st.n > kMaxSeg) return (int)cudaErrorInvalidValue;
    for (uint32_t l = 0; l < st.n; ++l)
      if (!st.layers[l]->mrecs) return (int)cudaErrorNotSupported;
    if (!same_columns(st.layers, st.n)) return (int)cudaErrorInvalidValue;
    MmaStepDesc& d = sd[s];
    std::memset(&d, 0, sizeof d);
    const DeviceLayer& L0 = *st.layers[0];
    for (uint32_t l = 0; l < kMaxSeg; ++l) {
      const DeviceLayer& L = *st.layers[std::min(l, st.n - 1)];
      d.recs[l] = L.mrecs, d.perm16[l] = L.perm16, d.row_ptr[l] = L.row_ptr, d.csr[l] = L.csr;
      d.y[l] = st.ys[std::min(l, st.n - 1)];
      d.part[l] = L.mpart, d.cnt[l] = L.mcnt;
      d.rows[l] = L.g.rows, d.RT[l] = L.mg.RT;
      d.inv_s_scale[l] = 1.0f / L.plan.s_scale;
    }
    d.x = st.x;
    d.cols = L0.g.cols, d.n2p = L0.g.n2p, d.G2 = L0.g.G2, d.T4 = L0.g.T4, d.nchunks = L0.mg.nchunks;
    d.depends = st.depends, d.hbm_stride = L0.mg.rec_stride;
    for (uint32_t c = 0; c < kMmaMaxChunks; ++c) d.chunk[c] = L0.mg.chunk[c];
    // every step's records share one ring: one slot stride for all
    rec_max = std::max(rec_max, L0.mg.rec_stride);
    cols_max = std::max(cols_max, L0.g.cols);
    csr_max = std::max(csr_max, csr_span_max(st.layers, st.host_row_ptrs, st.n));
    split_items(st.layers, st.n, grid, seg.data(), i0.data(), i1.data(), items_max);
    for (uint32_t b = 0; b < grid; ++b) rg[(size_t)s * grid + b] = MmaCtaRange{seg[b], i0[b], i1[b], 0};
  }
  auto P = std::make_unique<MmaChainPlan>();
  MmaLayout L;
  if (int e = make_layout(L, rec_max, cols_max, items_max, csr_max, P->smem, 2 * sizeof(StepView) + 16)) return e;
  std::vector<MmaProdStep> pd(rg.size());
  for (uint32_t s = 0; s < n; ++s)
    for (uint32_t b = 0; b < grid; ++b) {
      const MmaCtaRange& r = rg[(size_t)s * grid + b];
      MmaProdStep& q = pd[(size_t)s * grid + b];
      q = MmaProdStep{};
      q.recs = (uint64_t)(uintptr_t)sd[s].recs[r.seg];
      q.i0 = r.i0, q.i1 = r.i1, q.RT = sd[s].RT[r.seg], q.hbm_stride = sd[s].hbm_stride;
      for (uint32_t c = 0; c < kMmaMaxChunks; ++c) q.rec_bytes[c] = sd[s].chunk[c].rec_bytes;
    }
  // a layer's records were laid out with its own stride: the ring slot uses
  // the largest, the producer addresses records with the layer's stride
  const size_t b_steps = sizeof(MmaStepDesc) * n, b_ranges = sizeof(MmaCtaRange) * rg.size();
  const size_t b_prod = sizeof(MmaProdStep) * pd.size(), b_done = 4 * n;
  const char* tle = qwdev::knob_str("QW_DEBUG_MMA_TL");
  const size_t b_tl = (tle && tle[0] == '1') ? (size_t)n * grid * 8 * 8 : 0;
  cudaError_t e = cudaMalloc(&P->dmem, b_steps + b_ranges + b_prod + b_done + 64 + b_tl);
  if (e != cudaSuccess) return (int)e;
  uint8_t* base = static_cast<uint8_t*>(P->dmem);
  cudaMemcpy(base, sd.data(), b_steps, cudaMemcpyHostToDevice);
  cudaMemcpy(base + b_steps, rg.data(), b_ranges, cudaMemcpyHostToDevice);
  cudaMemcpy(base + b_steps + b_ranges, pd.data(), b_prod, cudaMemcpyHostToDevice);
  P->args.steps = reinterpret_cast<const MmaStepDesc*>(base);
  P->args.ranges = reinterpret_cast<const MmaCtaRange*>(base + b_steps);
  P->args.prod = reinterpret_cast<const MmaProdStep*>(base + b_steps + b_ranges);
  P->args.done = reinterpret_cast<uint32_t*>(base + b_steps + b_ranges + b_prod);
  P->args.tl = b_tl ? reinterpret_cast<unsigned long long*>(base + ((b_steps + b_ranges + b_prod + b_done + 63) & ~size_t(63)))
                    : nullptr;
  P->tl_count = b_tl / 8;
  P->args.nsteps = n, P->args.grid = grid, P->args.lay = L;
  if (int oe = opt_in_smem((const void*)mma_chain_kernel)) {
    cudaFree(P->dmem);
    return oe;
  }
  *out = P.release();
  return 0;
}

int launch_mma_chain(const MmaChainPlan* p, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(p->args.done, 0, 4 * (size_t)p->args.nsteps, st);
  if (e != cudaSuccess) return (int)e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->args.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p->smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the step counters are grid-wide
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {const_cast<MmaChainArgs*>(&p->args)};
  return (int)cudaLaunchKernelExC(&cfg, (const void*)mma_chain_kernel, params);
}

void free_mma_chain(MmaChainPlan* p) {
  if (!p) return;
  if (p->dmem) cudaFree(p->dmem);
  delete p;
}

}  // namespace qwdev
