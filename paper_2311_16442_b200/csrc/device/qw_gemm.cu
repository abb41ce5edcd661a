// qw_gemm.cu -- K4: the batched (2..16 activation columns) quantized linear on
// the 5th-generation tensor cores (north-star (d)).
//
// Same semantics as K2 (matvec_oracle per column, engine.cpp:169-183), but
// here the layer is a dense contraction, so the weights are dequantized once
// into fp16 tiles in shared memory and fed to tcgen05.mma (kind::f16, M=128,
// N=16, fp32 accumulation in TMEM) against the 16 activation columns.
//
//   xprep_kernel  one CTA per column n: x_n gathered into permuted order
//                 (apply_permutation, plan.cpp:107-116; pads 0), scaled by a
//                 power of two 2^-e_n (max |x'| in [2^14, 2^15)), stored as
//                 fp16 B tiles already in the UMMA K-major core-matrix layout
//                 (one contiguous 4 KB block per 128-channel stage).
//   gemm_kernel   CTA = (128-row M tile, K split).  Warp 0: TMA 2-D boxes of
//                 the quad records (code2 / meta / code4 / s4 / z4 of 32 quads
//                 per stage) + the stage's B tile.  Warps 2-9: dequantize one
//                 (quad, group) item each per stage -- the 2-order dequant
//                 s1 = (eff - zero2) * scale2 (engine.cpp:48-63) folded into
//                 w = (c - z) s1 with exactly one rounding to fp16 -- into an
//                 MN-major A tile (row pairs are adjacent M elements, so the
//                 packed fp16x2 results store directly; SBO/LBO chosen so the
//                 8-byte stores are bank-conflict free).  Warp 1: one thread
//                 issues 8 tcgen05.mma per stage, tcgen05.commit frees the A/B
//                 buffers.  Warps 2-5 read the 128x16 accumulator with
//                 tcgen05.ld, undo the power-of-two scales, add the CSR
//                 outliers (exact fp32) and store y.  Two K-split schedules:
//                 cluster split-K (the tile's splits form a cluster and sum
//                 through distributed shared memory in split order) and
//                 stream-K (gemm_kernel<true>: 148 CTAs take equal contiguous
//                 ranges of the tiles x weight-stages work, at most two tiles
//                 each with one TMEM accumulator per tile; partials go to
//                 global slots and a tile's last arrival sums them in
//                 contributor order).  Both deterministic; plan_gemm picks
//                 stream-K when it shortens the critical path (86-tile
//                 gate/up: every SM busy instead of 86).
//
// A tile value = RN_fp16((c - z) * (eff - zero2) * scale2 * 2^-P): the
// integer part is formed exactly by one HFMA2 on subnormal-coded operands
// (c 2^(b-24) * m 2^(12-b) + (-z m 2^-12)), the scale by one HMUL2, so each
// tile element is the correctly rounded fp16 of the reference's fp32 weight
// (reconstruct_dense) times 2^-P.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "qw_device.hpp"
#include "qw_ptx.cuh"

namespace qwdev {
namespace {

constexpr uint32_t kTileRows = 128, kTileQuads = 32;
constexpr uint32_t kStageK = 128;              // MMA sub-stage: 2 tiles = 96 2-bit + 32 4-bit channels
constexpr uint32_t kSubPerW = 4;               // a weight stage holds 4 sub-stages (8 tiles)
constexpr uint32_t kASbo = 144, kALbo = 2320;  // A tile: m-block / k-block strides (bytes)
constexpr uint32_t kATileBytes = 16 * kALbo;   // 16 k-blocks
constexpr uint32_t kBStageBytes = kStageK * 16 * 2;  // 4 KB: 8 slabs of 16 k x 16 n
// weight stage in shared memory: [32 quads][box] per field, boxes in u32 units
// over 8 tiles (wide rows keep the TMA request count low), plus the 2-order
// params of the tile's row blocks [<= 33][24 groups] (read from shared memory:
// a global load in flight would stall the async-proxy fence that publishes A)
// Box widths: the fields a sub-stage needs (96, 16, 64, 16, 4 u32) padded so
// the quad rows of a box sit at bank-spread strides (dequant lane = quad):
// conflict-free 16-byte code loads, at most 2-way for the small fields.
constexpr uint32_t kBoxC2 = 100, kBoxMeta = 20, kBoxC4 = 68, kBoxS4 = 20, kBoxZ4 = 8;  // u32
constexpr uint32_t kSoBoxG = 24, kSoRowsMax = 33;
constexpr uint32_t kOffC2 = 0, kOffMeta = kOffC2 + 32 * kBoxC2 * 4, kOffC4 = kOffMeta + 32 * kBoxMeta * 4,
                   kOffS4 = kOffC4 + 32 * kBoxC4 * 4, kOffZ4 = kOffS4 + 32 * kBoxS4 * 4,
                   kOffSo = kOffZ4 + 32 * kBoxZ4 * 4,
                   kWStageBytes = (kOffSo + kSoRowsMax * kSoBoxG * 4 + 1023) / 1024 * 1024;  // 28 KB
constexpr uint32_t kWSlots = 2, kBSlots = 8, kABufs = 3;
constexpr uint32_t kDqWarps = 16;
constexpr uint32_t kStreamMaxK = 8;       // stream-K: contributors per tile (partial slots) at most
constexpr uint32_t kDenseStride = 20;  // fp32 words per accumulator row in shared memory
constexpr uint32_t kThreads = (2 + kDqWarps) * 32;
static_assert(kThreads >= 128 * 4, "split-K epilogue: one (row, 4 columns) item per thread");

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);  // no swizzle, sm100 version
}
// kind::f16, D f32, A f16 MN-major, B f16 K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 15) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t h2u(half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ float p2(int e) { return __uint_as_float((uint32_t)(max(-126, min(127, e)) + 127) << 23); }

// ---------------------------------------------------------------- x prologue
// Column n of x (original order) -> fp16 B tiles in stage order: stage st
// holds 2-bit permuted channels [96 st, 96 st + 96) then 4-bit channels
// n2p + [32 st, 32 st + 32); element (k, n) of a stage at
// (k % 8) * 2 + (n % 8) * 16 + (n / 8) * 128 + (k / 8) * 256.
// Grid (chunks + csr_blocks, batch): a chunk CTA re-derives its column's
// power-of-two scale from a full (L2-resident, independent-load) max, then
// converts kPrepPer elements per thread (independent loads, so no thread waits
// on a chain); few enough CTAs to run in one wave beside the GEMM's.
constexpr uint32_t kPrepThreads = 256, kPrepPer = 4;
constexpr uint32_t kPrepPdlMaxBlocks = 192;  // launch_gemm: PDL for the x prologue up to this grid
// CSR outliers of every row for all columns: y_csr[n][r] = sum over the row's
// entries, in CSR order, of fp16(v) * x_n[perm[col]] (sparse_matvec,
// outliers.cpp:131-141), exact fp32.  One thread per (row, column); the row's
// entries are loaded first so the x gathers are independent.
constexpr uint32_t kCsrRound = 24;
__device__ __forceinline__ void csr_row(const float* __restrict__ xn, const uint32_t* __restrict__ row_ptr,
                                        const uint32_t* __restrict__ csr, uint32_t rows, float* __restrict__ yn,
                                        uint32_t row) {
  // the row's bounds and first kCsrRound entries are layer constants: loaded before
  // the dependency wait (under the previous kernel), only the x gathers after
  uint32_t e0 = 0, e1 = 0;
  if (row < rows) e0 = __ldg(row_ptr + row), e1 = __ldg(row_ptr + row + 1);
  float acc = 0.0f;
  // kCsrRound entries per round: a row of <= kCsrRound outliers costs one load
  // after the wait
  for (uint32_t e = e0, first = 1; first || e < e1; e += kCsrRound, first = 0) {
    uint32_t ent[kCsrRound];
#pragma unroll
    for (int u = 0; u < (int)kCsrRound; ++u) ent[u] = e + u < e1 ? __ldg(csr + e + u) : 0u;
    if (first) pdl_wait();  // x is the previous kernel's output
    if (e >= e1) break;
    float p[kCsrRound];
#pragma unroll
    for (int u = 0; u < (int)kCsrRound; ++u)
      p[u] = __fmul_rn(half_bits_to_float(ent[u] >> 16), __ldg(xn + (ent[u] & 0xFFFFu)));  // original channel
#pragma unroll
    for (int u = 0; u < (int)kCsrRound; ++u)
      if (e + u < e1) acc = __fadd_rn(acc, p[u]);
  }
  if (row < rows) yn[row] = acc;
}

__global__ void __launch_bounds__(kPrepThreads, 4) xprep_kernel(const float* __restrict__ x,
                                                             const uint16_t* __restrict__ perm, Geometry G,
                                                             uint32_t stages, uint32_t batch,
                                                             uint16_t* __restrict__ xpt, int* __restrict__ xexp,
                                                             uint32_t chunks, const uint32_t* __restrict__ row_ptr,
                                                             const uint32_t* __restrict__ csr,
                                                             float* __restrict__ ycsr) {
  // launched with PDL: resident under the previous kernel; layer constants
  // (perm, CSR) are read before griddepcontrol.wait, x after it
  pdl_launch_dependents();  // the GEMM's weight stream does not depend on us
  if (blockIdx.x >= chunks) {  // CSR blocks: one row of column blockIdx.y per thread
    if (blockIdx.y < batch)
      csr_row(x + (size_t)blockIdx.y * G.cols, row_ptr, csr, G.rows, ycsr + (size_t)blockIdx.y * G.rows,
              (blockIdx.x - chunks) * kPrepThreads + threadIdx.x);
    else
      pdl_wait();
    return;
  }
  const uint32_t n = blockIdx.y;
  const float* xn = x + (size_t)n * G.cols;
  __shared__ float red[kPrepThreads / 32];
  const uint32_t n2 = G.cols - G.n4;
  // the gathered elements are loaded before / beside the max pass (only the
  // scale depends on the max): two dependent loads per thread in total
  uint32_t ch[kPrepPer];
#pragma unroll
  for (uint32_t u = 0; u < kPrepPer; ++u) {
    const uint32_t i = (blockIdx.x * kPrepPer + u) * kPrepThreads + threadIdx.x;
    ch[u] = 0xFFFFFFFFu;
    if (i < stages * kStageK && n < batch) {
      const uint32_t st = i / kStageK, k = i % kStageK;
      const uint32_t slot = k < 96 ? 96 * st + k : G.n2p + 32 * st + (k - 96);
      if (!(slot >= n2 && slot < G.n2p)) ch[u] = __ldg(perm + slot);
    }
  }
  pdl_wait();  // x is the previous kernel's output
  float xv[kPrepPer];
#pragma unroll
  for (uint32_t u = 0; u < kPrepPer; ++u) xv[u] = ch[u] != 0xFFFFFFFFu ? __ldg(xn + ch[u]) : 0.0f;
  float m = 0.0f;
  if (n < batch) {
    const uint32_t n4v = G.cols >> 2;  // cols % 16 == 0 (validate_layer)
    const float4* x4 = reinterpret_cast<const float4*>(xn);
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < n4v; i += kPrepThreads) {
      const float4 v = __ldg(x4 + i);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < (int)(kPrepThreads / 32); ++w) m = fmaxf(m, red[w]);
  const int eb = (int)((__float_as_uint(m) >> 23) & 0xFFu);
  const int e = (eb == 0 ? -126 : eb - 127) - 14;  // max |x'| in [2^14, 2^15)
  if (threadIdx.x == 0 && blockIdx.x == 0) xexp[n] = e;
  const int ea = max(-126, min(127, -e));
  const float f1 = p2(ea), f2 = p2(-e - ea);
#pragma unroll
  for (uint32_t u = 0; u < kPrepPer; ++u) {
    const uint32_t i = (blockIdx.x * kPrepPer + u) * kPrepThreads + threadIdx.x;
    if (i >= stages * kStageK) break;
    const uint32_t st = i / kStageK, k = i % kStageK;
    const float v = xv[u] * f1 * f2;
    const uint32_t off = (k % 8) * 2 + (n % 8) * 16 + (n / 8) * 128 + (k / 8) * 256;
    xpt[(size_t)st * (kBStageBytes / 2) + off / 2] = __half_as_ushort(__float2half_rn(v));
  }
}

// ---------------------------------------------------------------- GEMM
struct GemmArgs {
  CUtensorMap tm[5];  // code2, meta, code4, s4, z4 boxes over [quads][dense_bytes]
  CUtensorMap tso;    // sorder box: [row blocks of a tile][8 groups]
  uint32_t so_rows;   // row blocks a tile spans (box height)
  Geometry g;
  const uint32_t* sorder;
  const uint32_t* row_ptr;
  const uint32_t* csr;
  const uint16_t* perm;
  const uint16_t* xpt;
  const int* xexp;
  const float* x;
  float* y;
  float* partial;
  const float* ycsr;  // [batch][rows] CSR outlier sums (prologue kernel)
  uint32_t* counters;
  uint32_t batch, ks, stages, wstages;
  uint32_t stream, W, C, kmax;  // stream-K: W = tiles x wstages over C CTAs; kmax partial slots per tile
  int shift;
  uint32_t rb_magic, rb_one;
  unsigned long long* dbg;  // optional [grid][8] %globaltimer stamps
};
__device__ __forceinline__ void gstamp(const GemmArgs& a, uint32_t ev) {
  if (a.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[blockIdx.x * 8 + ev] = t;
  }
}

// stream-K: the CTA whose weight-stage range holds flattened index i
// (ranges [c W / C, (c + 1) W / C)): the largest c with floor(c W / C) <= i
__device__ __forceinline__ uint32_t stream_first(const GemmArgs& a, uint32_t i) {
  return (uint32_t)(((uint64_t)(i + 1) * a.C - 1) / a.W);
}

// kStream: stream-K schedule (a separate instantiation: the cluster split-K
// kernel keeps its tighter hot loop)
template <bool kStream>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (an
  // integer round trip would make every A/W access a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const Geometry& G = a.g;
  uint8_t* sA = smem;                                // kABufs x kATileBytes
  uint8_t* sB = sA + kABufs * kATileBytes;           // kBSlots x 4 KB
  uint8_t* sW = sB + kBSlots * kBStageBytes;         // kWSlots x 6656
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + kWSlots * kWStageBytes);
  uint64_t* wfull = bars;              // [kWSlots]  TMA tx
  uint64_t* wempty = wfull + kWSlots;  // [kWSlots]  8 dequant warps
  uint64_t* bfull = wempty + kWSlots;  // [kBSlots]  TMA tx
  uint64_t* bempty = bfull + kBSlots;  // [kBSlots]  tcgen05.commit
  uint64_t* afull = bempty + kBSlots;  // [kABufs]   dequant warps
  uint64_t* aempty = afull + kABufs;   // [kABufs]   tcgen05.commit
  uint64_t* dfull = aempty + kABufs;   // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dfull + 1);
  uint32_t* s_last = tmem_slot + 1;
  // [128][kDenseStride]: 16-byte rows so the split-K reduction reads float4s
  float* s_dense = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(s_last + 3) +
                                            ((16u - (smem_addr(s_last + 3) & 15u)) & 15u));

  // Work: up to two segments (tile, weight-stage range).  Cluster split-K
  // (kStream false): CTA = (tile, split), one segment.  Stream-K: the
  // tiles x wstages weight stages are cut into C equal contiguous ranges (one
  // CTA each, every SM busy); a range spans at most two tiles (W / C <=
  // wstages), partials meet in global memory (stream_fixup).
  // (scalars, not arrays: dynamic indexing would put them on the stack)
  uint32_t tile, tile1, w00, nw0, nw1;
  const uint32_t split = kStream ? 0u : blockIdx.x % a.ks;
  if (kStream) {
    const uint32_t i0 = (uint32_t)((uint64_t)blockIdx.x * a.W / a.C);
    const uint32_t i1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * a.W / a.C);
    tile = i0 / a.wstages, w00 = i0 % a.wstages;
    const uint32_t e0 = min(i1, (tile + 1) * a.wstages);
    nw0 = e0 - i0, tile1 = tile + 1, nw1 = i1 - e0;
  } else {
    // K split over weight stages (8 tiles); sub-stages of 2 tiles feed the MMA
    const uint32_t w0 = (uint32_t)((uint64_t)split * a.wstages / a.ks);
    const uint32_t w1 = (uint32_t)((uint64_t)(split + 1) * a.wstages / a.ks);
    tile = tile1 = blockIdx.x / a.ks, w00 = w0, nw0 = w1 - w0, nw1 = 0;
  }
  const uint32_t nseg = (kStream && nw1) ? 2u : 1u;
  const uint32_t nw = nw0 + nw1;
  // sub-stages of this CTA (stream-K needs stages % kSubPerW == 0)
  const uint32_t nsub = kStream ? nw * kSubPerW : min((w00 + nw) * kSubPerW, a.stages) - w00 * kSubPerW;
  const uint32_t seg1_sub = nw0 * kSubPerW;  // first sub-stage of segment 1
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  auto rb_of = [&](uint32_t t) { return a.rb_one ? t * kTileRows : __umulhi(t * kTileRows, a.rb_magic); };
  // local weight stage j -> weight stage within its segment's tile
  auto wst_of = [&](uint32_t j) { return (!kStream || j < nw0) ? w00 + j : j - nw0; };

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < kWSlots; ++i) mbar_init(&wfull[i], 1), mbar_init(&wempty[i], kDqWarps);
    for (uint32_t i = 0; i < kBSlots; ++i) mbar_init(&bfull[i], 1), mbar_init(&bempty[i], 1);
    for (uint32_t i = 0; i < kABufs; ++i) mbar_init(&afull[i], kDqWarps / 2), mbar_init(&aempty[i], 1);
    mbar_init(dfull, 1);
    mbar_fence_init();
  }
  if (warp == 1) {  // TMEM: 32 columns (the 128 x 16 fp32 accumulator)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) gstamp(a, 0);  // setup done

  if (warp == 0) {
    // ---------------- producer: weight boxes (8 tiles) + B tiles (per sub-stage)
    if (lane == 0) {
      auto load_w = [&](uint32_t i) {
        const uint32_t t = (!kStream || i < nw0) ? tile : tile1;
        const int qy = (int)(t * kTileQuads);
        const uint32_t wst = wst_of(i), ws = i % kWSlots;
        if (i >= kWSlots) mbar_wait(&wempty[ws], ((i / kWSlots) - 1) & 1u);
        uint8_t* dst = sW + ws * kWStageBytes;
        mbar_expect_tx(&wfull[ws], kOffSo + a.so_rows * kSoBoxG * 4);
        tma_load_2d(dst + kOffC2, &a.tm[0], (int)(96 * wst), qy, &wfull[ws]);
        tma_load_2d(dst + kOffMeta, &a.tm[1], (int)(G.off_meta / 4 + 16 * wst), qy, &wfull[ws]);
        tma_load_2d(dst + kOffC4, &a.tm[2], (int)(G.off_c4 / 4 + 64 * wst), qy, &wfull[ws]);
        tma_load_2d(dst + kOffS4, &a.tm[3], (int)(G.off_s4 / 4 + 16 * wst), qy, &wfull[ws]);
        tma_load_2d(dst + kOffZ4, &a.tm[4], (int)(G.off_z4 / 4 + 4 * wst), qy, &wfull[ws]);
        tma_load_2d(dst + kOffSo, &a.tso, (int)(24 * wst), (int)rb_of(t), &wfull[ws]);
      };
      // the weights do not depend on x; a weight slot is refilled once every
      // dequant warp left it
      for (uint32_t i = 0; i < nw; ++i) load_w(i);
    } else if (lane == 1) {
      // B tiles (the prologue kernel's output) from their own thread: a B
      // refill must not wait behind a weight-slot refill (the MMA would
      // starve, the A buffers fill up and the dequant warps stall)
      pdl_wait();
      for (uint32_t i = 0; i < nsub; ++i) {
        const uint32_t bs = i % kBSlots;
        if (i >= kBSlots) mbar_wait(&bempty[bs], ((i / kBSlots) - 1) & 1u);
        mbar_expect_tx(&bfull[bs], kBStageBytes);
        const uint32_t u = wst_of(i / kSubPerW) * kSubPerW + i % kSubPerW;  // sub-stage within the tile's K
        bulk_load_nohint(sB + bs * kBStageBytes, a.xpt + (size_t)u * (kBStageBytes / 2), kBStageBytes,
                         &bfull[bs]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      for (uint32_t i = 0; i < nsub; ++i) {
        const uint32_t ab = i % kABufs, ph = (i / kABufs) & 1u, bs = i % kBSlots;
        mbar_wait(&afull[ab], ph);
        mbar_wait(&bfull[bs], (i / kBSlots) & 1u);

        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t abase = smem_addr(sA + ab * kATileBytes), bbase = smem_addr(sB + bs * kBStageBytes);
        // segment s accumulates in TMEM columns [16 s, 16 s + 16)
        const uint32_t first = (i == 0 || (kStream && i == seg1_sub)) ? 1u : 0u;
        const uint32_t dacc = tmem + ((kStream && i >= seg1_sub) ? 16u : 0u);
#pragma unroll
        for (uint32_t kk = 0; kk < kStageK / 16; ++kk) {
          const uint64_t da = umma_desc(abase + 2 * kk * kALbo, kALbo, kASbo);
          const uint64_t db = umma_desc(bbase + kk * 512, 256, 128);
          const uint32_t acc = (first && kk == 0) ? 0u : 1u;
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(dacc),
                       "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_addr(&aempty[ab])));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_addr(&bempty[bs])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_addr(dfull)));
    }
  } else {
    // ---------------- dequant warps: item = (quad q, group j) of a sub-stage, both
    // 8-channel halves (the per-(row pair, group) constants are formed once
    // for 16 channels).  Lane = quad; 8 warps per sub-stage, the two warp
    // halves take alternate sub-stages (two A buffers in flight); warps with
    // j < 6 take the 2-bit groups, j >= 6 the 4-bit ones, so no warp diverges
    // over the two decode paths.
    const uint32_t dw = warp - 2, q = lane;
    const uint32_t j = dw & 7u, par = dw >> 3;
    // the quad's row block relative to its tile's first, per segment
    auto rbl_of = [&](uint32_t t) {
      const uint32_t row0 = min((t * kTileQuads + q) * 4, G.rows - 1);
      return (a.rb_one ? row0 : __umulhi(row0, a.rb_magic)) - rb_of(t);
    };
    const uint32_t rbl0 = rbl_of(tile), rbl1 = kStream ? rbl_of(tile1) : rbl0;
    const float s2sc = p2(12 - a.shift), s4sc = p2(9 - a.shift);
    const uint32_t sub = j % 3;
    const uint32_t esh = sub == 0 ? 6u : (sub == 1 ? 10u : 13u), emask = sub == 0 ? 15u : 7u;
    const uint32_t eshl = sub == 0 ? 0u : 1u;
    // (1024 + field) 2^eshl - 1024 2^eshl = eff, exactly (fp16 integers <= 2078 are even above 2048)
    const half2 e2h = __float2half2_rn(eshl ? 2.0f : 1.0f), eoff = __float2half2_rn(eshl ? -2048.0f : -1024.0f);
    const half2 h1024 = __float2half2_rn(1024.0f);
    const uint32_t a_item = (q & 1u) * 8 + (q >> 1) * kASbo + (2 * j) * kALbo;  // + h kALbo + (c % 8) * 16
    for (uint32_t i = par; i < nsub; i += 2) {
      const uint32_t wi = i / kSubPerW, s4i = i % kSubPerW, ws = wi % kWSlots, ab = i % kABufs;
      if (s4i == par) mbar_wait(&wfull[ws], (wi / kWSlots) & 1u);  // this warp's first sub-stage of the stage
      if (threadIdx.x == 64 && i == 2) gstamp(a, 1);  // sub-stage 2 weights present
      const uint8_t* w = sW + ws * kWStageBytes;
      const uint32_t rb_local = (!kStream || wi < nw0) ? rbl0 : rbl1;
      uint32_t out[2][8][2];  // [half][channel pair][row pair]
      if (j < 6) {
        const uint32_t g6 = 6 * s4i + j;  // 2-bit group within the weight stage
        const uint32_t sc = *reinterpret_cast<const uint32_t*>(w + kOffSo + (rb_local * kSoBoxG + g6) * 4);
        const uint4 c = *reinterpret_cast<const uint4*>(w + kOffC2 + q * kBoxC2 * 4 + 16 * g6);
        const uint2 m = *reinterpret_cast<const uint2*>(w + kOffMeta + q * kBoxMeta * 4 + 8 * (g6 / 3));
        const half2 Sh = __float2half2_rn(half_bits_to_float(sc) * s2sc);  // scale2 2^(12-P)
        const half2 z2h = __float2half2_rn((float)(sc >> 16));                // zero2 (exact)
        const uint32_t mm[2] = {m.x, m.y}, cw[2][2] = {{c.x, c.z}, {c.y, c.w}};  // [half][row pair]
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t v = mm[p];
          // fp16 integers from 0x6400 (1024) | field, both rows at once, exact:
          // mrow = eff - zero2 (eff = field << eshl), z = the group's 2-bit zero
          const half2 e = __hfma2(as_h2(((v >> esh) & (emask | (emask << 16))) | 0x64006400u), e2h, eoff);
          const half2 mrow = __hsub2(e, z2h);
          const half2 zh = __hsub2(as_h2(((v >> (2 * sub)) & 0x00030003u) | 0x64006400u), h1024);
          half2 M[4];  // mrow 2^(12 - 2b): c 2^(2b-24) * M[b] = c mrow 2^-12
          M[0] = __hmul2(mrow, __float2half2_rn(4096.0f));
          M[1] = __hmul2(mrow, __float2half2_rn(1024.0f));
          M[2] = __hmul2(mrow, __float2half2_rn(256.0f));
          M[3] = __hmul2(mrow, __float2half2_rn(64.0f));
          const half2 Z = __hmul2(zh, __hmul2(mrow, __float2half2_rn(-1.0f / 4096.0f)));  // -z mrow 2^-12
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t src = cc < 4 ? cw[h][p] : cw[h][p] >> 8;
              const int b = cc & 3;
              const half2 t = as_h2(src & (0x00030003u << (2 * b)));
              out[h][cc][p] = h2u(__hmul2(__hfma2(t, M[b], Z), Sh));
            }
        }
      } else {
        const uint32_t b2 = 2 * s4i + (j - 6);  // 4-bit block within the weight stage
        const uint4 ca = *reinterpret_cast<const uint4*>(w + kOffC4 + q * kBoxC4 * 4 + 32 * b2);
        const uint4 cb = *reinterpret_cast<const uint4*>(w + kOffC4 + q * kBoxC4 * 4 + 32 * b2 + 16);
        const uint2 s4 = *reinterpret_cast<const uint2*>(w + kOffS4 + q * kBoxS4 * 4 + 8 * b2);
        const uint32_t z4 = *reinterpret_cast<const uint16_t*>(w + kOffZ4 + q * kBoxZ4 * 4 + 2 * b2);
        // [half][row pair][word]: half h is words (2h, 2h + 1) of each 16-byte code group
        const uint32_t cw[2][2][2] = {{{ca.x, ca.y}, {cb.x, cb.y}}, {{ca.z, ca.w}, {cb.z, cb.w}}};
        const uint32_t sw[2] = {s4.x, s4.y};
        const half2 M0 = __float2half2_rn(32768.0f), M1 = __float2half2_rn(2048.0f);  // 2^(15-b)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          // zeros of the row pair as fp16 integers (0x6400 | z - 1024), times -2^-9
          const uint32_t zz = ((z4 >> (8 * p)) & 0xFu) | (((z4 >> (8 * p + 4)) & 0xFu) << 16);
          const half2 Z = __hmul2(__hsub2(as_h2(zz | 0x64006400u), __float2half2_rn(1024.0f)),
                                  __float2half2_rn(-1.0f / 512.0f));
          const half2 Sh = as_h2(pack_h2(half_bits_to_float(sw[p]) * s4sc, half_bits_to_float(sw[p] >> 16) * s4sc));
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t word = cw[h][p][cc >> 2];
              const int nib = cc & 3;
              const uint32_t src = nib < 2 ? word : word >> 8;
              const half2 t = as_h2(src & (0x000F000Fu << (4 * (nib & 1))));
              out[h][cc][p] = h2u(__hmul2(__hfma2(t, (nib & 1) ? M1 : M0, Z), Sh));
            }
        }
      }
      if (s4i + 2 >= kSubPerW || i + 2 >= nsub) {  // this warp's last use of the weight slot
        __syncwarp();
        if (lane == 0) mbar_arrive(&wempty[ws]);
      }

      if (i >= kABufs) mbar_wait(&aempty[ab], ((i / kABufs) - 1) & 1u);

      uint8_t* at = sA + ab * kATileBytes + a_item;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<uint2*>(at + h * kALbo + cc * 16) = make_uint2(out[h][cc][0], out[h][cc][1]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
    }
    // ---------------- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
    if (warp < 6) {
      // the column scales (prologue output) are loaded while the last MMAs run
      pdl_wait();
      float csc[16];
#pragma unroll
      for (int n = 0; n < 16; ++n) csc[n] = p2(a.shift + __ldg(a.xexp + n));
      mbar_wait(dfull, 0);
      if (threadIdx.x == 64) gstamp(a, 7);  // accumulator ready
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t quarter = warp & 3u;
      const uint32_t t = quarter * 32 + lane;  // row within the tile
      for (uint32_t sg = 0; sg < nseg; ++sg) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tmem + 16u * sg + ((quarter * 32u) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        float v[16];
#pragma unroll
        for (int n = 0; n < 16; ++n) v[n] = __uint_as_float(r[n]) * csc[n];
        if (!kStream) {
#pragma unroll
          for (int n = 0; n < 16; ++n) s_dense[t * kDenseStride + n] = v[n];
          continue;
        }
        const uint32_t st = sg ? tile1 : tile, row = st * kTileRows + t;
        const uint32_t cf = stream_first(a, st * a.wstages), nc = stream_first(a, st * a.wstages + a.wstages - 1) + 1 - cf;
        if (nc == 1) {  // the whole tile's K is ours: finish the rows here
          if (row < G.rows) {
#pragma unroll
            for (uint32_t n = 0; n < 16; ++n)
              if (n < a.batch) a.y[(size_t)n * G.rows + row] = v[n] + __ldg(a.ycsr + (size_t)n * G.rows + row);
          }
        } else {  // partial slot (tile, contributor index)
          float4* dst = reinterpret_cast<float4*>(a.partial + ((size_t)(st * a.kmax + blockIdx.x - cf) * kTileRows + t) * 16);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) dst[c4] = make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) gstamp(a, 2);  // CTA joined after the accumulator read
  // the next launch (its x prologue, PDL) may become resident for our tail:
  // it reads nothing of ours before its griddepcontrol.wait
  pdl_launch_dependents();

  if (kStream) {
    // stream-K fixup: the last contributor of a tile (arrival counter) sums
    // the tile's partial slots in contributor order -- deterministic
    pdl_wait();  // the CSR sums are the prologue kernel's
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (uint32_t sg = 0; sg < 2; ++sg) {
        s_last[sg] = 0;
        if (sg >= nseg) continue;
        const uint32_t st = sg ? tile1 : tile;
        const uint32_t cf = stream_first(a, st * a.wstages), nc = stream_first(a, st * a.wstages + a.wstages - 1) + 1 - cf;
        if (nc > 1 && atomicAdd(a.counters + st, 1u) == nc - 1) s_last[sg] = nc;
      }
    }
    __syncthreads();
    for (uint32_t sg = 0; sg < nseg; ++sg) {
      const uint32_t nc = s_last[sg];
      if (!nc) continue;
      __threadfence();
      const uint32_t st = sg ? tile1 : tile;
      const float* part = a.partial + (size_t)st * a.kmax * kTileRows * 16;
      // item = (row, 4 columns): one float4 per contributor slot, all in
      // flight, summed in contributor order (one pass: <= 128 x 4 items)
      const uint32_t nc4 = (a.batch + 3) / 4;
      for (uint32_t i = threadIdx.x; i < kTileRows * nc4; i += blockDim.x) {
        const uint32_t t = i % kTileRows, c4 = i / kTileRows, row = st * kTileRows + t;
        float4 v[kStreamMaxK];
#pragma unroll
        for (uint32_t k = 0; k < kStreamMaxK; ++k)
          v[k] = k < nc ? __ldcg(reinterpret_cast<const float4*>(part + ((size_t)k * kTileRows + t) * 16) + c4)
                        : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        float csr[4];
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          csr[q] = (row < G.rows && 4 * c4 + q < a.batch) ? __ldg(a.ycsr + (size_t)(4 * c4 + q) * G.rows + row) : 0.0f;
        float4 sum = v[0];
#pragma unroll
        for (uint32_t k = 1; k < kStreamMaxK; ++k)
          if (k < nc) sum.x += v[k].x, sum.y += v[k].y, sum.z += v[k].z, sum.w += v[k].w;
        if (row < G.rows) {
          const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q)
            if (4 * c4 + q < a.batch) a.y[(size_t)(4 * c4 + q) * G.rows + row] = sv[q] + csr[q];
        }
      }
      if (threadIdx.x == 0) a.counters[st] = 0;  // every contributor has arrived: reset for the next call
    }
  } else if (a.ks == 1) {
    // dense part of this split is in s_dense[row][n] (row-major, padded stride)
    // the dense sum, then the outliers (row_fma, engine.cpp:111-122): their
    // per-row CSR sums (exact fp32, CSR order) come from the prologue kernel
    pdl_wait();
    // item = (row, 4 columns): the CSR sums loaded together, one pass
    const uint32_t nc4 = (a.batch + 3) / 4;
    for (uint32_t i = threadIdx.x; i < kTileRows * nc4; i += blockDim.x) {
      const uint32_t t = i % kTileRows, c4 = i / kTileRows, row = tile * kTileRows + t;
      if (row >= G.rows) continue;
      float csr[4];
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q)
        csr[q] = 4 * c4 + q < a.batch ? __ldg(a.ycsr + (size_t)(4 * c4 + q) * G.rows + row) : 0.0f;
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q)
        if (4 * c4 + q < a.batch)
          a.y[(size_t)(4 * c4 + q) * G.rows + row] = s_dense[t * kDenseStride + 4 * c4 + q] + csr[q];
    }
  } else {
    // split-K: the tile's K splits form one thread-block cluster; CTA `split`
    // sums rows [split * 128 / ks, ...) over the splits' shared-memory
    // partials (distributed shared memory) in split order -- deterministic.
    // Split-phase cluster barriers: arrive as soon as s_dense is complete,
    // load this thread's CSR sums (the prologue kernel's, in L2) before the
    // wait; after the remote reads arrive again, store y, then wait (no CTA
    // leaves while a peer may still read its shared memory).
    // item = (row, 4 columns), one per thread (<= 128 x 4 < kThreads)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    pdl_wait();
    if (threadIdx.x == 0) gstamp(a, 4);  // prologue kernel complete
    const uint32_t r0 = split * kTileRows / a.ks, r1 = (split + 1) * kTileRows / a.ks;
    const uint32_t nr = r1 - r0, nc4 = (a.batch + 3) / 4;
    const bool item = threadIdx.x < nr * nc4;
    const uint32_t t = r0 + (item ? threadIdx.x % nr : 0u), c4 = item ? threadIdx.x / nr : 0u;
    const uint32_t row = tile * kTileRows + t;
    float csr[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (item && row < G.rows) {
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k)
        if (4 * c4 + k < a.batch) csr[k] = __ldg(a.ycsr + (size_t)(4 * c4 + k) * G.rows + row);
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) gstamp(a, 3);  // cluster joined
    float4 sum = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (item) {
      const uint32_t local = smem_addr(s_dense);
      // the splits' float4 partials all in flight, then summed in split order
      float4 v[8];
#pragma unroll
      for (uint32_t sp = 0; sp < 8; ++sp) {
        v[sp] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (sp < a.ks) {
          uint32_t remote;
          asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local + (t * kDenseStride + 4 * c4) * 4), "r"(sp));
          asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v[sp].x), "=f"(v[sp].y), "=f"(v[sp].z), "=f"(v[sp].w)
                       : "r"(remote)
                       : "memory");
        }
      }
      sum = v[0];
#pragma unroll
      for (uint32_t sp = 1; sp < 8; ++sp)
        if (sp < a.ks) sum.x += v[sp].x, sum.y += v[sp].y, sum.z += v[sp].z, sum.w += v[sp].w;
    }
    // the remote reads are consumed: peers may leave once everyone got here
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if (item && row < G.rows) {
      const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) {
        const uint32_t n = 4 * c4 + k;
        if (n < a.batch) a.y[(size_t)n * G.rows + row] = sv[k] + csr[k];
      }
    }
    if (threadIdx.x == 0) gstamp(a, 5);  // partials summed (thread 0)
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) gstamp(a, 6);  // y stored
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

constexpr size_t kGemmSmem = 1024 + kABufs * kATileBytes + kBSlots * kBStageBytes + kWSlots * kWStageBytes + 512 +
                             kTileRows * kDenseStride * 4 + 16;
static_assert(kGemmSmem <= 227 * 1024, "gemm shared memory");

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

int plan_gemm(DeviceLayer& L, int num_sms, float max_scale2, float max_s4) {
  const Geometry& G = L.g;
  GemmPlan& p = L.gemm;
  p = GemmPlan{};
  // supported: paired tiles only (T2 == T4, even), 2-order blocks aligned to quads
  if (G.T2 != G.T4 || G.T2 % 2 != 0 || G.T2 == 0 || G.group2 % kRowsPerQuad != 0) return 0;
  auto enc = encode_fn();
  if (!enc) return 0;
  p.tiles = (G.rows + kTileRows - 1) / kTileRows;
  p.stages = G.T2 / 2;                               // MMA sub-stages per row
  p.wstages = (p.stages + kSubPerW - 1) / kSubPerW;  // weight stages per row
  p.ks = std::max<uint32_t>(1, std::min<uint32_t>(std::min<uint32_t>(p.wstages, 8u), (uint32_t)num_sms / p.tiles));
  const char* force_ks = qwdev::knob_str("QW_GEMM_KS");  // diagnostics: force the cluster K split
  if (force_ks)
    p.ks = std::max<uint32_t>(1, std::min<uint32_t>(std::min<uint32_t>(p.wstages, 8u), (uint32_t)std::atoi(force_ks)));
  // stream-K when it shortens the critical path: every SM takes an equal
  // contiguous range of the tiles x wstages weight stages (cluster split-K
  // leaves SMs idle when 148 / tiles is small, e.g. 86 tiles -> ks = 1)
  {
    const uint32_t W = p.tiles * p.wstages, C = std::min<uint32_t>((uint32_t)num_sms, W);
    const uint32_t crit_ks = (p.wstages + p.ks - 1) / p.ks, crit_stream = (W + C - 1) / C;
    if (!force_ks && !qwdev::knob_str("QW_GEMM_NOSTREAM") && p.stages % kSubPerW == 0 && p.tiles <= C &&
        crit_stream < crit_ks) {
      auto first = [&](uint64_t i) { return (uint32_t)(((i + 1) * C - 1) / W); };
      uint32_t kmax = 0;
      for (uint32_t t = 0; t < p.tiles; ++t)
        kmax = std::max(kmax, first((uint64_t)t * p.wstages + p.wstages - 1) + 1 - first((uint64_t)t * p.wstages));
      if (kmax <= kStreamMaxK) p.stream = 1, p.W = W, p.C = C, p.kmax = kmax;
    }
  }
  // A = w 2^-P in fp16: scale2 2^(12-P) <= 2^15 and s4 2^(9-P) <= 2^15
  int P = -126;
  if (max_scale2 > 0.0f && std::isfinite(max_scale2)) P = std::max(P, std::ilogb(max_scale2) - 2);
  if (max_s4 > 0.0f && std::isfinite(max_s4)) P = std::max(P, std::ilogb(max_s4) - 5);
  p.shift = std::max(-100, std::min(100, P == -126 ? 0 : P));
  const uint32_t boxw[5] = {kBoxC2, kBoxMeta, kBoxC4, kBoxS4, kBoxZ4};
  for (int f = 0; f < 5; ++f) {
    cuuint64_t dims[2] = {G.dense_bytes / 4, G.quads};
    cuuint64_t strides[1] = {G.dense_bytes};
    cuuint32_t box[2] = {boxw[f], kTileQuads};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(p.tmap[f]), CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, L.quads, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 0;
  }
  {  // sorder [row_blocks][G2s] u32, box [so_rows][8 groups]
    p.so_rows = (kTileRows + G.group2 - 1) / G.group2 + (kTileRows % G.group2 ? 1u : 0u);
    if (p.so_rows > kSoRowsMax) return 0;
    cuuint64_t dims[2] = {G.G2s, G.row_blocks};
    cuuint64_t strides[1] = {(cuuint64_t)G.G2s * 4};
    cuuint32_t box[2] = {kSoBoxG, p.so_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(p.tmap_so), CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, L.sorder, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 0;
  }
  cudaError_t e;
  // stream-K partial slots [tiles][kmax][128 rows][16 columns]
  if ((e = cudaMalloc((void**)&p.partial, p.stream ? (size_t)p.tiles * p.kmax * kTileRows * 16 * 4 : 16)) !=
      cudaSuccess)
    return (int)e;
  if ((e = cudaMalloc((void**)&p.counters, (size_t)p.tiles * 4)) != cudaSuccess) return (int)e;
  if ((e = cudaMemset(p.counters, 0, (size_t)p.tiles * 4)) != cudaSuccess) return (int)e;
  if ((e = cudaMalloc((void**)&p.xpt, (size_t)p.stages * kBStageBytes)) != cudaSuccess) return (int)e;
  if ((e = cudaMalloc((void**)&p.xexp, 16 * sizeof(int))) != cudaSuccess) return (int)e;
  if ((e = cudaMalloc((void**)&p.ycsr, (size_t)16 * G.rows * 4)) != cudaSuccess) return (int)e;
  // zeroed once: a call writes only its `batch` columns of the B tiles and
  // exponents, the MMA and the epilogue read all 16 (the rest never reach y;
  // compute-sanitizer initcheck)
  if ((e = cudaMemset(p.xpt, 0, (size_t)p.stages * kBStageBytes)) != cudaSuccess) return (int)e;
  if ((e = cudaMemset(p.xexp, 0, 16 * sizeof(int))) != cudaSuccess) return (int)e;
  // the opt-in limits are per device: one bit per device, set under a lock
  static std::mutex attr_mu;
  static uint64_t attr_dev = 0;
  int cur = 0;
  cudaGetDevice(&cur);
  std::lock_guard<std::mutex> lk(attr_mu);
  if (cur >= 64 || !(attr_dev & (1ull << cur))) {
    for (const void* k : {(const void*)gemm_kernel<false>, (const void*)gemm_kernel<true>}) {
      if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem)) != cudaSuccess)
        return (int)e;
      if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
        return (int)e;
    }
    if (cur < 64) attr_dev |= 1ull << cur;
  }
  p.ok = 1;
  return 0;
}

void free_gemm(DeviceLayer& L) {
  GemmPlan& p = L.gemm;
  cudaFree(p.partial), cudaFree(p.counters), cudaFree(p.xpt), cudaFree(p.xexp), cudaFree(p.ycsr);
  p.partial = nullptr, p.counters = nullptr, p.xpt = nullptr, p.xexp = nullptr, p.ycsr = nullptr;
  p.ok = 0;
}

int launch_gemm(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream,
                unsigned long long* dbg) {
  const Geometry& G = L.g;
  const GemmPlan& p = L.gemm;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t chunks = (p.stages * kStageK + kPrepThreads * kPrepPer - 1) / (kPrepThreads * kPrepPer);
  const uint32_t csr_blocks = (G.rows + kPrepThreads - 1) / kPrepThreads;
  // one grid row per live column: the B columns >= batch are never stored
  // (MMA columns are independent), and a small prologue grid leaves the SMs
  // free for the GEMM's CTAs, which launch as soon as it starts (PDL)
  static const bool no_pdl = qwdev::knob_str("QW_GEMM_NOPDL") != nullptr;  // diagnostics
  {
    // PDL: the prologue's CTAs become resident under the previous kernel and
    // wait for it in griddepcontrol.wait instead of a launch after it
    cudaLaunchConfig_t pc = {};
    pc.gridDim = dim3(chunks + csr_blocks, batch);
    pc.blockDim = dim3(kPrepThreads);
    pc.stream = st;
    cudaLaunchAttribute pa[1];
    pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pa[0].val.programmaticStreamSerializationAllowed = 1;
    pc.attrs = pa;
    // PDL only for a grid that fits beside the running kernel about once per
    // SM: the prologue CTAs sit resident (blocked in griddepcontrol.wait)
    // until the previous kernel completes, and an SM holding two of them has
    // no registers left for a GEMM CTA of the next launch (80 x 576 + 2 x 64
    // x 256 > 64 K), which then starts late (measured: 4096 x 11008 at b = 8
    // +8 us with PDL, 4096^2 at b = 2 -2.5 us)
    const uint32_t nblk = (chunks + csr_blocks) * batch;
    pc.numAttrs = (no_pdl || nblk > kPrepPdlMaxBlocks) ? 0 : 1;
    cudaError_t e = cudaLaunchKernelEx(&pc, xprep_kernel, x, (const uint16_t*)L.perm16, G, p.stages, batch, p.xpt,
                                       p.xexp, chunks, (const uint32_t*)L.row_ptr, (const uint32_t*)L.csr, p.ycsr);
    if (e != cudaSuccess) return (int)e;
  }
  GemmArgs a;
  std::memcpy(a.tm, p.tmap, sizeof(a.tm));
  std::memcpy(&a.tso, p.tmap_so, sizeof(a.tso));
  a.so_rows = p.so_rows;
  a.g = G;
  a.sorder = L.sorder, a.row_ptr = L.row_ptr, a.csr = L.csr, a.perm = L.perm16;
  a.xpt = p.xpt, a.xexp = p.xexp, a.x = x, a.y = y;
  a.partial = p.partial, a.counters = p.counters, a.ycsr = p.ycsr;
  a.batch = batch, a.ks = p.ks, a.stages = p.stages, a.wstages = p.wstages, a.shift = p.shift;
  a.stream = p.stream, a.W = p.W, a.C = p.C, a.kmax = p.kmax;
  a.rb_magic = L.plan.rb_magic, a.rb_one = L.plan.rb_one;
  a.dbg = dbg;
  // cluster = the tile's K splits (DSMEM reduction); PDL: the weight stream
  // starts while the prologue runs, B tiles / scales wait for it
  cudaLaunchConfig_t cfg = {};
  const bool use_stream = p.stream != 0;
  a.stream = use_stream;
  a.ks = use_stream ? 1u : p.ks;
  cfg.gridDim = dim3(use_stream ? p.C : p.tiles * p.ks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kGemmSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.ks, attr[0].val.clusterDim.y = 1, attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 1 : 2;
  void* params[] = {&a};
  return (int)cudaLaunchKernelExC(&cfg, use_stream ? (const void*)gemm_kernel<true> : (const void*)gemm_kernel<false>,
                                  params);
}

}  // namespace qwdev
