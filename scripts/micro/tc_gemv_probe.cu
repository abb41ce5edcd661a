// Throughput probe for a tcgen05 batch-1 main loop (DESIGN §8 item 2): the
// compute ceiling of "decode 2-bit codes to fp16 subnormals in registers ->
// tcgen05.st into TENSOR MEMORY (A) -> tcgen05.mma against a block-diagonal x
// (B, one 16-channel group per N column) -> tcgen05.ld of the per-group dots
// -> fp32 FMA with the per-(row, group) scales", against K2's ~55-64 weights
// per ns per SM.  Synthetic smem-resident data (no HBM): every CTA re-decodes
// the same 128-row x KCH-channel chunk ITER times, two A and two D buffers
// so the decode of chunk c overlaps the MMAs of chunk c-1; KCH / TMEM_COLS
// set how many CTAs (4 warps each) share an SM.  Checks the row sums against
// the host (exact), prints weights / ns / SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DKCH=80 -DTMEM_COLS=128 tc_gemv_probe.cu
// run:   ./a.out 592   (grid = 148 x CTAs per SM)
//
// Code layout (probe-specific): word w of a row holds channels 10w+b (low
// half) and 10w+5+b (high half) at bit 2b, b < 5, so one LOP3 yields the
// fp16 subnormal pair c 2^(2b-24) of TMEM column 5w+b; B holds x 2^(14-2b) at
// the matching K index, D = sum c x 2^-10 per group.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#ifndef NACC
#define NACC 1
#endif
#ifndef KCH
#define KCH 240
#endif
#ifndef TMEM_COLS
#define TMEM_COLS 512
#endif
// chunk of KCH channels (a multiple of 80: whole code words and whole MMA K steps)
constexpr int kRows = 128, kCh = KCH, kWords = kCh / 10, kGroups = kCh / 16, kCols = kCh / 2;
constexpr int kStride = (kWords / 4) % 2 ? kWords : kWords + 4;  // odd multiple of 4 words: conflict-free LDS.128
constexpr uint32_t kDBase = 2 * kCols;  // TMEM: A buffers at 0 and kCols, then the D buffers
constexpr int kNAcc = NACC;  // D accumulators per chunk: MMA kk writes D[kk % kNAcc] (independent chains)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

#define ST8(addr, r, o)                                                                                       \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),          \
               "r"(r[o]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3]), "r"(r[o + 4]), "r"(r[o + 5]), "r"(r[o + 6]), \
               "r"(r[o + 7]))

__global__ void __launch_bounds__(128, 512 / TMEM_COLS) probe(const uint32_t* g_codes, const uint16_t* g_b, const float* g_sc,
                                                float* out, int iters) {
  __shared__ __align__(16) uint32_t s_codes[kRows * kStride];
  __shared__ __align__(1024) uint16_t s_b[kCh * 16];
  __shared__ __align__(16) float s_sc[kRows * 20];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kRows * kWords; i += 128) s_codes[(i / kWords) * kStride + i % kWords] = g_codes[i];
  for (int i = tid; i < kCh * 16; i += 128) s_b[i] = g_b[i];
  for (int i = tid; i < kRows * 16; i += 128) s_sc[(i / 16) * 20 + i % 16] = g_sc[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot, lane_base = (uint32_t)(warp * 32) << 16;
  const uint32_t bdesc0 = smem_u32(s_b);
  float acc = 0.0f;
  float sc[16];
  for (int n = 0; n < 16; ++n) sc[n] = s_sc[tid * 20 + n];

  auto epilogue = [&](int c) {
    const uint32_t buf = c & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(smem_u32(&bar[buf])), "r"((uint32_t)((c >> 1) & 1)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int q = 0; q < kNAcc; ++q) {
      uint32_t d[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
            "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
          : "r"(tmem + lane_base + kDBase + 16u * (buf * kNAcc + q)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int n = 0; n < kGroups; ++n) acc = fmaf(sc[n], __uint_as_float(d[n]), acc);
    }
  };

  for (int c = 0; c < iters; ++c) {
    const uint32_t buf = c & 1;
    // decode: this thread's row, kWords words -> kCols TMEM columns
    uint32_t w[kWords];
#pragma unroll
    for (int q = 0; q < kWords / 4; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(&s_codes[tid * kStride + 4 * q]);
      w[4 * q] = v.x, w[4 * q + 1] = v.y, w[4 * q + 2] = v.z, w[4 * q + 3] = v.w;
    }
    uint32_t r[kCols];
#pragma unroll
    for (int i = 0; i < kWords; ++i)
#pragma unroll
      for (int b = 0; b < 5; ++b) r[5 * i + b] = w[i] & (0x00030003u << (2 * b));
    const uint32_t a = tmem + lane_base + (uint32_t)kCols * buf;
#pragma unroll
    for (int p = 0; p < kCols / 8; ++p) ST8(a + 8u * p, r, 8 * p);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
#pragma unroll
      for (int kk = 0; kk < kCh / 16; ++kk) {
        const uint64_t bd = desc(bdesc0 + kk * 512, 256, 128);
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(
                         tmem + kDBase + 16u * (buf * kNAcc + kk % kNAcc)),
                     "r"(tmem + (uint32_t)kCols * buf + 8u * kk), "l"(bd), "r"(kIdesc), "r"(kk >= kNAcc ? 1 : 0));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bar[buf])));
    }
    if (c > 0) epilogue(c - 1);
  }
  epilogue(iters - 1);
  out[blockIdx.x * kRows + tid] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
}

int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 148;
  srand(3);
  std::vector<uint32_t> codes(kRows * kWords);
  std::vector<int> cv(kRows * kCh);
  for (int r = 0; r < kRows; ++r)
    for (int i = 0; i < kWords; ++i) {
      uint32_t word = 0;
      for (int b = 0; b < 5; ++b)
        for (int h = 0; h < 2; ++h) {
          const int c = rand() & 3, ch = 10 * i + 5 * h + b;
          cv[r * kCh + ch] = c;
          word |= (uint32_t)c << (2 * b + 16 * h);
        }
      codes[r * kWords + i] = word;
    }
  std::vector<float> x(kCh);
  for (int ch = 0; ch < kCh; ++ch) x[ch] = (float)((rand() % 17) - 8) / 8.0f;
  // B[k][n], k = TMEM K index: column j = 5 i + b holds (ch 10 i + b, ch 10 i + 5 + b) as K (2 j, 2 j + 1)
  std::vector<uint16_t> hb(kCh * 16, 0);
  for (int j = 0; j < kCols; ++j)
    for (int h = 0; h < 2; ++h) {
      const int i = j / 5, b = j % 5, ch = 10 * i + 5 * h + b, k = 2 * j + h, n = ch / 16;
      const __half v = __float2half(x[ch] * ldexpf(1.0f, 14 - 2 * b));
      uint16_t bits;
      memcpy(&bits, &v, 2);
      hb[((k % 8) * 2 + (n % 8) * 16 + (n / 8) * 128 + (k / 8) * 256) / 2] = bits;
    }
  std::vector<float> sc(kRows * 16, 0.0f);
  for (auto& s : sc) s = (float)((rand() % 15) + 1) / 16.0f;
  uint32_t* d_codes; uint16_t* d_b; float *d_sc, *d_out;
  cudaMalloc(&d_codes, codes.size() * 4); cudaMalloc(&d_b, hb.size() * 2);
  cudaMalloc(&d_sc, sc.size() * 4); cudaMalloc(&d_out, (size_t)grid * kRows * 4);
  cudaMemcpy(d_codes, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_b, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(d_sc, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice);
  for (int iters : {1, 7, 4000}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<<<grid, 128>>>(d_codes, d_b, d_sc, d_out, iters);  // warm
    cudaEventRecord(e0);
    probe<<<grid, 128>>>(d_codes, d_b, d_sc, d_out, iters);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<float> out((size_t)grid * kRows);
    cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int r = 0; r < kRows; ++r) {
      double ref = 0;
      for (int n = 0; n < kGroups; ++n) {
        double dot = 0;
        for (int ch = 16 * n; ch < 16 * n + 16; ++ch) dot += cv[r * kCh + ch] * (double)x[ch];
        ref += sc[r * 16 + n] * dot * ldexp(1.0, -10);
      }
      ref *= iters;
      for (int b = 0; b < grid; ++b) {
        const double err = fabs(out[(size_t)b * kRows + r] - ref) / fmax(fabs(ref), 1e-6);
        worst = fmax(worst, err);
      }
    }
    const double weights = (double)grid * iters * kRows * kCh;
    printf("KCH %d, TMEM %d cols, grid %d (%d CTAs/SM) iters %d: %.3f ms, %.1f weights/ns/SM (%.2f T weights/s), "
           "max rel err %.2e\n", KCH, TMEM_COLS, grid, grid / 148, iters, ms, weights / (ms * 1e6) / 148,
           weights / (ms * 1e9), worst);
  }
  return 0;
}
