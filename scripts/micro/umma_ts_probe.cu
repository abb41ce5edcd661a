// Probe for a tcgen05 batch-1 design (DESIGN §8 item 2): one
// tcgen05.mma.cta_group::1.kind::f16 with A read from TENSOR MEMORY (written
// by tcgen05.st from registers, as a decode warp would after its LOP3s) and B
// from shared memory, M = 128, N = 16, K = 16.  A holds fp16 SUBNORMALS
// c 2^(p-24) (a 2-bit code masked into a zero exponent field, K2m's decode
// trick) and B small normal fp16 values, so every product is exact; the
// fp32 accumulator D is compared with the exact sums computed on the host.
// Prints max |D - ref| / |ref| and times a chain of MMAs (cycles per MMA).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// kind::f16: D f32 (bit 4), A/B f16, A K-major (A from TMEM), B K-major, N=16, M=128
constexpr uint32_t kIdesc = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__global__ void probe(const uint32_t* a_words, const uint16_t* b_km, float* d_out, unsigned long long* cyc,
                      int reps) {
  __shared__ __align__(1024) uint16_t sB[16 * 16];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 256; i += blockDim.x) sB[i] = b_km[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  // A: row = tid (TMEM lane), 8 columns (K = 16 fp16) at column 16
  uint32_t r[8];
  for (int c = 0; c < 8; ++c) r[c] = a_words[tid * 8 + c];
  const uint32_t a_addr = tmem + ((uint32_t)(warp * 32) << 16) + 16u;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a_addr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint64_t bd = desc(smem_u32(sB), 256, 128);
    unsigned long long t0 = clock64();
    for (int i = 0; i < reps; ++i) {
      const uint32_t acc = i == 0 ? 0u : 1u;
      asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(tmem), "r"(tmem + 16u),
                   "l"(bd), "r"(kIdesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    cyc[0] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t d[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                 "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
               : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < 16; ++n) d_out[tid * 16 + n] = __uint_as_float(d[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

static float h2f(uint16_t h) {
  __half x;
  memcpy(&x, &h, 2);
  return __half2float(x);
}

int main() {
  // A[row][k]: code c in 0..3 at bit position p (fp16 subnormal c 2^(p-24));
  // word w of a row = (k = 2w low half, k = 2w + 1 high half)
  uint32_t ha[128 * 8];
  double A[128][16];
  srand(7);
  for (int r = 0; r < 128; ++r)
    for (int w = 0; w < 8; ++w) {
      uint32_t word = 0;
      for (int h = 0; h < 2; ++h) {
        const int k = 2 * w + h, c = rand() & 3, p = 2 * (k % 5);
        const uint32_t bits = (uint32_t)c << p;
        word |= bits << (16 * h);
        A[r][k] = c * ldexp(1.0, p - 24);
      }
      ha[r * 8 + w] = word;
    }
  // B[k][n] K-major core-matrix layout: (k % 8) * 2 + (n % 8) * 16 + (n / 8) * 128 + (k / 8) * 256 bytes
  uint16_t hb[256];
  double B[16][16];
  for (int k = 0; k < 16; ++k)
    for (int n = 0; n < 16; ++n) {
      const float v = (float)((rand() % 2001) - 1000) / 8.0f;  // exact in fp16 (11 bits)
      __half hv = __float2half(v);
      uint16_t bits;
      memcpy(&bits, &hv, 2);
      hb[((k % 8) * 2 + (n % 8) * 16 + (n / 8) * 128 + (k / 8) * 256) / 2] = bits;
      B[k][n] = h2f(bits);
    }
  uint32_t* da; uint16_t* db; float* dd; unsigned long long* dc;
  cudaMalloc(&da, sizeof ha); cudaMalloc(&db, sizeof hb); cudaMalloc(&dd, 128 * 16 * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(da, ha, sizeof ha, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, sizeof hb, cudaMemcpyHostToDevice);
  for (int reps : {1, 64}) {
    probe<<<1, 128>>>(da, db, dd, dc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float hd[128 * 16];
    unsigned long long cyc;
    cudaMemcpy(hd, dd, sizeof hd, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double worst = 0, worst_abs = 0; int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < 16; ++n) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) ref += A[r][k] * B[k][n];
        ref *= reps;
        const double err = fabs(hd[r * 16 + n] - ref);
        worst_abs = fmax(worst_abs, err);
        if (ref != 0) worst = fmax(worst, err / fabs(ref));
        if (err > 1e-6 * fabs(ref) + 1e-30) ++bad;
      }
    printf("reps %d: max rel err %.3e (abs %.3e), %d of 2048 outside 1e-6, %llu cycles for %d MMAs (%.1f / MMA)\n",
           reps, worst, worst_abs, bad, cyc, reps, (double)cyc / reps);
  }
  return 0;
}
