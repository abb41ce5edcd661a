// Probe: one tcgen05.mma.cta_group::1.kind::f16 (M=128, N=16, K=16), A and B
// from shared memory through hand-built descriptors (no swizzle), D in TMEM,
// read back with tcgen05.ld.  A is MN-major (rows contiguous, core matrix =
// 8 rows x 8 k, 16 B per k), B is K-major (core matrix = 8 n x 8 k, 16 B per n).
// Checks D == A B on the host for a few (SBO, LBO) choices.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)layout << 61;
  return d;
}
// A[m][k] element offset (bytes) in MN-major no-swizzle layout
__host__ __device__ uint32_t a_off(int m, int k, uint32_t lbo, uint32_t sbo) {
  return (m % 8) * 2 + (k % 8) * 16 + (m / 8) * sbo + (k / 8) * lbo;
}
// B[k][n] element offset (bytes) in K-major no-swizzle layout
__host__ __device__ uint32_t b_off(int n, int k, uint32_t lbo, uint32_t sbo) {
  return (k % 8) * 2 + (n % 8) * 16 + (n / 8) * sbo + (k / 8) * lbo;
}

__global__ void probe(const __half* A, const __half* B, float* D, uint32_t a_lbo, uint32_t a_sbo,
                      uint32_t b_lbo, uint32_t b_sbo, int a_major_mn) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + 32768;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 128 * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    uint32_t off = a_major_mn ? a_off(m, k, a_lbo, a_sbo)
                              : (k % 8) * 2 + (m % 8) * 16 + (m / 8) * a_sbo + (k / 8) * a_lbo;
    *reinterpret_cast<__half*>(sA + off) = A[i];
  }
  for (int i = t; i < 16 * 16; i += blockDim.x) {
    const int k = i / 16, n = i % 16;
    *reinterpret_cast<__half*>(sB + b_off(n, k, b_lbo, b_sbo)) = B[i];
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(sa(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (t == 0) {
    const uint64_t da = desc(sa(sA), a_lbo, a_sbo, 0), db = desc(sa(sB), b_lbo, b_sbo, 0);
    uint32_t idesc = 0;
    idesc |= 1u << 4;                         // D f32
    idesc |= 0u << 7;                         // A f16
    idesc |= 0u << 10;                        // B f16
    idesc |= (a_major_mn ? 1u : 0u) << 15;    // A major
    idesc |= 0u << 16;                        // B K-major
    idesc |= (16u >> 3) << 17;                // N
    idesc |= (128u >> 4) << 24;               // M
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                 :: "r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&bar)));
  }
  // wait for the MMA
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(sa(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads lanes 32w..32w+31, 16 columns
  const int w = t / 32;
  if (w < 4) {
    uint32_t r[16];
    const uint32_t addr = tm + ((uint32_t)(w * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = w * 32 + (t % 32);
    for (int n = 0; n < 16; ++n) D[row * 16 + n] = __uint_as_float(r[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tm));
}

int main() {
  std::vector<__half> A(128 * 16), B(16 * 16);
  std::vector<float> Af(128 * 16), Bf(16 * 16);
  srand(1);
  for (int i = 0; i < 128 * 16; ++i) { float v = (rand() % 17 - 8) / 4.0f; A[i] = __float2half(v); Af[i] = v; }
  for (int i = 0; i < 16 * 16; ++i) { float v = (rand() % 13 - 6) / 2.0f; B[i] = __float2half(v); Bf[i] = v; }
  std::vector<float> ref(128 * 16, 0.0f);
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) { double s = 0; for (int k = 0; k < 16; ++k) s += Af[m * 16 + k] * Bf[k * 16 + n]; ref[m * 16 + n] = s; }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 128 * 16 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  struct Cfg { const char* name; uint32_t alb, asb, blb, bsb; int mn; } cfgs[] = {
    {"A MN-major sbo128 lbo2048 | B sbo128 lbo256", 2048, 128, 256, 128, 1},
    {"A MN-major sbo144 lbo2320 | B sbo128 lbo256", 2320, 144, 256, 128, 1},
    {"A MN-major lbo128 sbo2048 (swapped)", 128, 2048, 256, 128, 1},
    {"A K-major sbo128 lbo2048 | B sbo128 lbo256", 2048, 128, 256, 128, 0},
    {"B swapped lbo/sbo", 2048, 128, 128, 256, 1},
  };
  for (auto& c : cfgs) {
    cudaMemset(dD, 0, 128 * 16 * 4);
    probe<<<1, 128, 65536>>>(dA, dB, dD, c.alb, c.asb, c.blb, c.bsb, c.mn);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(128 * 16);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0; int bad = 0;
    for (int i = 0; i < 128 * 16; ++i) { double d = fabs(D[i] - ref[i]); err = fmax(err, d); bad += d > 1e-3; }
    printf("%-48s err=%s  maxabs=%.4g  bad=%d  D[0..3]=%g %g %g %g ref=%g %g\n", c.name, cudaGetErrorString(e), err, bad, D[0], D[1], D[2], D[3], ref[0], ref[1]);
  }
  return 0;
}
