// Closer mimic of the GEMV's smem fill: per CTA one small copy then nq quad
// copies of Q bytes; 8 "consumer" warps wait on each quad in order; optional
// concurrent x-gather LDG traffic.  Prints per-quad ready cycles of CTA 0
// averaged over CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void fill(const uint8_t* src, int Q, int nq, const float* x, int gather, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[32];
  const uint8_t* base = src + (size_t)blockIdx.x * Q * nq;
  if (threadIdx.x < nq) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bars[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned long long t0 = clock64();
  const int warp = threadIdx.x / 32;
  if (warp == 8) {
    if (threadIdx.x % 32 == 0)
      for (int i = 0; i < nq; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bars[i])), "r"(Q) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(sa(sm + (size_t)i * Q)), "l"(base + (size_t)i * Q), "r"(Q), "r"(sa(&bars[i])) : "memory");
      }
    return;
  }
  if (warp == 9) return;
  float acc = 0.f;
  if (gather) {
    for (int k = 0; k < 16; ++k) acc += __ldg(x + ((threadIdx.x * 16 + k * 7) & 4095));
  }
  for (int i = 0; i < nq; ++i) {
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(&bars[i])) : "memory");
    if (threadIdx.x == 0 && i < 16) out[blockIdx.x * 17 + i] = clock64() - t0;
    acc += sm[i * Q + threadIdx.x];
  }
  if (threadIdx.x == 0) out[blockIdx.x * 17 + 16] = (unsigned long long)acc;
}
int main() {
  const size_t total = 2ull << 30;
  uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
  float* x; cudaMalloc(&x, 4096 * 4); cudaMemset(x, 0, 4096 * 4);
  unsigned long long* d; cudaMalloc(&d, 148 * 17 * 8);
  unsigned long long h[148 * 17];
  cudaFuncSetAttribute(fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  auto run = [&](const char* name, int Q, int nq, int gather, bool hot) {
    size_t off = 0;
    for (int rep = 0; rep < 4; ++rep) {
      if (!hot) off = (size_t)(rep + 1) * 148 * Q * nq * 3 % (total / 2);
      fill<<<148, 320, Q * nq>>>(buf + off, Q, nq, x, gather, d);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("%-28s ready:", name);
    for (int i = 0; i < nq && i < 16; ++i) { double m = 0; for (int b = 0; b < 148; ++b) m += h[b * 17 + i]; printf(" %5.0f", m / 148); }
    printf("\n");
  };
  run("Q=6272 nq=7 hbm", 6272, 7, 0, false);
  run("Q=6272 nq=7 hot", 6272, 7, 0, true);
  run("Q=6272 nq=7 hot +gather", 6272, 7, 1, true);
  run("Q=6144 nq=8 hbm", 6144, 8, 0, false);
  run("Q=6144 nq=8 hot", 6144, 8, 0, true);
  run("Q=12544 nq=4 hot", 12544, 4, 0, true);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
