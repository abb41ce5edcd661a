// ring_bench.cu -- HBM streaming through a shared-memory ring of TMA bulk
// copies (the K2/K2m producer pattern) with no compute: 148 CTAs, each streams
// its own contiguous range through S slots of B bytes; one consumer warp per
// slot-phase waits full and hands the slot back (or `work` spin cycles per
// slot to emulate compute).  Prints GB/s per (B, S).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring_bench ring_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
}

__global__ void ring(const uint8_t* src, size_t per_cta, uint32_t B, uint32_t S, uint32_t nconsumer, int work,
                     float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * B);
  uint64_t* empty = full + S;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < S) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[threadIdx.x])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[threadIdx.x])), "r"(nconsumer));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const uint32_t n = (uint32_t)(per_cta / B);
  if (warp == nconsumer) {
    if (lane == 0) {
      uint32_t slot = 0, ph = 0;
      for (uint32_t k = 0; k < n; ++k) {
        if (k >= S) wait(&empty[slot], ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[slot])), "r"(B)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sa(sm + (size_t)slot * B)),
            "l"(base + (size_t)k * B), "r"(B), "r"(sa(&full[slot]))
            : "memory");
        if (++slot == S) slot = 0, ph ^= 1;
      }
    }
    return;
  }
  float acc = 0.f;
  uint32_t slot = 0, ph = 0;
  for (uint32_t k = 0; k < n; ++k) {
    wait(&full[slot], ph);
    acc += reinterpret_cast<const float*>(sm + (size_t)slot * B)[lane];
    for (int i = 0; i < work; ++i) acc = acc * 1.0000001f + 1e-7f;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[slot])) : "memory");
    if (++slot == S) slot = 0, ph ^= 1;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t per_cta = 3u << 20;  // 3 MB per CTA: 444 MB total (>> L2)
  uint8_t* src;
  float* sink;
  cudaMalloc(&src, per_cta * sms);
  cudaMemset(src, 1, per_cta * sms);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int work : {0, 400}) {
    for (uint32_t B : {6144u, 12288u, 26624u, 53248u}) {
      for (uint32_t S : {2u, 3u, 4u, 6u, 8u, 12u, 16u, 24u, 32u}) {
        if ((size_t)S * B + 2 * S * 8 > 220 * 1024) continue;
        const size_t pc = per_cta / B * B;
        const uint32_t nc = 16;
        const size_t smem = (size_t)S * B + 2 * S * 8;
        ring<<<sms, (nc + 1) * 32, smem>>>(src, pc, B, S, nc, work, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) ring<<<sms, (nc + 1) * 32, smem>>>(src, pc, B, S, nc, work, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("work %3d slot %6u B  slots %2u  in-flight %4zu KB  %7.1f GB/s\n", work, B, S, (size_t)S * B / 1024,
               3.0 * pc * sms / (ms * 1e6));
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
