// x staging latency: 148 CTAs x 512 threads each load 16 KB (float4) into
// shared memory, all from the SAME 16 KB (a broadcast read, as every GEMV
// CTA stages the whole activation) or each from its own copy.  Optionally
// under a concurrent HBM stream (other CTAs on the same SMs are not possible
// here, so the stream is modelled by a second kernel on another stream).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void stage(const float4* x, int distinct, unsigned long long* t, float* sink) {
  __shared__ float4 s[1024];
  unsigned long long t0, t1, t2, t3;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const float4* src = x + (distinct ? (size_t)blockIdx.x * 1024 : 0);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = __ldcg(src + i);
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  // the same loads again (TLB and L2 warm): the pure L2 round trip
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i].x += __ldcg(src + i).y;
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  // a different page of the same buffer (L2 warm: touched by the previous launch)
  const float4* src2 = x + (size_t)((blockIdx.x + 7) % 148) * 1024;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i].y += __ldcg(src2 + i).x;
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0, t[148 + blockIdx.x] = t2 - t1, t[296 + blockIdx.x] = t3 - t2;
  if (threadIdx.x == 0 && s[5].x == 12345.f) sink[0] = s[7].y;
}
__global__ void hog(const float4* a, float4* b, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  float4 *x, *big_a, *big_b; float* sink; unsigned long long* t;
  cudaMalloc(&x, 148 * 16384); cudaMalloc(&sink, 4); cudaMalloc(&t, 3 * 148 * 8);
  size_t n = (size_t)1 << 26;  // 1 GB
  cudaMalloc(&big_a, n * 16); cudaMalloc(&big_b, n * 16);
  cudaMemset(x, 0, 148 * 16384);
  unsigned long long h[3 * 148];
  cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int load = 0; load < 2; ++load)
    for (int distinct = 0; distinct < 2; ++distinct) {
      double acc = 0, mx = 0, acc2 = 0, acc3 = 0; int reps = 20;
      for (int r = 0; r < reps; ++r) {
        // x in L2 (touch it), then stage
        stage<<<148, 512>>>(x, distinct, t, sink);
        cudaDeviceSynchronize();
        if (load) { hog<<<148, 1024, 0, s2>>>(big_a, big_b, n / 4); }
        stage<<<148, 512>>>(x, distinct, t, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, t, sizeof h, cudaMemcpyDeviceToHost);
        double m = 0, a2 = 0, b2 = 0, c2 = 0;
        for (int i = 0; i < 148; ++i) { a2 += h[i]; b2 += h[148 + i]; c2 += h[296 + i]; if (h[i] > m) m = h[i]; }
        acc += a2 / 148; mx += m; acc2 += b2 / 148; acc3 += c2 / 148;
      }
      printf("hbm_load %d distinct %d: x staging mean %.0f ns (max-over-CTAs %.0f), again %.0f ns, other page %.0f ns\n", load, distinct, acc / reps, mx / reps, acc2 / reps, acc3 / reps);
    }
  return 0;
}
