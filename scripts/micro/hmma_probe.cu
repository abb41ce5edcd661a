// hmma_probe.cu -- can the warp-level tensor-core MMA (mma.sync m16n8k16,
// fp16 in, fp32 accumulate) serve the batch-1 decode?  Two questions:
//  (1) exactness: A holds 2-bit codes masked into fp16 subnormals
//      (c * 2^(2j-24)), B holds x' * 2^-2j; is D the fp32 sum of the exact
//      products (no denormal flush)?
//  (2) throughput: HMMA.16816.F32 / .F16 per SM per clock on sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_probe hmma_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ void mma_f32(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_f16(uint32_t* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
      : "+r"(d[0]), "+r"(d[1])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// (1) one warp: A[16][16] fp16 bits, B[16][8] fp16 bits (k-major per column), D[16][8]
__global__ void exact_kernel(const uint16_t* A, const uint16_t* B, float* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  auto pa = [&](int r, int k) { return (uint32_t)A[r * 16 + k] | ((uint32_t)A[r * 16 + k + 1] << 16); };
  auto pb = [&](int k, int n) { return (uint32_t)B[n * 16 + k] | ((uint32_t)B[n * 16 + k + 1] << 16); };
  uint32_t a[4] = {pa(g, 2 * t), pa(g + 8, 2 * t), pa(g, 2 * t + 8), pa(g + 8, 2 * t + 8)};
  uint32_t b[2] = {pb(2 * t, g), pb(2 * t + 8, g)};
  float d[4] = {0, 0, 0, 0};
  mma_f32(d, a, b);
  D[g * 8 + 2 * t] = d[0], D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2], D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

template <int ACC, bool F32>
__global__ void tput_kernel(int iters, float* sink) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * (i + 1));
  b[0] = 0x3c003c00u, b[1] = 0x00010001u;
  float d[ACC][4] = {};
  uint32_t h[ACC][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ACC; ++j) {
      if (F32) mma_f32(d[j], a, b);
      else mma_f16(h[j], a, b);
    }
  }
  float s = 0;
  for (int j = 0; j < ACC; ++j) s += d[j][0] + d[j][3] + __uint_as_float(h[j][0]);
  if (s == 12345.0f) sink[0] = s;
}

static uint16_t f2h_bits(float f) { __half h = __float2half_rn(f); return *reinterpret_cast<uint16_t*>(&h); }
static double h2d(uint16_t b) { __half h; *reinterpret_cast<uint16_t*>(&h) = b; return (double)__half2float(h); }

int main() {
  // ---- exactness
  const int trials = 200;
  double worst = 0;
  int inexact = 0;
  srand(1);
  uint16_t *dA, *dB;
  float* dD;
  cudaMalloc(&dA, 512); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
  for (int tr = 0; tr < trials; ++tr) {
    uint16_t A[256], B[128];
    int j = tr % 5;  // bit position 2j in the mantissa
    int code[256];
    for (int i = 0; i < 256; ++i) { code[i] = rand() & 3; A[i] = (uint16_t)(code[i] << (2 * j)); }
    double xv[128];
    for (int i = 0; i < 128; ++i) {
      // x' in [2^10, 2^11) magnitude range as the kernel prepares it, then * 2^-2j
      float x = (float)((rand() / (double)RAND_MAX) * 4096.0 - 2048.0);
      uint16_t xb = f2h_bits(x);
      xv[i] = h2d(xb);
      B[i] = f2h_bits((float)(xv[i] * std::ldexp(1.0, -2 * j)));
    }
    cudaMemcpy(dA, A, 512, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice);
    exact_kernel<<<1, 32>>>(dA, dB, dD);
    float D[128];
    cudaMemcpy(D, dD, 512, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 16; ++r)
      for (int n = 0; n < 8; ++n) {
        double ex = 0;
        for (int k = 0; k < 16; ++k) ex += (double)code[r * 16 + k] * h2d(B[n * 16 + k]) * std::ldexp(1.0, 2 * j - 24);
        double got = D[r * 8 + n];
        double err = std::fabs(got - ex) / (std::fabs(ex) + 1e-30);
        if (got != (float)ex) ++inexact;
        if (err > worst) worst = err;
      }
  }
  printf("exactness: %d of %d outputs differ from fp32(exact), worst rel err %.3e\n", inexact, trials * 128, worst);

  // ---- throughput
  float* sink;
  cudaMalloc(&sink, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int f32 : {1, 0}) {
      auto fn = f32 ? tput_kernel<4, true> : tput_kernel<4, false>;
      fn<<<sms, warps * 32>>>(iters, sink);
      cudaEventRecord(e0);
      fn<<<sms, warps * 32>>>(iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double mmas = (double)sms * warps * iters * 4;
      double per_sm_per_ns = mmas / sms / (ms * 1e6);
      printf("HMMA.16816.%s warps/SM %2d: %.3f ms, %.3f mma/ns/SM (%.1f TFLOP/s dense-equivalent)\n",
             f32 ? "F32" : "F16", warps, ms, per_sm_per_ns, mmas * 4096.0 / (ms * 1e-3) / 1e12);
    }
  }
  printf("sms %d clock %d kHz; %s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
