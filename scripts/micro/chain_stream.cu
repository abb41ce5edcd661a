// Microbenchmark: per-kernel time of a chain of streaming-read kernels, each
// reading its own `bytes` buffer (distinct HBM copies), captured in a CUDA
// graph, with and without programmatic dependent launch.  Gives the practical
// floor for a chain of memory-bound GEMVs of the same byte count.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512) stream_k(const uint4* __restrict__ src, size_t n16, uint32_t* out, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) { uint4 a = __ldg(src + i); acc ^= a.x; }
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (acc == 0x12345678u) out[blockIdx.x] = acc;
}
int main() {
  const int NK = 224;
  size_t sizes[] = {6884428, 18474252};
  for (size_t bytes : sizes) {
    size_t n16 = bytes / 16;
    std::vector<uint4*> bufs(NK);
    for (auto& b : bufs) { cudaMalloc(&b, n16 * 16); cudaMemset(b, 1, n16 * 16); }
    uint32_t* out; cudaMalloc(&out, 1 << 20);
    cudaStream_t st; cudaStreamCreate(&st);
    for (int grid : {148, 296, 592}) for (int thr : {256, 512}) for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < NK; ++k) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = thr; cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
        if (pdl) { cfg.attrs = at; cfg.numAttrs = 1; }
        cudaLaunchKernelEx(&cfg, stream_k, (const uint4*)bufs[k], n16, out, pdl);
      }
      cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
      cudaEventRecord(e0, st);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double us = ms * 1e3 / (10.0 * NK);
      printf("bytes %9zu grid %4d thr %3d pdl %d : %7.3f us/kernel  %7.1f GB/s  err=%s\n", bytes, grid, thr, pdl, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    for (auto& b : bufs) cudaFree(b);
  }
  return 0;
}
