// qw_peer.cu -- the local steps of the tensor-parallel exchange over peer
// memory (the collective fused with the GEMV).  The GEMV's
// epilogue (qw_gemv.cu, GemvArgs::peers) stores its y rows straight into
// every rank's buffer and adds one arrival per CTA to every rank's counter;
// a rank then waits for all arrivals (qw_peer_wait) and, for the row split,
// sums the ranks' partial slots in rank order (qw_peer_reduce).
#include <cuda_runtime.h>

#include <algorithm>

#include "qw_device.hpp"

namespace qwdev {
namespace {

// one thread: spin (acquire, system scope) until `expected` arrivals, then
// take them off the counter -- arrivals of the next launch that raced ahead
// stay counted, so the counter needs no reset and CUDA-graph replays work
__global__ void peer_wait_kernel(uint32_t* flag, uint32_t expected) {
  // the next kernel may launch (and stream its weights) now: it reads y only
  // after this grid completes (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x != 0) return;
  uint32_t seen = 0;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(flag) : "memory");
  } while (seen < expected);
  atomicSub_system(flag, expected);
}

__global__ void peer_reduce_kernel(const float* __restrict__ staging, uint32_t world, uint32_t n,
                                   float* __restrict__ y) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float s = staging[i];
    for (uint32_t r = 1; r < world; ++r) s += staging[(size_t)r * n + i];  // rank order: deterministic
    y[i] = s;
  }
}

}  // namespace

int launch_peer_wait(uint32_t* flag, uint32_t expected, void* stream) {
  // programmatic dependent launch: the wait only polls the counter, so it
  // starts under the push kernel instead of after it
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, peer_wait_kernel, flag, expected);
}

int launch_peer_reduce(const float* staging, uint32_t world, uint32_t n, float* y, void* stream) {
  if (n == 0) return 0;
  const uint32_t blocks = std::min<uint32_t>((n + 255) / 256, 592);
  peer_reduce_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(staging, world, n, y);
  return (int)cudaGetLastError();
}

}  // namespace qwdev
