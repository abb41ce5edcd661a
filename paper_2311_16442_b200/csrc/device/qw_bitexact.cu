// qw_bitexact.cu -- bit-exact decode kernels (the parity anchors).
//
//   K1 dequant  reconstruct_dense (reference engine.cpp:151-167)
//   K0 unpack   unpack_layer codes (reference bitpack.cpp:149-173)
//
// Both read the 4-row device records (qw_device.hpp) directly from HBM, one
// thread per (row, 16-channel group).  All products are exact in fp32
// (SURVEY.md H9), so the results match the reference bit for bit.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "qw_device.hpp"
#include "qw_layout.hpp"
#include "qw_ptx.cuh"

namespace qwdev {
namespace {

// ------------------------------------------------------------ K1 dequant
// One thread per (row, group); products are exact in fp32, so any
// evaluation order reproduces reconstruct_dense bit for bit.
__global__ void dequant_kernel(const uint8_t* __restrict__ quads,
                               const uint32_t* __restrict__ sorder, Geometry G,
                               float* __restrict__ w) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)G.rows * G.G) return;
  const uint32_t r = (uint32_t)(tid / G.G), g = (uint32_t)(tid % G.G);
  const uint8_t* qr = quads + (size_t)(r / kRowsPerQuad) * G.dense_bytes;
  const uint32_t i = r % kRowsPerQuad;
  float out[16];
  if (g < G.G2) {
    const uint32_t word = unpack_pair2(reinterpret_cast<const uint32_t*>(qr + 16u * g + 8u * (i >> 1)), i & 1u);
    const uint32_t t = g / 3u, sub = g - 3u * t;
    const uint32_t meta = *reinterpret_cast<const uint16_t*>(qr + G.off_meta + 8u * t + 2u * i);
    const int z = (int)((meta >> (2 * sub)) & 3u);
    const uint32_t sc = sub == 0 ? (meta >> 6) & 15u : ((meta >> (sub == 1 ? 10 : 13)) & 7u) << 1;
    const uint32_t e = sorder[(size_t)(r / G.group2) * G.G2s + g];
    const float s1 = (float)((int)sc - (int)(e >> 16)) * half_bits_to_float(e);
#pragma unroll
    for (int k = 0; k < 16; ++k) out[k] = (float)((int)((word >> (2 * k)) & 3u) - z) * s1;
  } else {
    const uint32_t b = g - G.G2;
    uint32_t w0, w1;
    unpack_pair4(reinterpret_cast<const uint32_t*>(qr + G.off_c4 + 32u * b + 16u * (i >> 1)), i & 1u, &w0, &w1);
    const float s4 = half_bits_to_float(*reinterpret_cast<const uint16_t*>(qr + G.off_s4 + 8u * b + 2u * i));
    const int z4 = (int)((*reinterpret_cast<const uint16_t*>(qr + G.off_z4 + 2u * b) >> (4 * i)) & 15u);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      out[k] = (float)((int)((w0 >> (4 * k)) & 15u) - z4) * s4;
      out[8 + k] = (float)((int)((w1 >> (4 * k)) & 15u) - z4) * s4;
    }
  }
  float4* dst = reinterpret_cast<float4*>(w + (size_t)r * G.padded_cols + 16u * g);
#pragma unroll
  for (int k = 0; k < 4; ++k) dst[k] = make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
}

// ------------------------------------------------------------ K0 unpack
__global__ void unpack_kernel(const uint8_t* __restrict__ quads, Geometry G, uint8_t* codes2,
                              uint8_t* zeros2, uint8_t* scodes, uint8_t* codes4) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)G.rows * G.G) return;
  const uint32_t r = (uint32_t)(tid / G.G), g = (uint32_t)(tid % G.G);
  const uint8_t* qr = quads + (size_t)(r / kRowsPerQuad) * G.dense_bytes;
  const uint32_t i = r % kRowsPerQuad;
  if (g < G.G2) {
    const uint32_t word = unpack_pair2(reinterpret_cast<const uint32_t*>(qr + 16u * g + 8u * (i >> 1)), i & 1u);
    const uint32_t t = g / 3u, sub = g - 3u * t;
    const uint32_t meta = *reinterpret_cast<const uint16_t*>(qr + G.off_meta + 8u * t + 2u * i);
    for (int k = 0; k < 16; ++k) codes2[(size_t)r * G.n2p + 16u * g + k] = (word >> (2 * k)) & 3u;
    zeros2[(size_t)r * G.G2 + g] = (meta >> (2 * sub)) & 3u;
    scodes[(size_t)r * G.G2 + g] = sub == 0 ? (meta >> 6) & 15u : (meta >> (sub == 1 ? 10 : 13)) & 7u;
  } else {
    const uint32_t b = g - G.G2;
    uint32_t w0, w1;
    unpack_pair4(reinterpret_cast<const uint32_t*>(qr + G.off_c4 + 32u * b + 16u * (i >> 1)), i & 1u, &w0, &w1);
    for (int k = 0; k < 8; ++k) {
      codes4[(size_t)r * G.n4 + 16u * b + k] = (w0 >> (4 * k)) & 15u;
      codes4[(size_t)r * G.n4 + 16u * b + 8 + k] = (w1 >> (4 * k)) & 15u;
    }
  }
}

}  // namespace

int launch_dequant(const DeviceLayer& L, float* w, void* stream) {
  const uint64_t n = (uint64_t)L.g.rows * L.g.G;
  const uint32_t threads = 256;
  dequant_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      L.quads, L.sorder, L.g, w);
  return (int)cudaGetLastError();
}

int launch_unpack(const DeviceLayer& L, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes,
                  uint8_t* codes4, void* stream) {
  const uint64_t n = (uint64_t)L.g.rows * L.g.G;
  const uint32_t threads = 256;
  unpack_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      L.quads, L.g, codes2, zeros2, scodes, codes4);
  return (int)cudaGetLastError();
}

}  // namespace qwdev
