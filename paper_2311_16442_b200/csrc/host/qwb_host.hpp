// qwb_host.hpp -- host-side types and producer of the B200 quantized-linear
// framework.
//
// These restate the reference's host API (namespace qweight in the artifact
// of arXiv 2311.16442) in namespace qwb so both libraries can be loaded into
// one process.  Type and function names follow the reference so callers and
// tests read the same; every function cites the reference function whose
// results it reproduces bit for bit.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace qwb {

// qweight::Error (types.hpp:11-14)
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// plan.hpp:12-17 -- fixed by the tile format
constexpr uint32_t kPad = 0xFFFFFFFFu;        // kPadChannel
constexpr uint32_t kG1 = 16;                  // kGroupSize
constexpr uint32_t kTile = 64;                // kTileChannels
constexpr uint32_t kTile2 = 48;               // kTileTwoBit
constexpr uint32_t kTile4 = 16;               // kTileFourBit
constexpr uint32_t kMaxSlots = 65536;         // kMaxPackedChannels

// types.hpp:16-26
struct WeightMatrix {
  uint32_t rows = 0, cols = 0;
  std::vector<float> data;
  float at(uint32_t r, uint32_t c) const { return data[(size_t)r * cols + c]; }
  float& at(uint32_t r, uint32_t c) { return data[(size_t)r * cols + c]; }
  bool valid() const { return data.size() == (size_t)rows * cols; }
};

// plan.hpp:31-42
struct ChannelPlan {
  uint32_t in_channels = 0, n4 = 0, pad2 = 0;
  std::vector<uint8_t> bits;
  std::vector<uint32_t> perm;
  uint32_t n2() const { return in_channels - n4; }
  uint32_t n2_padded() const { return n2() + pad2; }
  uint32_t padded_channels() const { return n2_padded() + n4; }
};

// outliers.hpp:16-22
struct CsrOutliers {
  std::vector<uint32_t> row_ptr;
  std::vector<uint16_t> col_ind, values;
  uint32_t nnz() const { return row_ptr.empty() ? 0u : row_ptr.back(); }
};

// bitpack.hpp:46-57 (kept as the reference's in-memory structs)
struct SorderParam {
  uint8_t zero2 = 0;
  uint16_t scale2 = 0;
};
struct FourBitParam {
  uint16_t scale = 0;
  uint8_t zero = 0;
};

// bitpack.hpp:59-98
struct LayerConfig {
  uint16_t n = 2, n2 = 4, group1 = 16, group2 = 16, tile = 64;
  uint32_t rows = 0, cols = 0, n4 = 0, pad2 = 0, outlier_count = 0;
  float alpha = 0.0f, outlier_ratio = 0.0f;

  uint32_t n2_padded() const { return cols - n4 + pad2; }
  uint32_t padded_cols() const { return n2_padded() + n4; }
  uint32_t triples() const { return n2_padded() / kTile2; }
  uint32_t blocks4() const { return n4 / kTile4; }
  uint32_t paired() const { return triples() < blocks4() ? triples() : blocks4(); }
  uint32_t tail2_blocks() const { return triples() - paired(); }
  uint32_t tail4_blocks() const { return blocks4() - paired(); }
  uint32_t groups_per_row() const { return 3 * triples(); }
  uint32_t row_blocks() const { return (rows + group2 - 1) / group2; }
  uint64_t main_bytes() const { return (uint64_t)rows * paired() * 16; }
  uint64_t tail2_bytes() const { return (uint64_t)rows * tail2_blocks() * 12; }
  uint64_t tail4_bytes() const { return (uint64_t)rows * tail4_blocks() * 4; }
  uint64_t secondary_bytes() const { return (uint64_t)rows * blocks4() * 4; }
  uint64_t meta_count() const { return (uint64_t)rows * triples(); }
  uint64_t sorder_count() const { return (uint64_t)row_blocks() * groups_per_row(); }
  uint64_t fourbit_count() const { return (uint64_t)rows * blocks4(); }
};

// bitpack.hpp:103-110
struct LayerGroups {
  std::vector<uint8_t> codes2, zeros2, scodes;
  std::vector<SorderParam> sorder;
  std::vector<uint8_t> codes4;
  std::vector<FourBitParam> fourbit;
};

// bitpack.hpp:112-124
struct PackedLayer {
  LayerConfig cfg;
  ChannelPlan plan;
  std::vector<uint8_t> main, tail2, tail4, secondary;
  std::vector<uint16_t> meta;
  std::vector<SorderParam> sorder;
  std::vector<FourBitParam> fourbit;
  CsrOutliers csr;
};

// quantizer.hpp:13-17
struct QuantizeParams {
  double alpha = 0.25;
  uint32_t group2 = 16;
  double outlier_ratio = 0.002;
};

struct SlotRef {
  uint32_t row = 0, col = 0;
};

// ---------------------------------------------------------------- numerics
uint16_t f32_to_f16(float f);  // fp16.cpp:8-38
float f16_to_f32(uint16_t h);  // fp16.cpp:40-64

struct ScaleZero {
  float scale = 1.0f;
  uint8_t zero = 0;
};
ScaleZero fit_scale_zero(std::span<const float> v, int bits);  // quant.cpp:18-52
void quantize_values(std::span<const float> v, float scale, uint8_t zero,
                     int bits, uint8_t* codes);                 // quant.cpp:54-68
inline float dequantize_one(uint8_t code, uint8_t zero, float scale) {
  return (float)((int)code - (int)zero) * scale;                // quant.hpp:30-32
}
inline float dequantize_scale(uint8_t code, uint8_t zero2, uint16_t scale2) {
  return (float)((int)code - (int)zero2) * f16_to_f32(scale2);  // quant.hpp:55-57
}

// ---------------------------------------------------------------- producer
WeightMatrix synth_gaussian(uint32_t rows, uint32_t cols, uint64_t seed);
void plant_outliers(std::span<float> w, double ratio, float scale, uint64_t seed);
std::vector<float> synth_calibration(uint32_t cols, uint64_t seed);
std::vector<float> synth_activation(uint32_t cols, uint64_t seed);

ChannelPlan build_plan_from(const WeightMatrix& w, std::span<const float> h,
                            double alpha, unsigned threads);
ChannelPlan plan_from_amplitudes(const std::vector<double>& amp, uint32_t ic, double alpha);
// quantize_layer with its data-parallel passes on the GPU (qwb_gpu_producer.cpp,
// qw_quantize.cu): bit-identical to quantize_layer.
PackedLayer quantize_layer_gpu(const float* w, uint32_t rows, uint32_t cols, std::span<const float> h,
                               const QuantizeParams& p, int device);
PackedLayer quantize_layer(const WeightMatrix& w, std::span<const float> h,
                           const QuantizeParams& p, unsigned threads);
PackedLayer pack_layer(const LayerConfig& cfg, const ChannelPlan& plan,
                       const LayerGroups& g, CsrOutliers csr);

// ---------------------------------------------------------------- format
void validate_plan(const ChannelPlan& plan);   // plan.cpp:75-105
void validate_layer(const PackedLayer& layer); // bitpack.cpp:212-247
uint64_t payload_bytes(const LayerConfig& cfg, uint64_t nnz);  // container.cpp:466-471
std::vector<uint8_t> serialize_layer(const PackedLayer& layer);      // container.cpp:321-359
PackedLayer deserialize_layer(std::span<const uint8_t> bytes);       // container.cpp:361-436
uint32_t crc32(std::span<const uint8_t> bytes);

PackedLayer shard_rows(const PackedLayer& layer, uint32_t r0, uint32_t r1);

}  // namespace qwb
namespace qwdev { struct MmaGeometry; }
namespace qwb {
// Tile format of the tensor-core batch-1 kernel (qwb_mma.cpp, qw_device.hpp).
void repack_mma(const PackedLayer& layer, const qwdev::MmaGeometry& m, float s_scale,
                std::vector<uint8_t>& out);
PackedLayer shard_tiles(const PackedLayer& layer, uint32_t t0, uint32_t t1);

// Parallel helper: run fn(begin, end) over [0, n) in at most `threads` chunks.
template <class F>
void parallel_for(uint64_t n, unsigned threads, F&& fn);

}  // namespace qwb

#include "qwb_parallel.inl"
