// qw_device.hpp -- device format of a packed layer and the launch API of the
// sm_100a kernels.  Host code (capi.cpp) fills these structs; the kernels in
// qw_kernels.cu consume them.
//
// HBM layout: rows are grouped in 4-row "quads".
// One quad record is contiguous so a single cp.async.bulk brings it to
// shared memory; inside it every field is interleaved over the 4 rows so one
// lane's 128-bit shared load returns the same group of all 4 rows:
//
//   code2 [G2][4] u32      2-bit group g of rows 0..3 (16 codes, code k at
//                          bits 2k: the reference's main/tail2 bytes 4*sub..)
//   code4 [T4][2][4] u32   4-bit block b: word 0 (codes 0-7, reference main
//                          bytes 12-15 / tail4), word 1 (codes 8-15,
//                          secondary); nibble n at bits 4n
//   meta  [T2][4] u16      reference meta words
//   s4    [T4][4] u16      fp16 scale of each 4-bit block
//   z4    [T4] u16         4-bit zero of rows 0..3 at bits 4i
//
// sorder is kept per 2-order row block as u32 (scale2 | zero2 << 16) with
// the row stride padded to 16 bytes.  Outliers are the reference CSR with
// col/value fused into one u32 (col | fp16 << 16) next to the original
// row_ptr.
#pragma once

#include <cstdint>

namespace qwdev {

constexpr int kRowsPerQuad = 4;

struct Geometry {
  uint32_t rows, cols, padded_cols, n2p, n4;
  uint32_t T2, T4, G2, G, G2s;  // G = G2 + T4 groups per row; G2s = padded sorder stride
  uint32_t group2, row_blocks, quads;
  uint32_t off_c4, off_meta, off_s4, off_z4, dense_bytes;  // quad record layout
  uint32_t max_rb_per_quad;  // 2-order row blocks one quad can touch
  uint64_t nnz;
};

struct DeviceLayer {
  Geometry g;
  uint8_t* quads = nullptr;      // quads * dense_bytes
  uint32_t* sorder = nullptr;    // row_blocks * G2s
  uint32_t* perm = nullptr;      // padded_cols (0xFFFFFFFF = pad)
  uint32_t* row_ptr = nullptr;   // rows + 1
  uint32_t* csr = nullptr;       // nnz (col | fp16 << 16)
};

// Activation prologue output for one column (the "xprep" block): per group
// 16 fp16 x' in the lane pairing the unpack uses, then sum(x') and the
// power-of-two unscale factor per group; followed by the permuted fp32 x.
struct XprepLayout {
  uint32_t groups;
  uint32_t xh_bytes() const { return groups * 32u; }
  uint32_t block_bytes() const { return (groups * 40u + 15u) & ~15u; }  // xh | sx | ex
};

struct Workspace {
  int device = 0;
  uint32_t max_cols = 0, max_batch = 0;
  uint8_t* xprep = nullptr;    // max_batch * block_bytes(max groups)
  float* xp = nullptr;         // max_batch * max padded cols
  uint32_t* flags = nullptr;   // non-finite activation flag
  uint32_t block_stride = 0, xp_stride = 0;
};

// Launchers (return cudaError_t as int).
int launch_prologue(const DeviceLayer& L, const float* x, uint32_t batch, const Workspace& ws,
                    void* stream, bool pdl);
int launch_gemv(const DeviceLayer& L, uint32_t batch, float* y, const Workspace& ws, void* stream,
                bool pdl, int num_sms);
int launch_dequant(const DeviceLayer& L, float* w, void* stream);
int launch_unpack(const DeviceLayer& L, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes,
                  uint8_t* codes4, void* stream);

}  // namespace qwdev
