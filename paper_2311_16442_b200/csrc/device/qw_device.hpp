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
// (original channel of the permuted col, fp16 value) fused into one u32
// (channel | fp16 << 16) next to the original
// row_ptr.
#pragma once

#include <cstdint>
#include <cstdlib>

namespace qwdev {

// Diagnostic knobs (QW_NQ1, QW_WIDE, QW_GEMM_KS, ...): read from the
// environment ONLY when QW_DEBUG_KNOBS=1 is set; otherwise every knob is its
// default -- the product's behaviour does not depend on the environment
// (tests/test_boundary.py pins this).
inline const char* knob_str(const char* name) {
  const char* gate = std::getenv("QW_DEBUG_KNOBS");
  if (!gate || gate[0] != '1') return nullptr;
  return std::getenv(name);
}
inline uint32_t knob(const char* name, uint32_t dflt) {
  const char* e = knob_str(name);
  return e ? (uint32_t)std::atoi(e) : dflt;
}

constexpr int kRowsPerQuad = 4;

struct Geometry {
  uint32_t rows, cols, padded_cols, n2p, n4;
  uint32_t T2, T4, G2, G, G2s;  // G = G2 + T4 groups per row; G2s = padded sorder stride
  uint32_t group2, row_blocks, quads;
  uint32_t off_c4, off_meta, off_s4, off_z4, dense_bytes;  // quad record layout
  uint32_t max_rb_per_quad;  // 2-order row blocks one quad can touch
  uint64_t nnz;
};

// Launch plan of the fused GEMV, fixed at upload so launches stay
// capture-safe (no attribute calls on the launch path).
constexpr uint32_t kMaxGrid = 448;

struct GemvPlan {
  uint32_t grid = 0;                   // CTAs (persistent, contiguous quad ranges)
  uint32_t warps = 0, warps2 = 0, teams = 1, kmax = 0;  // consumer warps, 32-group chunks per warp
  bool wide = false;  // W > 8 warps of KG = 2 (wide layers): one CTA per SM, the 576-thread kernel
  uint32_t nslot = 0, uq = 2, win = 0;  // slots, quads per slot, quads per reduction window
  uint32_t nchunks = 0, nq_max = 0, uniform_rb = 0, xsm = 0, rb_magic = 0, rb_one = 0;
  float s_scale = 1.0f;  // 2^-P applied to 2-bit s1 so 15 * max scale2 * 2^-P fits fp16
  uint32_t so_off = 0, part_off = 0, xg_off = 0, misc_off = 0, win_off = 0, pre_off = 0, bar_off = 0;  // smem layout
  uint32_t ent_off = 0, csr_stage = 0;  // CSR entries staged in shared memory (when they fit)
  uint32_t smem = 0;
  uint32_t pre = 1, npre_max = 0, x_first = 0, x_gate = 0, pf_late = 1;  // launch policy (plan_ctas)
  // decode chains: the next launch's packed weights (quad records, 2-order
  // rows), streamed into L2 by this launch's CTAs (one slice each) so HBM
  // keeps streaming while the SMs are still busy with this launch
  static constexpr uint32_t kMaxPf = 8;
  const uint8_t* pf_ptr[kMaxPf] = {};
  uint32_t pf_bytes[kMaxPf] = {};
  uint32_t pf_n = 0;
  // per CTA: layer (segment) of a group launch, quad range, CSR entry range
  uint8_t cta_seg[kMaxGrid] = {};
  uint32_t cta_q0[kMaxGrid] = {}, cta_q1[kMaxGrid] = {}, cta_e0[kMaxGrid] = {}, cta_e1[kMaxGrid] = {};
};

// A group launch: up to kMaxSeg layers of identical geometry that read the
// same activation (q/k/v, gate/up); the CTAs are split across the layers in
// proportion to their quads and each CTA owns a quad range of one layer, so
// the dependency wait, the activation staging and the launch are paid once.
constexpr uint32_t kMaxSeg = 8;

// Batched (2..16 columns) tensor-core plan: 128-row M tiles x KS K splits of
// 2-tile stages (96 2-bit + 32 4-bit channels); TMA 2-D boxes of the quad
// records; 1st-order scales applied while dequantizing into the A tile.
struct GemmPlan {
  uint32_t ok = 0;           // layer geometry supported (paired tiles, group2 % 4 == 0)
  uint32_t tiles = 0, ks = 1, stages = 0, wstages = 0;  // M tiles, K splits, 2-tile sub-stages and 8-tile weight stages per row
  int shift = 0;             // A tile holds w * 2^-shift (keeps fp16 scales in range)
  alignas(64) uint8_t tmap[5][128];  // CUtensorMap: code2, meta, code4, s4, z4 boxes
  alignas(64) uint8_t tmap_so[128];  // CUtensorMap: sorder box of a tile's row blocks
  uint32_t so_rows = 0;
  uint32_t stream = 0, W = 0, C = 0, kmax = 0;  // stream-K: W weight stages over C CTAs, kmax partial slots per tile
  float* partial = nullptr;  // [tiles][kmax][128][16] stream-K partial sums
  uint32_t* counters = nullptr;  // [tiles] split-K arrivals (self-resetting)
  uint16_t* xpt = nullptr;   // [stages][128 k][16 n] fp16 B tiles (UMMA K-major layout)
  int* xexp = nullptr;       // [16] per-column power-of-two exponents
  float* ycsr = nullptr;     // [16][rows] CSR outlier sums of the call
};

// ------------------------------------------------------------ K2m (batch 1, warp MMA)
// Tile format of the tensor-core batch-1 kernel (qw_mma.cu).  Rows are taken
// 16 at a time (one m16n8k16 M tile); the row's channel groups are taken 8 at
// a time ("blocks": the 8 N columns of the MMA, one group per column, the B
// operand block-diagonal in x).  2-bit groups go in super-blocks of 8 triples
// (24 groups, 3 blocks) so a lane's 6 groups are exactly 2 meta words; 4-bit
// blocks of 16 channels go 8 to a block.  A row tile's blocks are cut into
// chunks of at most 32 (16 consumer warps x 2 blocks, the B fragments stay in
// registers); one (tile, chunk) record is one contiguous TMA copy:
//   2-bit block: [SB header: meta 32 lanes x 2 u32 | sorder 3 b x 4 t x 2 u32]
//                (the first time the chunk touches the super-block), then
//                codes 32 lanes x 4 u32 (E_g, E_g+8, O_g, O_g+8)
//   4-bit block: codes 32 lanes x 8 u32, s4 32 lanes x 2 u32, z4 32 lanes x u16
// Lane (g, t) of a block owns rows {g, g+8} and columns {2t, 2t+1}.
#ifndef QW_MMA_NW
#define QW_MMA_NW 16
#endif
constexpr uint32_t kMmaMaxChunks = 16, kMmaMaxBlk = 32;
constexpr uint32_t kMmaChunkBlk = 2 * QW_MMA_NW;  // blocks per chunk: consumer warps x 2
constexpr uint32_t kMmaHdr2 = 352, kMmaCode2 = 512, kMmaCode4 = 1024, kMmaS4 = 256, kMmaZ4 = 64;
struct MmaChunk {
  uint32_t nblk = 0, rec_bytes = 0;
  uint8_t kind[kMmaMaxBlk] = {};   // 0..2: 2-bit block b of a super-block, 3: 4-bit
  uint16_t grp[kMmaMaxBlk] = {};   // super-block (2-bit) / 8-block index (4-bit)
  uint32_t code_off[kMmaMaxBlk] = {}, hdr_off[kMmaMaxBlk] = {};
};
struct MmaGeometry {
  uint32_t ok = 0;                  // layer supported (group2 % 16 == 0, <= kMmaMaxChunks chunks)
  uint32_t RT = 0, SB = 0, B4 = 0, nchunks = 0, rec_stride = 0;
  MmaChunk chunk[kMmaMaxChunks];
};
struct MmaPlan {
  uint32_t grid = 0, nslot = 0, smem = 0, items_max = 0;
  uint32_t x_off = 0, part_off = 0, csr_off = 0, ent_off = 0, csr_slot = 0, csr_nslot = 4, rp_off = 0, bst_off = 0, bar_off = 0;
  uint8_t cta_seg[kMaxGrid] = {};
  uint32_t cta_i0[kMaxGrid] = {}, cta_i1[kMaxGrid] = {};
  uint32_t cta_e0[kMaxGrid] = {}, cta_e1[kMaxGrid] = {};  // CSR entries of the CTA's chunk-0 rows
};

struct DeviceLayer {
  Geometry g;
  GemvPlan plan;
  GemmPlan gemm;
  MmaGeometry mg;
  MmaPlan mplan;
  GemvPlan cplan[kMaxSeg - 1];    // column launches of 2..kMaxSeg columns (grid 0: not planned)
  MmaPlan mcplan[kMaxSeg - 1];
  uint8_t* mrecs = nullptr;       // RT x nchunks records (chunk-major), rec_stride apart
  float* mpart = nullptr;         // per column slot (kMaxSeg): [nchunks][RT*16] chunk partials, [RT*16] CSR sums
  uint32_t* mcnt = nullptr;       // per column slot: [RT] chunk arrivals (self-resetting)
  uint8_t* quads = nullptr;      // quads * dense_bytes
  uint32_t* sorder = nullptr;    // row_blocks * G2s
  uint32_t* perm = nullptr;      // padded_cols (0xFFFFFFFF = pad)
  uint16_t* perm16 = nullptr;    // padded_cols, original channel (pads: cols, a zero slot of the staged x)
  uint32_t* row_ptr = nullptr;   // rows + 1
  uint32_t* csr = nullptr;       // nnz (perm[col] | fp16 << 16): x channel + value
};

// Fused exchange over peer memory (tensor parallel, batch 1): besides its own
// y, a launch stores its rows into every peer's buffer (NVLink P2P or
// same-device IPC mappings, offset by the caller) and each CTA then adds 1 to
// every peer's arrival counter (system scope, after a release fence).
constexpr uint32_t kMaxPeer = 8;
struct PeerOut {
  float* y[kMaxPeer];
  uint32_t* flag[kMaxPeer];
  uint32_t n;
};

// Per-stream scratch (kept in the ABI for the batched path; the fused
// batch-1 kernel needs none).
struct Workspace {
  int device = 0;
  uint32_t max_cols = 0, max_batch = 0;
  uint32_t* flags = nullptr;
};

// Geometry-dependent part of a batch-1 plan (warps, groups per lane, quads
// per slot, wide/x-staging decisions); cudaErrorInvalidConfiguration if too wide.
int plan_geometry(GemvPlan& p, const Geometry& G);
// Launchers (return cudaError_t as int).
// Fill L.plan for a device with num_sms SMs (returns cudaError_t).
int plan_gemv(DeviceLayer& L, int num_sms, const uint32_t* host_row_ptr);
// Plan a group launch over layers[0..n) (identical geometry); returns
// cudaError_t, cudaErrorInvalidValue when the geometries differ.
int plan_gemv_group(GemvPlan& p, const DeviceLayer* const* layers, const uint32_t* const* host_row_ptrs,
                    uint32_t n, int num_sms);
int launch_gemv_group(const GemvPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* x,
                      float* const* ys, void* stream, bool pdl, uint32_t flags);
int launch_gemv_group(const GemvPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* const* xs,
                      float* const* ys, void* stream, bool pdl, uint32_t flags, unsigned long long* dbg,
                      uint32_t repeat, bool global_clock, const PeerOut* peers = nullptr);
// peer-memory exchange kernels (qw_peer.cu): wait until *flag >= expected,
// then take `expected` off it (arrivals of a later launch stay counted)
int launch_peer_wait(uint32_t* flag, uint32_t expected, void* stream);
// y[i] = sum_{r < world} staging[r * n + i] in rank order (a P2P all-reduce's local step)
int launch_peer_reduce(const float* staging, uint32_t world, uint32_t n, float* y, void* stream);
// Batch of 2..16 columns on the batch-1 kernel of the layer (K2 or K2m): the
// columns go kMaxSeg to a launch, one grid split over them like a layer
// group (each segment its own x and y, the same weights, read once from HBM
// and shared through L2).  Plans: plan_columns at upload (cplan / mcplan).
int plan_columns(DeviceLayer& L, int num_sms, const uint32_t* host_row_ptr);
int launch_columns(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream, bool pdl,
                   uint32_t flags);
uint32_t column_launches(const DeviceLayer& L, uint32_t batch);
// y[col] = W_q x[col] for col < batch: one fused kernel per column.
constexpr uint32_t kTimelineEvents = 12;  // entry, copies issued, prologue, first quad, consumers, y, csr
// flags: kXIndependent = x was not written by the preceding kernel on the
// stream (skip the programmatic-dependency wait before reading it)
constexpr uint32_t kXIndependent = 2u;
int launch_gemv(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream,
                bool pdl, unsigned long long* dbg = nullptr, uint32_t repeat = 1,
                bool global_clock = false, uint32_t flags = 0);
int launch_dequant(const DeviceLayer& L, float* w, void* stream);
// Batched path (K4): plan at upload (allocates the layer's split-K scratch),
// launch = x prologue + tcgen05 GEMM.  free_gemm releases the scratch.
int plan_gemm(DeviceLayer& L, int num_sms, float max_scale2, float max_s4);
void free_gemm(DeviceLayer& L);
int launch_gemm(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream,
                unsigned long long* dbg = nullptr);  // 3 launches: x prologue, CSR, GEMM
int launch_unpack(const DeviceLayer& L, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes,
                  uint8_t* codes4, void* stream);

// K2m: geometry of the tile format (host, no CUDA calls); plan the CTA item
// ranges of a single layer or a group of layers (identical columns); launch.
void mma_geometry(MmaGeometry& m, const Geometry& g);
int plan_mma(MmaPlan& p, const DeviceLayer* const* layers, const uint32_t* const* host_row_ptrs, uint32_t n,
             int num_sms);
int launch_mma(const MmaPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* x,
               float* const* ys, void* stream, bool pdl, uint32_t flags);
// segment s reads xs[s]; slots (or null: slot 0): segment s uses its layer's
// chunk-partial scratch slot slots[s] (< kMaxSeg; distinct for the columns of one layer)
int launch_mma(const MmaPlan& p, const DeviceLayer* const* layers, uint32_t n, const float* const* xs,
               float* const* ys, void* stream, bool pdl, uint32_t flags, const uint32_t* slots,
               unsigned long long* dbg = nullptr);

// Decode chain (batch 1): a sequence of launch steps (each a group of 1..4
// layers of identical geometry reading one activation) run by ONE persistent
// kernel -- one CTA per SM streams the weights of step s+1 into its ring
// while step s computes; a step that depends on its predecessor waits on a
// grid-wide completion counter instead of a kernel boundary.
struct ChainStepDesc {
  const DeviceLayer* const* layers;
  const uint32_t* const* host_row_ptrs;
  uint32_t n;
  const float* x;     // device fp32 [cols]
  float* const* ys;   // device fp32 [rows] per layer
  uint32_t depends;   // x is produced by the previous step: wait for it
};
struct ChainPlan;
// cudaErrorInvalidValue: a step's layers differ in geometry;
// cudaErrorNotSupported: a geometry the chain kernel does not cover.
int plan_chain(ChainPlan** out, const ChainStepDesc* steps, uint32_t n, int num_sms);
int launch_chain(const ChainPlan* p, void* stream);
void free_chain(ChainPlan* p);
const unsigned* chain_watch();
// The same decode chain on the K2m tile format (every layer uploaded with
// it): one persistent tensor-core kernel; cudaErrorNotSupported otherwise.
struct MmaChainPlan;
int plan_mma_chain(MmaChainPlan** out, const ChainStepDesc* steps, uint32_t n, int num_sms);
int launch_mma_chain(const MmaChainPlan* p, void* stream);
void free_mma_chain(MmaChainPlan* p);
// diagnostics: [step][cta][8] %globaltimer stamps of the last run (QW_DEBUG_MMA_TL=1 at plan time)
int mma_chain_timeline(const MmaChainPlan* p, unsigned long long* out, size_t n);  // diagnostics (QW_CHAIN_WATCH): [cta][warp][8] hang records, host memory

}  // namespace qwdev
