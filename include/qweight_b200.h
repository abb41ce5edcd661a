/*
 * qweight_b200.h -- C-ABI boundary of the B200 quantized-linear path.
 *
 * The reference (arXiv 2311.16442 artifact, `qweight`) exposes its hot path as
 * a C++ library API in namespace qweight; it has no FFI.  This header is the
 * thin extern "C" layer the north star asks for: plain pointers and sizes, no
 * torch or STL types, integer status codes instead of exceptions.  Each entry
 * point names the reference interface it replaces (paths are relative to the
 * reference tree, proj/...).
 *
 * Device entry points are asynchronous on the caller's stream; *_host entry
 * points are synchronous and take host buffers.  No entry point falls back to
 * a CPU implementation: a missing or failing device is reported as
 * QW_ERR_CUDA.
 */
#ifndef QWEIGHT_B200_H
#define QWEIGHT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QW_ABI_VERSION 1

/* Status codes.  The reference throws qweight::Error (types.hpp:11-14) for
 * every failure; the C++ shim (qweight_b200.hpp) maps codes back to it. */
enum qw_status {
  QW_OK = 0,
  QW_ERR_ARG = 1,         /* bad argument: length mismatch, null, non-finite
                             activation (engine.cpp:126-130), workers == 0
                             (engine.cpp:187-188) */
  QW_ERR_LAYER = 2,       /* validate_layer failed (bitpack.cpp:212-247) */
  QW_ERR_CUDA = 3,        /* CUDA runtime / launch failure, no device */
  QW_ERR_NCCL = 4,        /* collective failure */
  QW_ERR_UNSUPPORTED = 5, /* geometry outside what the kernels stage */
  QW_ERR_NOMEM = 6,
  QW_ERR_IO = 7,          /* container file I/O (container.cpp:89-110) */
  QW_ERR_FORMAT = 8       /* container corrupt (container.cpp:361-436) */
};

/* Borrowed, read-only view of a reference PackedLayer (bitpack.hpp:112-124).
 * Scalars mirror LayerConfig (bitpack.hpp:59-98); sorder / fourbit are passed
 * as structure-of-arrays because the reference structs are padded
 * (SorderParam: zero2@0 scale2@2; FourBitParam: scale@0 zero@2, sizeof 4).
 * All *_len fields are element counts.  The view is only read during the
 * call that receives it. */
typedef struct qw_layer_view {
  uint16_t n, n2, group1, group2, tile;
  uint32_t rows, cols, n4, pad2, outlier_count;
  float alpha, outlier_ratio;

  const uint8_t* plan_bits;   /* ChannelPlan.bits, cols entries (plan.hpp:37) */
  uint64_t plan_bits_len;
  const uint32_t* plan_perm;  /* ChannelPlan.perm, padded_cols (plan.hpp:38) */
  uint64_t plan_perm_len;

  const uint8_t* main;        /* rows x paired x 16 */
  uint64_t main_len;
  const uint8_t* tail2;       /* rows x tail2_blocks x 12 */
  uint64_t tail2_len;
  const uint8_t* tail4;       /* rows x tail4_blocks x 4 */
  uint64_t tail4_len;
  const uint8_t* secondary;   /* rows x blocks4 x 4 */
  uint64_t secondary_len;
  const uint16_t* meta;       /* rows x triples */
  uint64_t meta_len;
  const uint8_t* sorder_zero2;   /* row_blocks x groups_per_row */
  const uint16_t* sorder_scale2; /* fp16 bits, same count */
  uint64_t sorder_len;
  const uint16_t* fourbit_scale; /* fp16 bits, rows x blocks4 */
  const uint8_t* fourbit_zero;   /* same count */
  uint64_t fourbit_len;
  const uint32_t* csr_row_ptr;   /* rows + 1 (outliers.hpp:16-22) */
  uint64_t csr_row_ptr_len;
  const uint16_t* csr_col_ind;   /* nnz, permuted 2-bit columns */
  const uint16_t* csr_values;    /* nnz, fp16 bits */
  uint64_t csr_nnz;
} qw_layer_view;

/* Geometry + byte accounting of a layer. */
typedef struct qw_layer_info {
  uint32_t rows, cols, padded_cols, n2_padded, n4;
  uint32_t triples, blocks4, groups, group2, row_blocks;
  uint32_t quads;            /* 4-row device records */
  uint32_t quad_bytes;       /* dense bytes of one device record */
  uint64_t nnz;
  uint64_t payload_bytes;    /* reference payload_bytes (container.cpp:466-471) */
  uint64_t device_bytes;     /* bytes the device format occupies in HBM */
  uint64_t stream_bytes;     /* bytes one matvec reads from the weight format */
} qw_layer_info;

/* ------------------------------------------------------------------ errors */
const char* qw_strerror(int status);
/* Thread-local detail message of the last failing call on this thread. */
const char* qw_last_error(void);
int qw_abi_version(void);

/* --------------------------------------------------- host layer (producer)
 * The reference's producer side (quantizer.hpp:21-34, bitpack.hpp:126-127,
 * synth.hpp, container.hpp) restated natively so the B200 framework can make
 * and persist its own inputs.  Results are bit-identical to the reference. */
typedef struct qw_host_layer qw_host_layer;

/* quantize_layer (quantizer.hpp:21-22 / quantizer.cpp:132-146).
 * w: rows x cols row-major fp32; h: cols calibration norms.
 * threads: worker threads for the per-row passes (0 = hardware default). */
int qw_host_quantize(const float* w, uint32_t rows, uint32_t cols,
                     const float* h, double alpha, uint32_t group2,
                     double outlier_ratio, uint32_t threads,
                     qw_host_layer** out);
/* Copy + validate_layer a borrowed view into an owning host layer. */
/* quantize_layer with its data-parallel passes on the GPU (channel
 * amplitudes, outlier scores + top-K candidates, group fits, the 2-order
 * pass): the same host layer as qw_host_quantize, bit for
 * bit (the plan ranking, final top-K order, CSR and pack stay on the host). */
int qw_device_quantize(const float* w, uint32_t rows, uint32_t cols, const float* h,
                       double alpha, uint32_t group2, double ratio, int device,
                       qw_host_layer** out);
int qw_host_from_view(const qw_layer_view* view, qw_host_layer** out);
/* Borrowed view of an owning host layer (valid until qw_host_free). */
int qw_host_view(const qw_host_layer* layer, qw_layer_view* view);
void qw_host_free(qw_host_layer* layer);
/* QWL1 container (container.hpp:50-58). */
int qw_host_write(const qw_host_layer* layer, const char* path);
int qw_host_read(const char* path, qw_host_layer** out);
/* Row shard [r0, r1) (column-parallel TP split; r0, r1 multiples of group2
 * except r1 == rows) and tile shard [t0, t1) (row-parallel TP split over
 * paired tiles).  Shards are themselves valid layers. */
int qw_host_shard_rows(const qw_host_layer* layer, uint32_t r0, uint32_t r1,
                       qw_host_layer** out);
int qw_host_shard_tiles(const qw_host_layer* layer, uint32_t t0, uint32_t t1,
                        qw_host_layer** out, uint32_t* col_offsets /* [4]:
                        2-bit slot lo, hi, 4-bit slot lo, hi in the parent's
                        permuted space */);

/* validate_layer (bitpack.cpp:212-247) on a view. */
int qw_validate_layer(const qw_layer_view* view);
/* payload_bytes (container.cpp:466-471). */
uint64_t qw_payload_bytes(const qw_layer_view* view);
int qw_layer_view_info(const qw_layer_view* view, qw_layer_info* info);

/* synth.hpp:12-22 */
int qw_synth_gaussian(uint32_t rows, uint32_t cols, uint64_t seed, float* out);
int qw_plant_outliers(float* w, uint64_t count, double ratio, float scale,
                      uint64_t seed);
int qw_synth_calibration(uint32_t cols, uint64_t seed, float* out);
int qw_synth_activation(uint32_t cols, uint64_t seed, float* out);

/* ------------------------------------------------------- device layer (B200)
 * Upload: validate_layer, repack into the 4-row device records (DESIGN.md
 * "HBM layout"), copy to HBM.  Batch-1 calls (the fused GEMV) only read the
 * handle and may run concurrently from several streams.  Batched calls
 * (batch 2..16, the tcgen05 path) use scratch owned by the layer (B tiles,
 * CSR sums, stream-K partials and arrival counters): order them on one
 * stream (or with events) per layer. */
typedef struct qw_layer qw_layer;
typedef struct qw_workspace qw_workspace;

int qw_layer_upload(const qw_layer_view* view, int device, qw_layer** out);
/* Upload with options: which batch-1 kernel serves the layer.
 *   0 (auto, what qw_layer_upload does): the SIMT kernel K2, except where
 *     the measured shape sweep has the warp-MMA kernel
 *     K2m ahead -- layers whose outliers do not fit K2's shared-memory CSR
 *     stage (K2 then falls back to a global-memory CSR loop) and layers
 *     wider than K2's two-groups-per-lane limit (70B down_proj), and
 *     layers K2 cannot take at all (more than 60 chunks of 32 groups, or x +
 *     2-order rows + a two-slot ring beyond shared memory even at three CTAs
 *     per SM);
 *   QW_UPLOAD_TENSOR_CORE: always K2m (16-row tile format, qw_mma.cu);
 *   QW_UPLOAD_SIMT: always K2 (QW_ERR_UNSUPPORTED where K2 cannot take it).
 * Layers whose group2 is not a multiple of 16 always keep K2. */
#define QW_UPLOAD_TENSOR_CORE 1u
#define QW_UPLOAD_SIMT 2u
int qw_layer_upload_ex(const qw_layer_view* view, int device, uint32_t flags, qw_layer** out);
/* A QWL1 container (container.cpp:321-471: header, section table, CRC32)
 * straight to the device: the bytes (e.g. an mmap'ed file) are parsed,
 * CRC-checked and validated (validate_layer) on the host and repacked into
 * the device formats, with no host PackedLayer handed back to the caller.
 * QW_ERR_FORMAT for a corrupt container (deserialize_packed_layer's errors). */
int qw_layer_upload_qwl(const uint8_t* bytes, uint64_t len, int device, uint32_t flags, qw_layer** out);
/* Same from a file path (read_packed_layer, container.hpp:50-58). */
int qw_layer_load(const char* path, int device, uint32_t flags, qw_layer** out);
int qw_layer_free(qw_layer* layer);
int qw_layer_get_info(const qw_layer* layer, qw_layer_info* info);
/* 1 when batch-1 calls of the layer run K2m (the warp-MMA kernel), 0 for K2. */
int qw_layer_uses_tensor_core(const qw_layer* layer);

/* Scratch for one stream (up to max_batch columns of up to max_cols
 * channels).  The fused batch-1 kernel needs none; kept for the batched
 * path and the non-finite-activation flag. */
int qw_workspace_create(int device, uint32_t max_cols, uint32_t max_batch,
                        qw_workspace** out);
int qw_workspace_free(qw_workspace* ws);

/* matvec_oracle / matvec_pipelined (engine.hpp:31-36), batched.
 * x: device fp32 [batch][cols] in ORIGINAL channel order.
 * y: device fp32 [batch][rows].  stream: cudaStream_t (NULL = legacy).
 * batch 1..16.  Asynchronous; activations are not checked for finiteness
 * here (use qw_matvec_host for the reference's checked semantics). */
int qw_matvec(const qw_layer* layer, const float* x, uint32_t batch, float* y,
              qw_workspace* ws, void* stream);
/* Same, launched with programmatic dependent launch so the weight stream of
 * this call starts before the previous kernel on the stream finishes. */
int qw_matvec_pdl(const qw_layer* layer, const float* x, uint32_t batch,
                  float* y, qw_workspace* ws, void* stream);
/* Launch flags for qw_matvec_ex. */
#define QW_LAUNCH_PDL 1u           /* programmatic dependent launch: this call's
                                      weight stream starts under the previous
                                      kernel on the stream */
#define QW_LAUNCH_X_INDEPENDENT 2u /* x was not written by the previous kernel
                                      on the stream: no dependency wait before
                                      reading it (q/k/v, gate/up share inputs) */
/* Batched calls (batch >= 2): by default batch >= QW_GEMM_MIN_BATCH runs the
 * tcgen05 GEMM K4; smaller batches run the batch-1 kernel over the columns,
 * up to 8 columns sharing one launch (the grid split over the columns, each
 * column's result bit-identical to its own batch-1 call; the weights are
 * read from HBM about once and shared through L2).  The crossover is
 * measured (profiles/r02_batch_sweep_*.jsonl).  These flags force one or the
 * other. */
#define QW_GEMM_MIN_BATCH 6u
#define QW_LAUNCH_FORCE_GEMM 4u
#define QW_LAUNCH_FORCE_COLUMNS 8u
int qw_matvec_ex(const qw_layer* layer, const float* x, uint32_t batch, float* y,
                 qw_workspace* ws, void* stream, uint32_t flags);
/* Group launch (batch 1): up to 8 layers that read the same activation
 * (q/k/v, gate/up) in ONE fused launch -- one dependency wait, one activation
 * staging.  The layers share cols, channel split and group2; rows may differ
 * (GQA q/k/v).  The layers must outlive the group.
 * ys[i]: device fp32 [rows] output of layers[i]. */
typedef struct qw_group qw_group;
int qw_group_create(const qw_layer* const* layers, uint32_t n, qw_group** out);
int qw_group_free(qw_group* group);
int qw_group_matvec(const qw_group* group, const float* x, float* const* ys, void* stream,
                    uint32_t flags);
/* Batched group launch: x device fp32 [batch][cols], ys[i] device fp32
 * [batch][rows_i]; up to 8 / n columns of every layer share one launch (one
 * segment per (layer, column), the layers' weights read once per launch and
 * shared through L2), each output bit-identical to the layer's batch-1 call. */
int qw_group_matvec_batch(const qw_group* group, const float* x, uint32_t batch, float* const* ys,
                          void* stream, uint32_t flags);
/* Decode chains: while a launch of `layer` (or `group`) runs, its CTAs also
 * stream the packed weights of `next` (the layers of the launch that follows
 * on the stream) from HBM into L2, so HBM keeps streaming while the SMs finish
 * this launch and the next one reads L2.  A hint: results never depend on it.
 * n = 0 clears.  The next layers must outlive the setting. */
int qw_layer_set_prefetch(qw_layer* layer, const qw_layer* const* next, uint32_t n);
int qw_group_set_prefetch(qw_group* group, const qw_layer* const* next, uint32_t n);
/* Decode chain (batch 1): a fixed sequence of launch steps -- each a group of
 * 1..8 layers of identical geometry reading one activation x -- executed by
 * ONE persistent kernel: one CTA per SM streams the packed weights of all
 * steps through a single shared-memory ring (step s+1's weights land while
 * step s computes), and a step with depends != 0 reads x only after every CTA
 * stored its outputs of the previous step (a grid-wide counter replaces the
 * kernel boundary).  Buffers are bound at creation; qw_chain_run launches the
 * whole sequence (a counter reset + 1 kernel, CUDA-graph capturable).
 * Results equal the per-step launches' (qw_group_matvec / qw_matvec_ex).
 * QW_ERR_UNSUPPORTED: a step geometry the chain kernel does not cover
 * (group2 % 4 != 0, more than 16384 columns). */
typedef struct qw_chain qw_chain;
typedef struct {
  const qw_layer* const* layers; /* n layers, identical geometry */
  uint32_t n;
  const float* x;                /* device fp32 [cols], original channel order */
  float* const* ys;              /* device fp32 [rows] per layer */
  uint32_t depends;              /* x is produced by the previous step */
} qw_chain_step;
int qw_chain_create(const qw_chain_step* steps, uint32_t n, qw_chain** out);
int qw_chain_run(const qw_chain* chain, void* stream);
int qw_chain_free(qw_chain* chain);
/* Diagnostics: with QW_CHAIN_WATCH set at chain creation, a chain wait that
 * spins for seconds records {code, arg, parity, cta, thread} per warp into
 * host memory and traps; this copies those records out. */
int qw_debug_chain_watch(uint32_t* out, uint32_t n);
/* Diagnostics: per (step, CTA) 8 %globaltimer stamps of the last run of a
 * tensor-core chain planned with QW_DEBUG_MMA_TL=1 (step start, x staged,
 * items done, CSR met, dependency resolved, reduction done, counter
 * released, producer's last copy issued). */
int qw_debug_chain_timeline(const qw_chain* chain, unsigned long long* out, uint64_t n);
/* Host-buffer, synchronous, checked: length and finiteness as the reference
 * (engine.cpp:124-132).  x_len must equal batch * cols. */
int qw_matvec_host(const qw_layer* layer, const float* x, uint64_t x_len,
                   uint32_t batch, float* y, qw_workspace* ws, void* stream);
/* Same with per-stage device times (MatvecResult.stage_ns, engine.hpp:19-23):
 * stage_ns[0] = host->device copy of x, [1] = [2] = 0 (the 2-order scales and
 * the decode are fused into the kernel), [3] = the fused kernel(s).  The x / y
 * device buffers live in the workspace (grown once, reused). */
int qw_matvec_host_ex(const qw_layer* layer, const float* x, uint64_t x_len, uint32_t batch,
                      float* y, qw_workspace* ws, void* stream, uint64_t* stage_ns);

/* reconstruct_dense (engine.hpp:26): w device fp32 [rows][padded_cols],
 * permuted order, bit-exact with the reference. */
int qw_dequant(const qw_layer* layer, float* w, void* stream);
/* Same with a host buffer of rows * padded_cols floats, synchronous. */
int qw_dequant_host(const qw_layer* layer, float* w, uint64_t w_len);
/* unpack_layer (bitpack.hpp:128): device u8 outputs
 * codes2 [rows][n2_padded], zeros2 [rows][groups_per_row],
 * scodes [rows][groups_per_row], codes4 [rows][n4]. */
int qw_unpack(const qw_layer* layer, uint8_t* codes2, uint8_t* zeros2,
              uint8_t* scodes, uint8_t* codes4, void* stream);

/* Device-to-device copy of an uploaded layer (same device). */
int qw_layer_clone(const qw_layer* layer, qw_layer** out);

/* Diagnostics: one batch-1 matvec that records qw_debug_timeline_events()
 * stamps per CTA into device buffer `stamps` (grid x events):
 * 0 entry, 1 all weight copies issued, 2 activation prologue done,
 * 3 first unit landed, 4 consumers done, 5 y written, 6 outliers done.
 * flags: bit 0 = launch with programmatic dependent launch, bit 1 = stamp
 * %globaltimer (ns, comparable across SMs and kernels) instead of clock64,
 * bit 2 = x independent of the preceding kernel (no dependency wait).
 * repeat > 1 makes the consumers re-run the resident quads (compute-rate
 * measurement; y is then not meaningful). */
int qw_debug_timeline(const qw_layer* layer, const float* x, float* y,
                      unsigned long long* stamps, uint32_t repeat, uint32_t flags,
                      void* stream);
int qw_debug_timeline_events(void);
/* Same for a group launch (flags as qw_debug_timeline). */
int qw_debug_group_timeline(const qw_group* group, const float* x, float* const* ys,
                            unsigned long long* stamps, uint32_t flags, void* stream);
/* Diagnostics: one batched (K4) matvec stamping %globaltimer per CTA into
 * stamps [grid][8]: 0 setup, 1 first A tile, 2 last A tile, 3 accumulator
 * ready, 4 epilogue staged, 5 split partials parked, 6 y stored. */
int qw_debug_gemm_timeline(const qw_layer* layer, const float* x, uint32_t batch, float* y,
                           unsigned long long* stamps, void* stream);

/* Number of kernels one qw_matvec call launches. */
int qw_launches_per_matvec(const qw_layer* layer, uint32_t batch);
int qw_launches_per_matvec_ex(const qw_layer* layer, uint32_t batch, uint32_t flags);
/* Tensor parallel over peer memory (the collective fused with
 * the GEMV; NVLink P2P between GPUs, CUDA IPC mappings between processes).
 * qw_matvec_push: y = W_q x (batch 1, the SIMT kernel: upload with
 * QW_UPLOAD_SIMT) and the kernel's epilogue also stores the rows into
 * peer_y[i] (the caller offsets each pointer to where this rank's rows go),
 * then every CTA adds 1 to *peer_flag[i] (system scope, after a release).
 * qw_push_arrivals: the arrivals one push adds to each peer's counter (its
 * grid).  qw_peer_wait: stream-ordered wait until *flag >= expected (the
 * sum of the ranks' arrivals), which then takes `expected` off the counter
 * (no reset needed; CUDA-graph capturable).  qw_peer_reduce: y[i] =
 * sum_r staging[r * n + i] in rank order (the row split's partial sums).
 * qw_ipc_*: 64-byte CUDA IPC handles of device buffers for the exchange. */
int qw_matvec_push(const qw_layer* layer, const float* x, float* y, float* const* peer_y,
                   uint32_t* const* peer_flag, uint32_t npeer, void* stream, uint32_t flags);
int qw_push_arrivals(const qw_layer* layer);
int qw_peer_wait(uint32_t* flag, uint32_t expected, void* stream);
int qw_peer_reduce(const float* staging, uint32_t world, uint32_t n, float* y, void* stream);
int qw_ipc_handle(const void* dev_ptr, uint8_t handle[64]);
int qw_ipc_open(const uint8_t handle[64], void** dev_ptr);
int qw_ipc_close(void* dev_ptr);
/* 1 if a qw_matvec_ex call of `batch` columns with `flags` runs the tcgen05
 * GEMM K4, 0 if it runs the batch-1 kernel over the columns; < 0 on error. */
int qw_matvec_uses_gemm(const qw_layer* layer, uint32_t batch, uint32_t flags);
/* Diagnostics: the power of two P of the batched path's fp16 A tiles (each
 * element is RN_fp16(w * 2^-P), w the reconstruct_dense weight). */
int qw_debug_gemm_shift(const qw_layer* layer, int* shift);
/* Diagnostic knobs (QW_NQ1, QW_GEMM_KS, ... DESIGN.md section 6): the value
 * the library uses for `name` -- the environment is consulted only when
 * QW_DEBUG_KNOBS=1, otherwise every knob is its default. */
uint32_t qw_debug_knob(const char* name, uint32_t dflt);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* QWEIGHT_B200_H */
