/* qweight_b200_tp.h -- tensor-parallel quantized linear over NCCL (C ABI).
 *
 * SURVEY.md section 8(e) / BASELINE config 5: the layer is quantized ONCE as a
 * whole (outlier top-K, channel plan and 2-order groups are global:
 * outliers.cpp:81-97, plan.cpp:32-73) and the packed layer is sharded:
 *   QW_TP_COLUMN  rank r owns whole 2-order row blocks of the output rows
 *                 (qw_host_shard_rows); y = ncclAllGather of the shards
 *                 (Megatron q/k/v/gate/up);
 *   QW_TP_ROW     rank r owns a contiguous range of paired tiles
 *                 (qw_host_shard_tiles) and reads the matching slice of the
 *                 permuted activation; y = ncclAllReduce(sum) of the partial y
 *                 (Megatron o/down).
 * The caller owns the NCCL communicator (one rank per GPU, ncclCommInitRank)
 * and the stream; every call is asynchronous on that stream.  Library:
 * libqweight_b200_tp.so (depends on libqweight_b200.so and libnccl.so.2).
 * The reference has no distributed layer: these entries are new.
 */
#ifndef QWEIGHT_B200_TP_H
#define QWEIGHT_B200_TP_H

#include <nccl.h>
#include <stdint.h>

#include "qweight_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define QW_TP_COLUMN 0
#define QW_TP_ROW 1

typedef struct qw_tp qw_tp;

/* Shard `layer` (the whole, globally quantized layer) for `rank` of `world`
 * and upload the shard to `device` (upload_flags as qw_layer_upload_ex). */
int qw_tp_create(const qw_host_layer* layer, int rank, int world, int mode, int device,
                 uint32_t upload_flags, qw_tp** out);
/* y = W_q x across the ranks: x device fp32 [batch][cols] (original channel
 * order, identical on every rank), y device fp32 [batch][rows] (the full
 * output on every rank).  batch 1..16. */
int qw_tp_matvec(qw_tp* tp, const float* x, uint32_t batch, float* y, ncclComm_t comm, void* stream);
/* The same exchange without NCCL, fused with the GEMV over peer memory
 * (batch 1; the shard must run the SIMT kernel: create with QW_UPLOAD_SIMT).
 * Each rank allocates an exchange buffer of qw_tp_exchange_bytes and a
 * zeroed uint32 arrival counter, maps the other ranks' buffers and counters
 * (qw_ipc_handle / qw_ipc_open, NVLink P2P), and binds them in rank order;
 * `expected` is the sum over the ranks of qw_tp_arrivals.  qw_tp_matvec_peer
 * then runs qw_matvec_push into every rank's buffer, the wait on this rank's
 * counter, and (row split) the rank-order sum; y: device fp32 [rows]. */
int qw_tp_exchange_bytes(const qw_tp* tp, uint64_t* bytes);
int qw_tp_arrivals(const qw_tp* tp);
int qw_tp_bind_peers(qw_tp* tp, float* const* peer_buf, uint32_t* const* peer_flag, uint32_t expected);
int qw_tp_matvec_peer(qw_tp* tp, const float* x, float* y, void* stream);
/* Rows this rank computes (column split) or the shard's input channels (row split). */
int qw_tp_local_extent(const qw_tp* tp, uint32_t* rows, uint32_t* cols);
int qw_tp_free(qw_tp* tp);

#ifdef __cplusplus
}
#endif
#endif
