// qw_tp.cu -- tensor-parallel quantized linear over NCCL (qweight_b200_tp.h).
//
// Sharding follows tp.py (the same split_rows / split_tiles rules) through the
// main library's C ABI (qw_host_shard_rows / qw_host_shard_tiles, upload,
// matvec); the exchange is one NCCL collective on the caller's communicator:
//   column split: local y -> padded [batch][max_rows] slot, ncclAllGather,
//                 then one kernel drops each rank's padding into y;
//   row split:    one gather kernel builds the shard's input slice from x
//                 (pads read 0), local partial y, ncclAllReduce(sum) into y.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "../../../include/qweight_b200.h"
#include "../../../include/qweight_b200_tp.h"

struct qw_tp {
  int mode = 0, rank = 0, world = 1, device = 0;
  qw_layer* shard = nullptr;
  qw_workspace* ws = nullptr;
  uint32_t rows = 0, cols = 0, srows = 0, scols = 0, max_rows = 0;
  std::vector<uint32_t> ranges;    // column split: [world][2] row ranges
  uint32_t* d_ranges = nullptr;    // device copy
  int32_t* d_idx = nullptr;        // row split: original channel per shard channel (-1: pad)
  float* d_xs = nullptr;           // row split: the shard's input [16][scols]
  float* d_yloc = nullptr;         // column split: [16][max_rows] padded local y
  float* d_gather = nullptr;       // column split: [world][16][max_rows]
  // peer-memory exchange (qw_tp_bind_peers)
  std::vector<float*> peer_y;      // where this rank's rows / partial go in each rank's buffer
  std::vector<uint32_t*> peer_flag;
  float* own_buf = nullptr;
  uint32_t* own_flag = nullptr;
  uint32_t expected = 0;
  ~qw_tp() {
    if (shard) qw_layer_free(shard);
    if (ws) qw_workspace_free(ws);
    cudaFree(d_ranges), cudaFree(d_idx), cudaFree(d_xs), cudaFree(d_yloc), cudaFree(d_gather);
  }
};

namespace {

__global__ void gather_cols(const float* __restrict__ x, uint32_t cols, const int32_t* __restrict__ idx,
                            uint32_t scols, uint32_t batch, float* __restrict__ xs) {
  const uint32_t n = batch * scols;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t b = i / scols, c = i - b * scols;
    const int32_t src = idx[c];
    xs[i] = src >= 0 ? x[(size_t)b * cols + src] : 0.0f;
  }
}

// y[b][row] for row in rank r's range = gathered[r][b][row - start_r]
__global__ void unpad_rows(const float* __restrict__ g, const uint32_t* __restrict__ ranges, uint32_t world,
                           uint32_t batch, uint32_t max_rows, uint32_t rows, float* __restrict__ y) {
  const uint32_t n = batch * rows;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t b = i / rows, row = i - b * rows;
    uint32_t r = 0;
    while (r + 1 < world && row >= ranges[2 * r + 1]) ++r;
    y[i] = g[((size_t)r * batch + b) * max_rows + (row - ranges[2 * r])];
  }
}

int nccl_status(ncclResult_t r) { return r == ncclSuccess ? QW_OK : QW_ERR_NCCL; }

}  // namespace

extern "C" {

int qw_tp_create(const qw_host_layer* layer, int rank, int world, int mode, int device, uint32_t upload_flags,
                 qw_tp** out) {
  if (!layer || !out || world < 1 || rank < 0 || rank >= world || (mode != QW_TP_COLUMN && mode != QW_TP_ROW))
    return QW_ERR_ARG;
  auto T = std::make_unique<qw_tp>();
  T->mode = mode, T->rank = rank, T->world = world, T->device = device;
  qw_layer_view v{};
  if (int s = qw_host_view(layer, &v)) return s;
  T->rows = v.rows, T->cols = v.cols;
  if (cudaSetDevice(device) != cudaSuccess) return QW_ERR_CUDA;
  qw_host_layer* shard = nullptr;
  if (mode == QW_TP_COLUMN) {
    // whole 2-order row blocks per rank (tp.py split_rows)
    const uint32_t blocks = (v.rows + v.group2 - 1) / v.group2;
    for (int r = 0; r < world; ++r) {
      const uint32_t b0 = blocks * r / world, b1 = blocks * (r + 1) / world;
      T->ranges.push_back(std::min(b0 * v.group2, v.rows));
      T->ranges.push_back(std::min(b1 * v.group2, v.rows));
      T->max_rows = std::max(T->max_rows, T->ranges.back() - T->ranges[T->ranges.size() - 2]);
    }
    if (int s = qw_host_shard_rows(layer, T->ranges[2 * rank], T->ranges[2 * rank + 1], &shard)) return s;
  } else {
    // a contiguous range of paired tiles (tp.py split_tiles)
    const uint32_t n2p = v.cols - v.n4 + v.pad2, tiles = n2p / 48;
    if (tiles != v.n4 / 16) return QW_ERR_UNSUPPORTED;  // row split needs paired tiles (T2 == T4)
    const uint32_t t0 = tiles * rank / world, t1 = tiles * (rank + 1) / world;
    uint32_t offs[4];
    if (int s = qw_host_shard_tiles(layer, t0, t1, &shard, offs)) return s;
    // shard channel i reads the parent's permuted slot: [2-bit lo, hi) then [4-bit lo, hi)
    std::vector<int32_t> idx;
    for (uint32_t k = offs[0]; k < offs[1]; ++k)
      idx.push_back(v.plan_perm[k] == 0xFFFFFFFFu ? -1 : (int32_t)v.plan_perm[k]);
    for (uint32_t k = offs[2]; k < offs[3]; ++k)
      idx.push_back(v.plan_perm[k] == 0xFFFFFFFFu ? -1 : (int32_t)v.plan_perm[k]);
    T->scols = (uint32_t)idx.size();
    if (cudaMalloc((void**)&T->d_idx, idx.size() * 4) != cudaSuccess ||
        cudaMemcpy(T->d_idx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc((void**)&T->d_xs, (size_t)16 * T->scols * 4) != cudaSuccess) {
      qw_host_free(shard);
      return QW_ERR_CUDA;
    }
  }
  qw_layer_view sv{};
  int s = qw_host_view(shard, &sv);
  if (!s) s = qw_layer_upload_ex(&sv, device, upload_flags, &T->shard);
  if (!s) {
    T->srows = sv.rows;
    if (mode == QW_TP_ROW && sv.cols != T->scols) s = QW_ERR_LAYER;
  }
  qw_host_free(shard);
  if (s) return s;
  if ((s = qw_workspace_create(device, std::max(T->cols, T->scols) + 64, 16, &T->ws))) return s;
  if (mode == QW_TP_COLUMN) {
    if (cudaMalloc((void**)&T->d_ranges, T->ranges.size() * 4) != cudaSuccess ||
        cudaMemcpy(T->d_ranges, T->ranges.data(), T->ranges.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc((void**)&T->d_yloc, (size_t)16 * T->max_rows * 4) != cudaSuccess ||
        cudaMemset(T->d_yloc, 0, (size_t)16 * T->max_rows * 4) != cudaSuccess ||
        cudaMalloc((void**)&T->d_gather, (size_t)world * 16 * T->max_rows * 4) != cudaSuccess)
      return QW_ERR_CUDA;
  }
  *out = T.release();
  return QW_OK;
}

int qw_tp_matvec(qw_tp* T, const float* x, uint32_t batch, float* y, ncclComm_t comm, void* stream) {
  if (!T || !x || !y || batch == 0 || batch > 16) return QW_ERR_ARG;
  cudaSetDevice(T->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (T->mode == QW_TP_COLUMN) {
    // local rows -> the padded slot [batch][max_rows] (rows beyond stay 0)
    float* ytmp = T->d_gather;  // scratch for the contiguous local result
    if (int s = qw_matvec(T->shard, x, batch, ytmp, T->ws, stream)) return s;
    if (cudaMemcpy2DAsync(T->d_yloc, (size_t)T->max_rows * 4, ytmp, (size_t)T->srows * 4, (size_t)T->srows * 4,
                          batch, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return QW_ERR_CUDA;
    const size_t slot = (size_t)batch * T->max_rows;
    if (int s = nccl_status(ncclAllGather(T->d_yloc, T->d_gather, slot, ncclFloat32, comm, st))) return s;
    unpad_rows<<<std::min<uint32_t>((batch * T->rows + 255) / 256, 1184), 256, 0, st>>>(
        T->d_gather, T->d_ranges, (uint32_t)T->world, batch, T->max_rows, T->rows, y);
  } else {
    gather_cols<<<std::min<uint32_t>((batch * T->scols + 255) / 256, 1184), 256, 0, st>>>(
        x, T->cols, T->d_idx, T->scols, batch, T->d_xs);
    if (int s = qw_matvec(T->shard, T->d_xs, batch, y, T->ws, stream)) return s;
    if (int s = nccl_status(ncclAllReduce(y, y, (size_t)batch * T->rows, ncclFloat32, ncclSum, comm, st)))
      return s;
  }
  return cudaGetLastError() == cudaSuccess ? QW_OK : QW_ERR_CUDA;
}

int qw_tp_exchange_bytes(const qw_tp* T, uint64_t* bytes) {
  if (!T || !bytes) return QW_ERR_ARG;
  *bytes = (uint64_t)4 * T->rows * (T->mode == QW_TP_COLUMN ? 1u : (uint32_t)T->world);
  return QW_OK;
}

int qw_tp_arrivals(const qw_tp* T) { return T ? qw_push_arrivals(T->shard) : -QW_ERR_ARG; }

int qw_tp_bind_peers(qw_tp* T, float* const* peer_buf, uint32_t* const* peer_flag, uint32_t expected) {
  if (!T || !peer_buf || !peer_flag || expected == 0) return QW_ERR_ARG;
  if (qw_layer_uses_tensor_core(T->shard)) return QW_ERR_UNSUPPORTED;  // the exchange runs on the SIMT kernel
  T->peer_y.clear(), T->peer_flag.clear();
  for (int r = 0; r < T->world; ++r) {
    if (!peer_buf[r] || !peer_flag[r]) return QW_ERR_ARG;
    const uint32_t off = T->mode == QW_TP_COLUMN ? T->ranges[2 * T->rank] : (uint32_t)T->rank * T->rows;
    T->peer_y.push_back(peer_buf[r] + off);
    T->peer_flag.push_back(peer_flag[r]);
  }
  T->own_buf = peer_buf[T->rank], T->own_flag = peer_flag[T->rank], T->expected = expected;
  return QW_OK;
}

int qw_tp_matvec_peer(qw_tp* T, const float* x, float* y, void* stream) {
  if (!T || !x || !y) return QW_ERR_ARG;
  if (T->peer_y.empty()) return QW_ERR_ARG;  // not bound
  cudaSetDevice(T->device);
  cudaStream_t st = (cudaStream_t)stream;
  const float* xin = x;
  if (T->mode == QW_TP_ROW) {
    gather_cols<<<std::min<uint32_t>((T->scols + 255) / 256, 1184), 256, 0, st>>>(x, T->cols, T->d_idx, T->scols,
                                                                                  1, T->d_xs);
    xin = T->d_xs;
  }
  // the shard's own result goes to scratch (the exchange buffers hold the output)
  float* ytmp = T->mode == QW_TP_COLUMN ? T->d_gather : y;
  if (int s = qw_matvec_push(T->shard, xin, ytmp, T->peer_y.data(), T->peer_flag.data(), (uint32_t)T->world, stream,
                             QW_LAUNCH_PDL))
    return s;
  if (int s = qw_peer_wait(T->own_flag, T->expected, stream)) return s;
  if (T->mode == QW_TP_COLUMN) {
    if (cudaMemcpyAsync(y, T->own_buf, (size_t)4 * T->rows, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return QW_ERR_CUDA;
  } else if (int s = qw_peer_reduce(T->own_buf, (uint32_t)T->world, T->rows, y, stream)) {
    return s;
  }
  return cudaGetLastError() == cudaSuccess ? QW_OK : QW_ERR_CUDA;
}

int qw_tp_local_extent(const qw_tp* T, uint32_t* rows, uint32_t* cols) {
  if (!T || !rows || !cols) return QW_ERR_ARG;
  *rows = T->srows, *cols = T->mode == QW_TP_ROW ? T->scols : T->cols;
  return QW_OK;
}

int qw_tp_free(qw_tp* T) {
  delete T;
  return QW_OK;
}

}  // extern "C"
