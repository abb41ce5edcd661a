// capi.cpp -- extern "C" implementation of include/qweight_b200.h.
//
// Converts between the borrowed qw_layer_view and the host PackedLayer,
// repacks a validated layer into the 4-row device records (qw_device.hpp),
// owns device memory, and maps every failure to a status code plus a
// thread-local message.  Nothing here computes y on the CPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/qweight_b200.h"
#include "device/qw_device.hpp"
#include "device/qw_layout.hpp"
#include "host/qwb_host.hpp"

struct qw_host_layer {
  qwb::PackedLayer L;
  // structure-of-arrays mirrors for views
  std::vector<uint8_t> sorder_zero2, fourbit_zero;
  std::vector<uint16_t> sorder_scale2, fourbit_scale;
  void refresh_soa() {
    sorder_zero2.resize(L.sorder.size());
    sorder_scale2.resize(L.sorder.size());
    for (size_t i = 0; i < L.sorder.size(); ++i)
      sorder_zero2[i] = L.sorder[i].zero2, sorder_scale2[i] = L.sorder[i].scale2;
    fourbit_zero.resize(L.fourbit.size());
    fourbit_scale.resize(L.fourbit.size());
    for (size_t i = 0; i < L.fourbit.size(); ++i)
      fourbit_zero[i] = L.fourbit[i].zero, fourbit_scale[i] = L.fourbit[i].scale;
  }
};

struct qw_layer {
  qwdev::DeviceLayer dev;
  int device = 0;
  int num_sms = 148;
  float max_scale2 = 0.0f, max_s4 = 0.0f;  // for the batched path's fp16 range
  std::vector<uint32_t> host_row_ptr;       // CSR row pointers (group launch plans)
  qw_layer_info info{};
  bool k2_ok = true;  // the SIMT batch-1 kernel's shared-memory plan fits (else the layer runs on K2m)
};

struct qw_group {
  qwdev::GemvPlan plan;
  qwdev::MmaPlan mplan;
  bool mma = false;  // every layer has the tensor-core tile format
  std::vector<const qwdev::DeviceLayer*> layers;  // borrowed
  int device = 0;
  // batches: c columns of every layer in one launch (n * c <= kMaxSeg
  // segments, layer-major); index c, grid 0 = not planned
  std::vector<qwdev::GemvPlan> cplans;
  std::vector<qwdev::MmaPlan> mcplans;
};

struct qw_chain {
  qwdev::ChainPlan* plan = nullptr;      // SIMT chain kernel
  qwdev::MmaChainPlan* mplan = nullptr;  // tensor-core chain kernel (every layer in the K2m format)
  int device = 0;
  ~qw_chain() {
    qwdev::free_chain(plan);
    qwdev::free_mma_chain(mplan);
  }
};

struct qw_workspace {
  qwdev::Workspace ws;
  // host-buffer calls (qw_matvec_host*): device copies of x / y, grown on
  // demand and reused (no allocation on the steady-state call path), and
  // events for the per-stage device times
  float* dx = nullptr;
  float* dy = nullptr;
  size_t dx_cap = 0, dy_cap = 0;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& what) {
  g_last_error = what;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(QW_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& fn) {
  try {
    return fn();
  } catch (const qwb::Error& e) {
    const std::string m = e.what();
    const bool layer = m.rfind("layer", 0) == 0 || m.rfind("plan", 0) == 0 || m.rfind("csr", 0) == 0;
    const bool format = m.rfind("container", 0) == 0;
    return fail(format ? QW_ERR_FORMAT : (layer ? QW_ERR_LAYER : QW_ERR_ARG), m);
  } catch (const std::bad_alloc&) {
    return fail(QW_ERR_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(QW_ERR_ARG, e.what());
  }
}

template <class T>
void take(std::vector<T>& dst, const T* src, uint64_t n, const char* name) {
  if (n && !src) throw qwb::Error(std::string("view: null pointer for ") + name);
  dst.assign(src, src + n);
}

qwb::PackedLayer from_view(const qw_layer_view& v) {
  qwb::PackedLayer L;
  auto& c = L.cfg;
  c.n = v.n, c.n2 = v.n2, c.group1 = v.group1, c.group2 = v.group2, c.tile = v.tile;
  c.rows = v.rows, c.cols = v.cols, c.n4 = v.n4, c.pad2 = v.pad2;
  c.outlier_count = v.outlier_count, c.alpha = v.alpha, c.outlier_ratio = v.outlier_ratio;
  L.plan.in_channels = v.cols, L.plan.n4 = v.n4, L.plan.pad2 = v.pad2;
  take(L.plan.bits, v.plan_bits, v.plan_bits_len, "plan_bits");
  take(L.plan.perm, v.plan_perm, v.plan_perm_len, "plan_perm");
  take(L.main, v.main, v.main_len, "main");
  take(L.tail2, v.tail2, v.tail2_len, "tail2");
  take(L.tail4, v.tail4, v.tail4_len, "tail4");
  take(L.secondary, v.secondary, v.secondary_len, "secondary");
  take(L.meta, v.meta, v.meta_len, "meta");
  if (v.sorder_len && (!v.sorder_zero2 || !v.sorder_scale2)) throw qwb::Error("view: null sorder");
  L.sorder.resize(v.sorder_len);
  for (uint64_t i = 0; i < v.sorder_len; ++i) L.sorder[i] = {v.sorder_zero2[i], v.sorder_scale2[i]};
  if (v.fourbit_len && (!v.fourbit_zero || !v.fourbit_scale)) throw qwb::Error("view: null fourbit");
  L.fourbit.resize(v.fourbit_len);
  for (uint64_t i = 0; i < v.fourbit_len; ++i) L.fourbit[i] = {v.fourbit_scale[i], v.fourbit_zero[i]};
  take(L.csr.row_ptr, v.csr_row_ptr, v.csr_row_ptr_len, "csr_row_ptr");
  take(L.csr.col_ind, v.csr_col_ind, v.csr_nnz, "csr_col_ind");
  take(L.csr.values, v.csr_values, v.csr_nnz, "csr_values");
  return L;
}

void fill_view(const qw_host_layer& h, qw_layer_view* v) {
  const auto& L = h.L;
  const auto& c = L.cfg;
  std::memset(v, 0, sizeof *v);
  v->n = c.n, v->n2 = c.n2, v->group1 = c.group1, v->group2 = c.group2, v->tile = c.tile;
  v->rows = c.rows, v->cols = c.cols, v->n4 = c.n4, v->pad2 = c.pad2;
  v->outlier_count = c.outlier_count, v->alpha = c.alpha, v->outlier_ratio = c.outlier_ratio;
  v->plan_bits = L.plan.bits.data(), v->plan_bits_len = L.plan.bits.size();
  v->plan_perm = L.plan.perm.data(), v->plan_perm_len = L.plan.perm.size();
  v->main = L.main.data(), v->main_len = L.main.size();
  v->tail2 = L.tail2.data(), v->tail2_len = L.tail2.size();
  v->tail4 = L.tail4.data(), v->tail4_len = L.tail4.size();
  v->secondary = L.secondary.data(), v->secondary_len = L.secondary.size();
  v->meta = L.meta.data(), v->meta_len = L.meta.size();
  v->sorder_zero2 = h.sorder_zero2.data(), v->sorder_scale2 = h.sorder_scale2.data();
  v->sorder_len = L.sorder.size();
  v->fourbit_scale = h.fourbit_scale.data(), v->fourbit_zero = h.fourbit_zero.data();
  v->fourbit_len = L.fourbit.size();
  v->csr_row_ptr = L.csr.row_ptr.data(), v->csr_row_ptr_len = L.csr.row_ptr.size();
  v->csr_col_ind = L.csr.col_ind.data(), v->csr_values = L.csr.values.data();
  v->csr_nnz = L.csr.col_ind.size();
}

qwdev::Geometry geometry_of(const qwb::LayerConfig& c, uint64_t nnz) {
  qwdev::Geometry g{};
  g.rows = c.rows, g.cols = c.cols, g.padded_cols = c.padded_cols();
  g.n2p = c.n2_padded(), g.n4 = c.n4;
  g.T2 = c.triples(), g.T4 = c.blocks4(), g.G2 = 3 * g.T2, g.G = g.G2 + g.T4;
  g.G2s = (g.G2 + 3u) & ~3u;
  g.group2 = c.group2, g.row_blocks = c.row_blocks();
  g.quads = (c.rows + qwdev::kRowsPerQuad - 1) / qwdev::kRowsPerQuad;
  auto a16 = [](uint32_t v) { return (v + 15u) & ~15u; };
  g.off_c4 = 16u * g.G2;
  g.off_meta = g.off_c4 + 32u * g.T4;
  g.off_s4 = g.off_meta + a16(8u * g.T2);
  g.off_z4 = g.off_s4 + a16(8u * g.T4);
  g.dense_bytes = g.off_z4 + a16(2u * g.T4);
  uint32_t mx = 1;
  for (uint32_t q = 0; q < g.quads; ++q) {
    const uint32_t r0 = q * 4, r1 = std::min(r0 + 4, c.rows) - 1;
    mx = std::max(mx, r1 / c.group2 - r0 / c.group2 + 1);
    if (c.group2 % 4 == 0) break;
  }
  g.max_rb_per_quad = mx;
  g.nnz = nnz;
  return g;
}

void fill_info(const qwb::LayerConfig& c, uint64_t nnz, qw_layer_info* info) {
  const qwdev::Geometry g = geometry_of(c, nnz);
  std::memset(info, 0, sizeof *info);
  info->rows = c.rows, info->cols = c.cols, info->padded_cols = c.padded_cols();
  info->n2_padded = c.n2_padded(), info->n4 = c.n4, info->triples = c.triples();
  info->blocks4 = c.blocks4(), info->groups = g.G, info->group2 = c.group2;
  info->row_blocks = c.row_blocks(), info->quads = g.quads, info->quad_bytes = g.dense_bytes;
  info->nnz = nnz;
  info->payload_bytes = qwb::payload_bytes(c, nnz);
  const uint64_t sorder = (uint64_t)g.row_blocks * g.G2s * 4;
  info->device_bytes = (uint64_t)g.quads * g.dense_bytes + sorder + (uint64_t)g.padded_cols * 4 +
                       ((uint64_t)c.rows + 1) * 4 + nnz * 4;
  // one matvec streams every quad record, the sorder rows of each quad, the
  // quads' row_ptr words and the fused CSR entries
  uint64_t sorder_reads = 0;
  for (uint32_t q = 0; q < g.quads; ++q) {
    const uint32_t r0 = q * 4, r1 = std::min(r0 + 4, c.rows) - 1;
    sorder_reads += (uint64_t)(r1 / c.group2 - r0 / c.group2 + 1) * g.G2s * 4;
  }
  info->stream_bytes = (uint64_t)g.quads * g.dense_bytes + std::min(sorder_reads, sorder) +
                       ((uint64_t)c.rows + 1) * 4 + nnz * 4;
}

// Reference stream accessors (bitpack.cpp:175-210) for one row.
struct RowSrc {
  const qwb::PackedLayer& L;
  uint32_t code2_word(uint32_t r, uint32_t g) const {  // 16 codes of 2-bit group g
    const auto& c = L.cfg;
    const uint32_t t = g / 3, sub = g % 3, P = c.paired();
    const uint8_t* b = t < P ? &L.main[((size_t)r * P + t) * 16]
                             : &L.tail2[((size_t)r * c.tail2_blocks() + (t - P)) * 12];
    uint32_t w;
    std::memcpy(&w, b + 4 * sub, 4);
    return w;
  }
  uint32_t code4_word(uint32_t r, uint32_t b, uint32_t half) const {
    const auto& c = L.cfg;
    const uint32_t P = c.paired();
    const uint8_t* p;
    if (half == 0)
      p = b < P ? &L.main[((size_t)r * P + b) * 16 + 12]
                : &L.tail4[((size_t)r * c.tail4_blocks() + (b - P)) * 4];
    else
      p = &L.secondary[((size_t)r * c.blocks4() + b) * 4];
    uint32_t w;
    std::memcpy(&w, p, 4);
    return w;
  }
};

// North-star (a): the aligned device format.
void repack(const qwb::PackedLayer& L, const qwdev::Geometry& g, std::vector<uint8_t>& quads,
            std::vector<uint32_t>& sorder, std::vector<uint32_t>& csr) {
  const auto& c = L.cfg;
  quads.assign((size_t)g.quads * g.dense_bytes, 0);
  RowSrc src{L};
  for (uint32_t q = 0; q < g.quads; ++q) {
    uint8_t* rec = &quads[(size_t)q * g.dense_bytes];
    // reference words of the quad's rows (rows past the end stay zero)
    const uint32_t nr = std::min<uint32_t>(4, c.rows - q * 4);
    for (uint32_t gi = 0; gi < g.G2; ++gi) {
      uint32_t w[4] = {0, 0, 0, 0};
      for (uint32_t i = 0; i < nr; ++i) w[i] = src.code2_word(q * 4 + i, gi);
      uint32_t out[4];
      qwdev::pack_pair2(w[0], w[1], out);
      qwdev::pack_pair2(w[2], w[3], out + 2);
      std::memcpy(rec + 16 * gi, out, 16);
    }
    for (uint32_t b = 0; b < g.T4; ++b) {
      uint32_t lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
      for (uint32_t i = 0; i < nr; ++i) {
        lo[i] = src.code4_word(q * 4 + i, b, 0);
        hi[i] = src.code4_word(q * 4 + i, b, 1);
      }
      uint32_t out[8];
      qwdev::pack_pair4(lo[0], hi[0], lo[1], hi[1], out);
      qwdev::pack_pair4(lo[2], hi[2], lo[3], hi[3], out + 4);
      std::memcpy(rec + g.off_c4 + 32 * b, out, 32);
    }
    for (uint32_t i = 0; i < nr; ++i) {
      const uint32_t r = q * 4 + i;
      for (uint32_t b = 0; b < g.T4; ++b) {
        const auto& fb = L.fourbit[(size_t)r * g.T4 + b];
        std::memcpy(rec + g.off_s4 + 8 * b + 2 * i, &fb.scale, 2);
        uint16_t z4;
        std::memcpy(&z4, rec + g.off_z4 + 2 * b, 2);
        z4 = (uint16_t)(z4 | ((fb.zero & 15u) << (4 * i)));
        std::memcpy(rec + g.off_z4 + 2 * b, &z4, 2);
      }
      for (uint32_t t = 0; t < g.T2; ++t)
        std::memcpy(rec + g.off_meta + 8 * t + 2 * i, &L.meta[(size_t)r * g.T2 + t], 2);
    }
  }
  sorder.assign((size_t)g.row_blocks * g.G2s, 0);
  for (uint32_t rb = 0; rb < g.row_blocks; ++rb)
    for (uint32_t j = 0; j < g.G2; ++j) {
      const auto& p = L.sorder[(size_t)rb * g.G2 + j];
      sorder[(size_t)rb * g.G2s + j] = (uint32_t)p.scale2 | ((uint32_t)p.zero2 << 16);
    }
  csr.resize(L.csr.col_ind.size());
  for (size_t e = 0; e < csr.size(); ++e)
    // the entry names the ORIGINAL channel of its permuted column (perm[col],
    // a real channel: outliers live in the 2-bit non-pad region), so the
    // kernels read x without a perm lookup
    csr[e] = L.plan.perm[L.csr.col_ind[e]] | ((uint32_t)L.csr.values[e] << 16);
}

template <class T>
cudaError_t upload(T** dst, const std::vector<T>& src, size_t min_elems = 1) {
  const size_t n = std::max(src.size(), min_elems);
  cudaError_t e = cudaMalloc((void**)dst, n * sizeof(T));
  if (e != cudaSuccess) return e;
  if (!src.empty()) e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

void free_dev(qwdev::DeviceLayer& d) {
  qwdev::free_gemm(d);
  cudaFree(d.quads), cudaFree(d.sorder), cudaFree(d.perm), cudaFree(d.row_ptr), cudaFree(d.csr);
  cudaFree(d.perm16);
  cudaFree(d.mrecs), cudaFree(d.mpart), cudaFree(d.mcnt);
  d = qwdev::DeviceLayer{};
}

// K2m scratch: chunk partials + CSR sums, arrival counters (zeroed; the
// kernel leaves them zero)
cudaError_t alloc_mma_scratch(qwdev::DeviceLayer& d) {
  const auto& m = d.mg;
  cudaError_t e = cudaSuccess;
  if (m.nchunks > 1) {  // one slot per column of a column launch (launch_columns)
    const size_t slots = qwdev::kMaxSeg;
    if ((e = cudaMalloc((void**)&d.mpart, slots * (m.nchunks + 1) * m.RT * 16 * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc((void**)&d.mcnt, slots * m.RT * 4)) != cudaSuccess) return e;
    e = cudaMemset(d.mcnt, 0, slots * m.RT * 4);
  }
  return e;
}

int check_ws(const qw_layer* L, const qw_workspace* ws, uint32_t batch) {
  if (!L || !ws) return fail(QW_ERR_ARG, "matvec: null layer or workspace");
  if (batch == 0 || batch > 16) return fail(QW_ERR_ARG, "matvec: batch must be in 1..16");
  if (batch > ws->ws.max_batch) return fail(QW_ERR_ARG, "matvec: batch exceeds workspace");
  if (L->dev.g.padded_cols > ws->ws.max_cols)
    return fail(QW_ERR_ARG, "matvec: layer wider than workspace max_cols");
  if (L->device != ws->ws.device) return fail(QW_ERR_ARG, "matvec: layer and workspace on different devices");
  return QW_OK;
}

// batched policy (qweight_b200.h): K4 from QW_GEMM_MIN_BATCH columns up, the
// batch-1 kernel over the columns (8 to a launch) below -- up to 5 columns
// one column launch beats K4 on every 7B shape; from 6 columns K4 wins
// (q_proj 12.7 vs 13.2 us, gate/up 28.3 vs 29.1, down_proj 25.7 vs 30.6;
// profiles/r02_batch_sweep_simt.jsonl)
bool uses_gemm(const qw_layer* L, uint32_t batch, uint32_t flags) {
  static const uint32_t forced = qwdev::knob("QW_GEMM_MIN_BATCH", 0);
  if (batch < 2 || !L->dev.gemm.ok || (flags & QW_LAUNCH_FORCE_COLUMNS)) return false;
  const uint32_t min_batch = forced ? forced : QW_GEMM_MIN_BATCH;
  return (flags & QW_LAUNCH_FORCE_GEMM) || batch >= min_batch;
}

// columns of a batch share launches (qw_columns.cu); QW_COLUMN_GROUP=0 (debug
// knob) runs one launch per column for A/B measurements
bool column_groups() {
  static const uint32_t on = qwdev::knob("QW_COLUMN_GROUP", 1);
  return on != 0;
}

int run_matvec(const qw_layer* L, const float* x, uint32_t batch, float* y, qw_workspace* ws,
               void* stream, bool pdl, uint32_t flags = 0) {
  if (int s = check_ws(L, ws, batch)) return s;
  if (!x || !y) return fail(QW_ERR_ARG, "matvec: null activation or output");
  int dev_now = -1;
  cudaGetDevice(&dev_now);
  if (dev_now != L->device) {
    cudaError_t e = cudaSetDevice(L->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  }
  const uint32_t xflags = (flags & QW_LAUNCH_X_INDEPENDENT) ? qwdev::kXIndependent : 0u;
  int e = 0;
  if (uses_gemm(L, batch, flags)) {
    e = qwdev::launch_gemm(L->dev, x, batch, y, stream);
  } else if (batch > 1 && column_groups()) {
    e = qwdev::launch_columns(L->dev, x, batch, y, stream, pdl, xflags);
  } else if (L->dev.mrecs) {
    const qwdev::DeviceLayer* one[1] = {&L->dev};
    for (uint32_t col = 0; col < batch && !e; ++col) {
      float* ys[1] = {y + (size_t)col * L->dev.g.rows};
      e = qwdev::launch_mma(L->dev.mplan, one, 1, x + (size_t)col * L->dev.g.cols, ys, stream, pdl, xflags);
    }
  } else {
    e = qwdev::launch_gemv(L->dev, x, batch, y, stream, pdl, nullptr, 1, false, xflags);
  }
  if (e) return cuda_fail((cudaError_t)e, "gemv launch");
  return QW_OK;
}

int upload_packed(const qwb::PackedLayer& L, int device, uint32_t flags, qw_layer** out) {
  {
    qwb::validate_layer(L);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return fail(QW_ERR_CUDA, "upload: no CUDA device available");
    if (device < 0 || device >= ndev) return fail(QW_ERR_ARG, "upload: device index out of range");
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    auto H = std::make_unique<qw_layer>();
    H->device = device;
    cudaDeviceGetAttribute(&H->num_sms, cudaDevAttrMultiProcessorCount, device);
    H->dev.g = geometry_of(L.cfg, L.csr.nnz());
    fill_info(L.cfg, L.csr.nnz(), &H->info);
    std::vector<uint8_t> quads;
    std::vector<uint32_t> sorder, csr;
    repack(L, H->dev.g, quads, sorder, csr);
    csr.resize(csr.size() + 4, 0u);  // padding: 16-byte aligned bulk copies of a CTA's entries may overrun
    std::vector<uint16_t> perm16(L.plan.perm.size());
    for (size_t i = 0; i < perm16.size(); ++i)
      perm16[i] = L.plan.perm[i] == qwb::kPad ? (uint16_t)L.cfg.cols : (uint16_t)L.plan.perm[i];  // pads: x[cols] = 0 slot
    H->host_row_ptr = L.csr.row_ptr;
    if (H->host_row_ptr.empty()) H->host_row_ptr.assign((size_t)L.cfg.rows + 1, 0u);
    if (int pe = qwdev::plan_gemv(H->dev, H->num_sms, H->host_row_ptr.data())) {
      // the SIMT kernel cannot take the layer (more than 60 chunks of 32
      // groups, or its x / 2-order rows / ring do not fit in shared memory):
      // the tensor-core kernel K2m serves it, decided below
      if (pe != (int)cudaErrorInvalidConfiguration) return cuda_fail((cudaError_t)pe, "gemv plan");
      H->k2_ok = false;
    }
    {  // 2^-P so that 15 * max|scale2| * 2^-P lies in [2^14, 2^15): fp16 1st-order scales
      float mx = 0.0f;
      for (const auto& sp : L.sorder) mx = std::max(mx, std::fabs(qwb::f16_to_f32(sp.scale2)));
      int P = 0;
      if (mx > 0.0f && std::isfinite(mx)) P = std::ilogb(15.0f * mx) - 14;
      H->dev.plan.s_scale = std::ldexp(1.0f, -std::max(-100, std::min(100, P)));
      H->max_scale2 = mx;
      float m4 = 0.0f;
      for (const auto& fb : L.fourbit) m4 = std::max(m4, std::fabs(qwb::f16_to_f32(fb.scale)));
      H->max_s4 = m4;
    }
    if ((e = upload(&H->dev.quads, quads)) != cudaSuccess ||
        (e = upload(&H->dev.sorder, sorder)) != cudaSuccess ||
        (e = upload(&H->dev.perm, L.plan.perm)) != cudaSuccess ||
        (e = upload(&H->dev.row_ptr, L.csr.row_ptr)) != cudaSuccess ||
        (e = upload(&H->dev.csr, csr)) != cudaSuccess ||
        (e = upload(&H->dev.perm16, perm16)) != cudaSuccess) {
      free_dev(H->dev);
      return cuda_fail(e, "upload");
    }
    if (int ge = qwdev::plan_gemm(H->dev, H->num_sms, H->max_scale2, H->max_s4)) {
      free_dev(H->dev);
      return cuda_fail((cudaError_t)ge, "gemm plan");
    }
    qwdev::mma_geometry(H->dev.mg, H->dev.g);
    // batch-1 kernel policy (header): auto picks K2m where K2's plan falls
    // back to its global-memory CSR loop with more than ~1.5 K outliers per
    // CTA (13B down_proj: K2 12.5 / 13.5 us vs K2m 15.6 at 0.1 / 0.2 %, but
    // 25.1 / 46.0 vs 15.8 / 16.5 at 0.5 / 1 %), needs more than two groups
    // per lane outside the wide layout, or cannot stage x (> 16384 columns)
    const auto& gp = H->dev.plan;
    uint32_t ent_max = 0;
    for (uint32_t c = 0; c < gp.grid; ++c) ent_max = std::max(ent_max, gp.cta_e1[c] - gp.cta_e0[c]);
    const bool k2_slow = (L.csr.nnz() > 0 && !gp.csr_stage && ent_max > 1536) || (gp.kmax > 2 && !gp.wide) || !gp.xsm;
    const bool want_mma = (flags & QW_UPLOAD_TENSOR_CORE) || (!(flags & QW_UPLOAD_SIMT) && (k2_slow || !H->k2_ok));
    if (!H->k2_ok && !(H->dev.mg.ok && want_mma)) {
      free_dev(H->dev);
      return fail(QW_ERR_UNSUPPORTED, (flags & QW_UPLOAD_SIMT)
                                          ? "upload: the SIMT batch-1 kernel cannot take this layer (more than 60 "
                                            "chunks of 32 groups, or its shared-memory plan does not fit); "
                                            "upload without QW_UPLOAD_SIMT"
                                          : "upload: neither batch-1 kernel can take this layer");
    }
    if (H->dev.mg.ok && want_mma) {
      std::vector<uint8_t> recs;
      qwb::repack_mma(L, H->dev.mg, H->dev.plan.s_scale, recs);
      const qwdev::DeviceLayer* one[1] = {&H->dev};
      if ((e = upload(&H->dev.mrecs, recs)) != cudaSuccess || (e = alloc_mma_scratch(H->dev)) != cudaSuccess) {
        free_dev(H->dev);
        return cuda_fail(e, "upload (mma tiles)");
      }
      const uint32_t* rp[1] = {H->host_row_ptr.data()};
      if (int pe = qwdev::plan_mma(H->dev.mplan, one, rp, 1, H->num_sms)) {
        free_dev(H->dev);
        return cuda_fail((cudaError_t)pe, "mma plan");
      }
    }
    qwdev::plan_columns(H->dev, H->num_sms, H->host_row_ptr.data());
    *out = H.release();
    return (int)QW_OK;
  }
}
}  // namespace

extern "C" {

int qw_abi_version(void) { return QW_ABI_VERSION; }

const char* qw_strerror(int s) {
  switch (s) {
    case QW_OK: return "ok";
    case QW_ERR_ARG: return "invalid argument";
    case QW_ERR_LAYER: return "invalid layer";
    case QW_ERR_CUDA: return "CUDA error";
    case QW_ERR_NCCL: return "NCCL error";
    case QW_ERR_UNSUPPORTED: return "unsupported geometry";
    case QW_ERR_NOMEM: return "out of memory";
    case QW_ERR_IO: return "I/O error";
    case QW_ERR_FORMAT: return "corrupt container";
    default: return "unknown status";
  }
}

const char* qw_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ host
int qw_host_quantize(const float* w, uint32_t rows, uint32_t cols, const float* h, double alpha,
                     uint32_t group2, double ratio, uint32_t threads, qw_host_layer** out) {
  return guarded([&] {
    if (!w || !h || !out) return fail(QW_ERR_ARG, "quantize: null argument");
    qwb::WeightMatrix W;
    W.rows = rows, W.cols = cols;
    W.data.assign(w, w + (size_t)rows * cols);
    qwb::QuantizeParams p;
    p.alpha = alpha, p.group2 = group2, p.outlier_ratio = ratio;
    auto H = std::make_unique<qw_host_layer>();
    H->L = qwb::quantize_layer(W, {h, cols}, p, threads);
    H->refresh_soa();
    *out = H.release();
    return (int)QW_OK;
  });
}

int qw_device_quantize(const float* w, uint32_t rows, uint32_t cols, const float* h, double alpha,
                       uint32_t group2, double ratio, int device, qw_host_layer** out) {
  return guarded([&] {
    if (!w || !h || !out) return fail(QW_ERR_ARG, "quantize: null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      return fail(QW_ERR_CUDA, "device quantize: no CUDA device available");
    if (device < 0 || device >= ndev) return fail(QW_ERR_ARG, "device quantize: device index out of range");
    qwb::QuantizeParams p;
    p.alpha = alpha, p.group2 = group2, p.outlier_ratio = ratio;
    auto H = std::make_unique<qw_host_layer>();
    H->L = qwb::quantize_layer_gpu(w, rows, cols, {h, cols}, p, device);
    H->refresh_soa();
    *out = H.release();
    return (int)QW_OK;
  });
}

int qw_host_from_view(const qw_layer_view* v, qw_host_layer** out) {
  return guarded([&] {
    if (!v || !out) return fail(QW_ERR_ARG, "from_view: null argument");
    auto H = std::make_unique<qw_host_layer>();
    H->L = from_view(*v);
    qwb::validate_layer(H->L);
    H->refresh_soa();
    *out = H.release();
    return (int)QW_OK;
  });
}

int qw_host_view(const qw_host_layer* h, qw_layer_view* v) {
  if (!h || !v) return fail(QW_ERR_ARG, "view: null argument");
  fill_view(*h, v);
  return QW_OK;
}

void qw_host_free(qw_host_layer* h) { delete h; }

int qw_host_write(const qw_host_layer* h, const char* path) {
  return guarded([&] {
    if (!h || !path) return fail(QW_ERR_ARG, "write: null argument");
    const std::vector<uint8_t> bytes = qwb::serialize_layer(h->L);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) return fail(QW_ERR_IO, std::string("cannot open ") + path + " for writing");
    f.write((const char*)bytes.data(), (std::streamsize)bytes.size());
    if (!f) return fail(QW_ERR_IO, std::string("failed to write ") + path);
    return (int)QW_OK;
  });
}

int qw_host_read(const char* path, qw_host_layer** out) {
  return guarded([&] {
    if (!path || !out) return fail(QW_ERR_ARG, "read: null argument");
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(QW_ERR_IO, std::string("cannot open ") + path);
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    auto H = std::make_unique<qw_host_layer>();
    H->L = qwb::deserialize_layer(bytes);
    H->refresh_soa();
    *out = H.release();
    return (int)QW_OK;
  });
}

int qw_host_shard_rows(const qw_host_layer* h, uint32_t r0, uint32_t r1, qw_host_layer** out) {
  return guarded([&] {
    if (!h || !out) return fail(QW_ERR_ARG, "shard_rows: null argument");
    auto H = std::make_unique<qw_host_layer>();
    H->L = qwb::shard_rows(h->L, r0, r1);
    H->refresh_soa();
    *out = H.release();
    return (int)QW_OK;
  });
}

int qw_host_shard_tiles(const qw_host_layer* h, uint32_t t0, uint32_t t1, qw_host_layer** out,
                        uint32_t* offs) {
  return guarded([&] {
    if (!h || !out) return fail(QW_ERR_ARG, "shard_tiles: null argument");
    auto H = std::make_unique<qw_host_layer>();
    H->L = qwb::shard_tiles(h->L, t0, t1);
    H->refresh_soa();
    if (offs) {
      const auto& c = h->L.cfg;
      offs[0] = 48 * t0;
      offs[1] = std::min(48 * t1, c.cols - c.n4);
      offs[2] = c.n2_padded() + 16 * t0;
      offs[3] = c.n2_padded() + 16 * t1;
    }
    *out = H.release();
    return (int)QW_OK;
  });
}

int qw_validate_layer(const qw_layer_view* v) {
  return guarded([&] {
    if (!v) return fail(QW_ERR_ARG, "validate: null view");
    qwb::validate_layer(from_view(*v));
    return (int)QW_OK;
  });
}

uint64_t qw_payload_bytes(const qw_layer_view* v) {
  if (!v) return 0;
  qwb::LayerConfig c;
  c.rows = v->rows, c.cols = v->cols, c.n4 = v->n4, c.pad2 = v->pad2, c.group2 = v->group2;
  return qwb::payload_bytes(c, v->csr_nnz);
}

int qw_layer_view_info(const qw_layer_view* v, qw_layer_info* info) {
  return guarded([&] {
    if (!v || !info) return fail(QW_ERR_ARG, "info: null argument");
    qwb::LayerConfig c;
    c.rows = v->rows, c.cols = v->cols, c.n4 = v->n4, c.pad2 = v->pad2, c.group2 = v->group2;
    if (c.group2 == 0 || c.rows == 0) return fail(QW_ERR_LAYER, "info: malformed config");
    fill_info(c, v->csr_nnz, info);
    return (int)QW_OK;
  });
}

int qw_synth_gaussian(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  return guarded([&] {
    if (!out) return fail(QW_ERR_ARG, "synth: null output");
    const qwb::WeightMatrix w = qwb::synth_gaussian(rows, cols, seed);
    std::memcpy(out, w.data.data(), w.data.size() * 4);
    return (int)QW_OK;
  });
}

int qw_plant_outliers(float* w, uint64_t count, double ratio, float scale, uint64_t seed) {
  return guarded([&] {
    if (!w && count) return fail(QW_ERR_ARG, "plant: null weights");
    qwb::plant_outliers({w, count}, ratio, scale, seed);
    return (int)QW_OK;
  });
}

int qw_synth_calibration(uint32_t cols, uint64_t seed, float* out) {
  return guarded([&] {
    if (!out) return fail(QW_ERR_ARG, "synth: null output");
    const auto h = qwb::synth_calibration(cols, seed);
    std::memcpy(out, h.data(), h.size() * 4);
    return (int)QW_OK;
  });
}

int qw_synth_activation(uint32_t cols, uint64_t seed, float* out) {
  return guarded([&] {
    if (!out) return fail(QW_ERR_ARG, "synth: null output");
    const auto x = qwb::synth_activation(cols, seed);
    std::memcpy(out, x.data(), x.size() * 4);
    return (int)QW_OK;
  });
}

// ------------------------------------------------------------------ device
int qw_layer_upload(const qw_layer_view* v, int device, qw_layer** out) {
  return qw_layer_upload_ex(v, device, 0u, out);
}

int qw_layer_upload_ex(const qw_layer_view* v, int device, uint32_t flags, qw_layer** out) {
  return guarded([&] {
    if (!v || !out) return fail(QW_ERR_ARG, "upload: null argument");
    return upload_packed(from_view(*v), device, flags, out);
  });
}

// QWL1 container (container.cpp:321-471) straight to the device: parse +
// CRC + validate_layer on the host, no intermediate host object for the caller
int qw_layer_upload_qwl(const uint8_t* bytes, uint64_t len, int device, uint32_t flags, qw_layer** out) {
  return guarded([&] {
    if (!bytes || !out) return fail(QW_ERR_ARG, "upload qwl: null argument");
    return upload_packed(qwb::deserialize_layer(std::span<const uint8_t>(bytes, len)), device, flags, out);
  });
}

int qw_layer_load(const char* path, int device, uint32_t flags, qw_layer** out) {
  return guarded([&] {
    if (!path || !out) return fail(QW_ERR_ARG, "load: null argument");
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(QW_ERR_IO, std::string("cannot open ") + path);
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return upload_packed(qwb::deserialize_layer(bytes), device, flags, out);
  });
}


int qw_layer_free(qw_layer* L) {
  if (!L) return QW_OK;
  cudaSetDevice(L->device);
  free_dev(L->dev);
  delete L;
  return QW_OK;
}

int qw_layer_uses_tensor_core(const qw_layer* L) { return L && L->dev.mrecs ? 1 : 0; }

int qw_layer_get_info(const qw_layer* L, qw_layer_info* info) {
  if (!L || !info) return fail(QW_ERR_ARG, "info: null argument");
  *info = L->info;
  return QW_OK;
}

int qw_workspace_create(int device, uint32_t max_cols, uint32_t max_batch, qw_workspace** out) {
  if (!out || max_batch == 0 || max_batch > 16 || max_cols == 0)
    return fail(QW_ERR_ARG, "workspace: bad arguments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(QW_ERR_CUDA, "workspace: no CUDA device available");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  auto W = std::make_unique<qw_workspace>();
  W->ws.device = device;
  W->ws.max_cols = max_cols + 48;  // room for 2-bit pads
  W->ws.max_batch = max_batch;
  if ((e = cudaMalloc((void**)&W->ws.flags, 16)) != cudaSuccess) return cuda_fail(e, "workspace alloc");
  cudaMemset(W->ws.flags, 0, 16);
  *out = W.release();
  return QW_OK;
}

int qw_workspace_free(qw_workspace* W) {
  if (!W) return QW_OK;
  cudaSetDevice(W->ws.device);
  cudaFree(W->ws.flags);
  cudaFree(W->dx), cudaFree(W->dy);
  for (auto& e : W->ev)
    if (e) cudaEventDestroy(e);
  delete W;
  return QW_OK;
}

int qw_matvec(const qw_layer* L, const float* x, uint32_t batch, float* y, qw_workspace* ws,
              void* stream) {
  return run_matvec(L, x, batch, y, ws, stream, false);
}

int qw_matvec_ex(const qw_layer* L, const float* x, uint32_t batch, float* y, qw_workspace* ws,
                 void* stream, uint32_t flags) {
  return run_matvec(L, x, batch, y, ws, stream, (flags & QW_LAUNCH_PDL) != 0, flags);
}

int qw_matvec_pdl(const qw_layer* L, const float* x, uint32_t batch, float* y, qw_workspace* ws,
                  void* stream) {
  return run_matvec(L, x, batch, y, ws, stream, true);
}

int qw_matvec_host(const qw_layer* L, const float* x, uint64_t x_len, uint32_t batch, float* y,
                   qw_workspace* ws, void* stream) {
  return qw_matvec_host_ex(L, x, x_len, batch, y, ws, stream, nullptr);
}

int qw_matvec_host_ex(const qw_layer* L, const float* x, uint64_t x_len, uint32_t batch, float* y,
                      qw_workspace* ws, void* stream, uint64_t* stage_ns) {
  if (int s = check_ws(L, ws, batch)) return s;
  if (!x || !y) return fail(QW_ERR_ARG, "matvec: null activation or output");
  // checked_permute (engine.cpp:124-132)
  if (x_len != (uint64_t)batch * L->info.cols)
    return fail(QW_ERR_ARG, "matvec: activation length != input channels");
  for (uint64_t i = 0; i < x_len; ++i)
    if (!std::isfinite(x[i])) return fail(QW_ERR_ARG, "matvec: non-finite activation");
  cudaSetDevice(L->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t xb = x_len * 4, yb = (size_t)batch * L->info.rows * 4;
  cudaError_t e;
  if (xb > ws->dx_cap) {  // grow once, keep: the steady-state call allocates nothing
    cudaFree(ws->dx);
    ws->dx = nullptr, ws->dx_cap = 0;
    if ((e = cudaMalloc((void**)&ws->dx, xb)) != cudaSuccess) return cuda_fail(e, "alloc x");
    ws->dx_cap = xb;
  }
  if (yb > ws->dy_cap) {
    cudaFree(ws->dy);
    ws->dy = nullptr, ws->dy_cap = 0;
    if ((e = cudaMalloc((void**)&ws->dy, yb)) != cudaSuccess) return cuda_fail(e, "alloc y");
    ws->dy_cap = yb;
  }
  if (stage_ns && !ws->ev[0])
    for (auto& ev : ws->ev)
      if ((e = cudaEventCreate(&ev)) != cudaSuccess) return cuda_fail(e, "event");
  int status = QW_OK;
  if (stage_ns) cudaEventRecord(ws->ev[0], st);
  if ((e = cudaMemcpyAsync(ws->dx, x, xb, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    status = cuda_fail(e, "copy x");
  if (stage_ns) cudaEventRecord(ws->ev[1], st);
  if (!status) status = run_matvec(L, ws->dx, batch, ws->dy, ws, stream, false);
  if (stage_ns) cudaEventRecord(ws->ev[2], st);
  if (!status && (e = cudaMemcpyAsync(y, ws->dy, yb, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    status = cuda_fail(e, "copy y");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess && !status) status = cuda_fail(e, "sync");
  if (stage_ns && !status) {
    // MatvecResult.stage_ns (engine.hpp:19-23) on the GPU: [0] the x copy
    // (activation fetch), [1] [2] 0 (scales and decode are fused into the
    // kernel), [3] the fused kernel(s)
    float ms0 = 0.f, ms1 = 0.f;
    cudaEventElapsedTime(&ms0, ws->ev[0], ws->ev[1]);
    cudaEventElapsedTime(&ms1, ws->ev[1], ws->ev[2]);
    stage_ns[0] = (uint64_t)(ms0 * 1e6), stage_ns[1] = 0, stage_ns[2] = 0, stage_ns[3] = (uint64_t)(ms1 * 1e6);
  }
  return status;
}

int qw_dequant(const qw_layer* L, float* w, void* stream) {
  if (!L || !w) return fail(QW_ERR_ARG, "dequant: null argument");
  cudaSetDevice(L->device);
  const int e = qwdev::launch_dequant(L->dev, w, stream);
  return e ? cuda_fail((cudaError_t)e, "dequant launch") : QW_OK;
}

int qw_dequant_host(const qw_layer* L, float* w, uint64_t w_len) {
  if (!L || !w) return fail(QW_ERR_ARG, "dequant: null argument");
  const uint64_t n = (uint64_t)L->info.rows * L->info.padded_cols;
  if (w_len != n) return fail(QW_ERR_ARG, "dequant: output length != rows * padded_cols");
  cudaSetDevice(L->device);
  float* dw = nullptr;
  cudaError_t e = cudaMalloc((void**)&dw, n * 4 + 4);
  if (e != cudaSuccess) return cuda_fail(e, "alloc w");
  int status = QW_OK;
  if (int k = qwdev::launch_dequant(L->dev, dw, nullptr)) status = cuda_fail((cudaError_t)k, "dequant launch");
  if (!status && (e = cudaMemcpy(w, dw, n * 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
    status = cuda_fail(e, "copy w");
  cudaFree(dw);
  return status;
}

int qw_unpack(const qw_layer* L, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes, uint8_t* codes4,
              void* stream) {
  if (!L || ((!codes2 || !zeros2 || !scodes) && L->dev.g.G2) || (!codes4 && L->dev.g.n4))
    return fail(QW_ERR_ARG, "unpack: null argument");
  cudaSetDevice(L->device);
  const int e = qwdev::launch_unpack(L->dev, codes2, zeros2, scodes, codes4, stream);
  return e ? cuda_fail((cudaError_t)e, "unpack launch") : QW_OK;
}

int qw_layer_clone(const qw_layer* L, qw_layer** out) {
  if (!L || !out) return fail(QW_ERR_ARG, "clone: null argument");
  cudaSetDevice(L->device);
  auto H = std::make_unique<qw_layer>();
  H->device = L->device, H->num_sms = L->num_sms, H->info = L->info, H->k2_ok = L->k2_ok;
  H->dev.g = L->dev.g;
  H->dev.plan = L->dev.plan;
  const auto& g = L->dev.g;
  auto dup = [](auto** dst, const auto* src, size_t bytes) {
    cudaError_t e = cudaMalloc((void**)dst, bytes ? bytes : 4);
    if (e == cudaSuccess && bytes) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyDeviceToDevice);
    return e;
  };
  cudaError_t e;
  if ((e = dup(&H->dev.quads, L->dev.quads, (size_t)g.quads * g.dense_bytes)) != cudaSuccess ||
      (e = dup(&H->dev.sorder, L->dev.sorder, (size_t)g.row_blocks * g.G2s * 4)) != cudaSuccess ||
      (e = dup(&H->dev.perm, L->dev.perm, (size_t)g.padded_cols * 4)) != cudaSuccess ||
      (e = dup(&H->dev.row_ptr, L->dev.row_ptr, ((size_t)g.rows + 1) * 4)) != cudaSuccess ||
      (e = dup(&H->dev.csr, L->dev.csr, ((size_t)g.nnz + 4) * 4)) != cudaSuccess ||
      (e = dup(&H->dev.perm16, L->dev.perm16, (size_t)g.padded_cols * 2)) != cudaSuccess) {
    free_dev(H->dev);
    return cuda_fail(e, "clone");
  }
  H->max_scale2 = L->max_scale2, H->max_s4 = L->max_s4;
  H->host_row_ptr = L->host_row_ptr;
  H->dev.gemm = qwdev::GemmPlan{};
  if (int ge = qwdev::plan_gemm(H->dev, H->num_sms, H->max_scale2, H->max_s4)) {
    free_dev(H->dev);
    return cuda_fail((cudaError_t)ge, "gemm plan");
  }
  H->dev.mg = L->dev.mg;
  if (L->dev.mrecs) {
    const auto& m = L->dev.mg;
    const qwdev::DeviceLayer* one[1] = {&H->dev};
    if ((e = dup(&H->dev.mrecs, L->dev.mrecs, (size_t)m.RT * m.nchunks * m.rec_stride)) != cudaSuccess ||
        (e = alloc_mma_scratch(H->dev)) != cudaSuccess) {
      free_dev(H->dev);
      return cuda_fail(e, "clone (mma tiles)");
    }
    const uint32_t* rp[1] = {H->host_row_ptr.data()};
    if (int pe = qwdev::plan_mma(H->dev.mplan, one, rp, 1, H->num_sms)) {
      free_dev(H->dev);
      return cuda_fail((cudaError_t)pe, "mma plan");
    }
  }
  qwdev::plan_columns(H->dev, H->num_sms, H->host_row_ptr.data());
  *out = H.release();
  return QW_OK;
}

int qw_debug_timeline(const qw_layer* L, const float* x, float* y, unsigned long long* stamps,
                      uint32_t repeat, uint32_t flags, void* stream) {
  if (!L || !x || !y || !stamps) return fail(QW_ERR_ARG, "timeline: null argument");
  cudaSetDevice(L->device);
  const int e = qwdev::launch_gemv(L->dev, x, 1, y, stream, flags & 1u, stamps, repeat,
                                   (flags & 2u) != 0, (flags & 4u) ? qwdev::kXIndependent : 0u);
  return e ? cuda_fail((cudaError_t)e, "gemv launch") : QW_OK;
}

int qw_group_create(const qw_layer* const* layers, uint32_t n, qw_group** out) {
  return guarded([&] {
    if (!layers || !out || n == 0) return fail(QW_ERR_ARG, "group: null argument");
    if (n > qwdev::kMaxSeg) return fail(QW_ERR_UNSUPPORTED, "group: at most 8 layers");
    auto G = std::make_unique<qw_group>();
    std::vector<const uint32_t*> rps;
    for (uint32_t i = 0; i < n; ++i) {
      if (!layers[i]) return fail(QW_ERR_ARG, "group: null layer");
      if (layers[i]->device != layers[0]->device) return fail(QW_ERR_ARG, "group: layers on different devices");
      G->layers.push_back(&layers[i]->dev);
      rps.push_back(layers[i]->host_row_ptr.data());
    }
    G->device = layers[0]->device;
    cudaSetDevice(G->device);
    G->mma = true;
    for (uint32_t i = 0; i < n; ++i) G->mma = G->mma && layers[i]->dev.mrecs != nullptr;
    const int e = qwdev::plan_gemv_group(G->plan, G->layers.data(), rps.data(), n, layers[0]->num_sms);
    if (e == (int)cudaErrorInvalidValue)
      return fail(QW_ERR_ARG, "group: layers must share cols, channel split and group2 (rows may differ)");
    if (e == (int)cudaErrorInvalidConfiguration && !G->mma)
      return fail(QW_ERR_UNSUPPORTED, "group: the SIMT kernel's plan does not fit these layers (upload them with "
                                      "the tensor-core kernel)");
    if (e && e != (int)cudaErrorInvalidConfiguration) return cuda_fail((cudaError_t)e, "group plan");
    if (e) G->plan.grid = 0;  // K2m group: the SIMT plan is never launched
    if (G->mma) {
      if (int me = qwdev::plan_mma(G->mplan, G->layers.data(), rps.data(), n, layers[0]->num_sms))
        return cuda_fail((cudaError_t)me, "group mma plan");
    }
    // batched group launches: c columns x n layers as one grid
    const uint32_t cmax = qwdev::kMaxSeg / n;
    G->cplans.assign(cmax + 1, qwdev::GemvPlan{});
    G->mcplans.assign(cmax + 1, qwdev::MmaPlan{});
    for (uint32_t c = 2; c <= cmax; ++c) {
      std::vector<const qwdev::DeviceLayer*> lay;
      std::vector<const uint32_t*> rp;
      for (uint32_t i = 0; i < n; ++i)
        for (uint32_t k = 0; k < c; ++k) lay.push_back(G->layers[i]), rp.push_back(rps[i]);
      if (qwdev::plan_gemv_group(G->cplans[c], lay.data(), rp.data(), n * c, layers[0]->num_sms))
        G->cplans[c] = qwdev::GemvPlan{}, G->cplans[c].grid = 0;
      if (G->mma && qwdev::plan_mma(G->mcplans[c], lay.data(), rp.data(), n * c, layers[0]->num_sms))
        G->mcplans[c] = qwdev::MmaPlan{}, G->mcplans[c].grid = 0;
    }
    *out = G.release();
    return (int)QW_OK;
  });
}

int qw_group_free(qw_group* g) {
  delete g;
  return QW_OK;
}

int qw_group_matvec_batch(const qw_group* g, const float* x, uint32_t batch, float* const* ys, void* stream,
                          uint32_t flags) {
  if (!g || !x || !ys) return fail(QW_ERR_ARG, "group matvec: null argument");
  if (batch == 0 || batch > 16) return fail(QW_ERR_ARG, "group matvec: batch must be in 1..16");
  const uint32_t n = (uint32_t)g->layers.size();
  for (uint32_t i = 0; i < n; ++i)
    if (!ys[i]) return fail(QW_ERR_ARG, "group matvec: null output");
  int dev_now = -1;
  cudaGetDevice(&dev_now);
  if (dev_now != g->device) cudaSetDevice(g->device);
  const uint32_t xflags = (flags & QW_LAUNCH_X_INDEPENDENT) ? qwdev::kXIndependent : 0u;
  const bool pdl = (flags & QW_LAUNCH_PDL) != 0;
  const uint32_t cols = g->layers[0]->g.cols, cmax = std::max<uint32_t>(1, qwdev::kMaxSeg / n);
  for (uint32_t c0 = 0; c0 < batch;) {
    uint32_t cb = std::min(cmax, batch - c0);
    const bool planned = cb > 1 && (g->mma ? g->mcplans[cb].grid : g->cplans[cb].grid) != 0;
    if (!planned) cb = 1;
    const qwdev::DeviceLayer* lay[qwdev::kMaxSeg];
    const float* xs[qwdev::kMaxSeg];
    float* yo[qwdev::kMaxSeg];
    uint32_t slot[qwdev::kMaxSeg];
    uint32_t s = 0;
    for (uint32_t i = 0; i < n; ++i)  // layer-major segments, as planned
      for (uint32_t k = 0; k < cb; ++k, ++s) {
        lay[s] = g->layers[i], slot[s] = k;
        xs[s] = x + (size_t)(c0 + k) * cols;
        yo[s] = ys[i] + (size_t)(c0 + k) * g->layers[i]->g.rows;
      }
    int e;
    if (g->mma)
      e = qwdev::launch_mma(cb > 1 ? g->mcplans[cb] : g->mplan, lay, s, xs, yo, stream, pdl, xflags, slot);
    else
      e = qwdev::launch_gemv_group(cb > 1 ? g->cplans[cb] : g->plan, lay, s, xs, yo, stream, pdl, xflags, nullptr,
                                   1, false);
    if (e) return cuda_fail((cudaError_t)e, "group launch");
    c0 += cb;
  }
  return QW_OK;
}

int qw_group_matvec(const qw_group* g, const float* x, float* const* ys, void* stream, uint32_t flags) {
  if (!g || !x || !ys) return fail(QW_ERR_ARG, "group matvec: null argument");
  for (size_t i = 0; i < g->layers.size(); ++i)
    if (!ys[i]) return fail(QW_ERR_ARG, "group matvec: null output");
  int dev_now = -1;
  cudaGetDevice(&dev_now);
  if (dev_now != g->device) cudaSetDevice(g->device);
  const uint32_t xflags = (flags & QW_LAUNCH_X_INDEPENDENT) ? qwdev::kXIndependent : 0u;
  const int e = g->mma ? qwdev::launch_mma(g->mplan, g->layers.data(), (uint32_t)g->layers.size(), x, ys, stream,
                                           (flags & QW_LAUNCH_PDL) != 0, xflags)
                       : qwdev::launch_gemv_group(g->plan, g->layers.data(), (uint32_t)g->layers.size(), x, ys,
                                                  stream, (flags & QW_LAUNCH_PDL) != 0, xflags);
  return e ? cuda_fail((cudaError_t)e, "group launch") : QW_OK;
}

}  // extern "C"

namespace {
int set_prefetch(qwdev::GemvPlan& p, int device, const qw_layer* const* next, uint32_t n) {
  if (n && !next) return fail(QW_ERR_ARG, "prefetch: null layer list");
  if (2 * n > qwdev::GemvPlan::kMaxPf) return fail(QW_ERR_UNSUPPORTED, "prefetch: at most 4 next layers");
  for (uint32_t i = 0; i < n; ++i) {
    if (!next[i]) return fail(QW_ERR_ARG, "prefetch: null layer");
    if (next[i]->device != device) return fail(QW_ERR_ARG, "prefetch: layer on another device");
  }
  p.pf_n = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const qwdev::DeviceLayer& d = next[i]->dev;
    p.pf_ptr[p.pf_n] = d.quads;
    p.pf_bytes[p.pf_n++] = d.g.quads * d.g.dense_bytes;
    p.pf_ptr[p.pf_n] = reinterpret_cast<const uint8_t*>(d.sorder);
    p.pf_bytes[p.pf_n++] = d.g.row_blocks * d.g.G2s * 4u;
  }
  return QW_OK;
}
}  // namespace

extern "C" {

int qw_layer_set_prefetch(qw_layer* L, const qw_layer* const* next, uint32_t n) {
  if (!L) return fail(QW_ERR_ARG, "prefetch: null layer");
  return set_prefetch(L->dev.plan, L->device, next, n);
}

int qw_group_set_prefetch(qw_group* g, const qw_layer* const* next, uint32_t n) {
  if (!g) return fail(QW_ERR_ARG, "prefetch: null group");
  return set_prefetch(g->plan, g->device, next, n);
}

int qw_chain_create(const qw_chain_step* steps, uint32_t n, qw_chain** out) {
  return guarded([&] {
    if (!steps || !out || n == 0) return fail(QW_ERR_ARG, "chain: null argument");
    std::vector<qwdev::ChainStepDesc> d(n);
    std::vector<std::vector<const qwdev::DeviceLayer*>> lay(n);
    std::vector<std::vector<const uint32_t*>> rps(n);
    const int device = steps[0].n && steps[0].layers && steps[0].layers[0] ? steps[0].layers[0]->device : 0;
    int num_sms = 148;
    for (uint32_t s = 0; s < n; ++s) {
      const qw_chain_step& st = steps[s];
      if (!st.layers || !st.ys || !st.x || st.n == 0) return fail(QW_ERR_ARG, "chain: null step field");
      if (st.n > qwdev::kMaxSeg) return fail(QW_ERR_UNSUPPORTED, "chain: at most 8 layers per step");
      for (uint32_t l = 0; l < st.n; ++l) {
        if (!st.layers[l] || !st.ys[l]) return fail(QW_ERR_ARG, "chain: null layer or output");
        if (st.layers[l]->device != device) return fail(QW_ERR_ARG, "chain: layers on different devices");
        lay[s].push_back(&st.layers[l]->dev);
        rps[s].push_back(st.layers[l]->host_row_ptr.data());
        num_sms = st.layers[l]->num_sms;
      }
      d[s] = qwdev::ChainStepDesc{lay[s].data(), rps[s].data(), st.n, st.x, st.ys, st.depends};
    }
    cudaSetDevice(device);
    auto C = std::make_unique<qw_chain>();
    C->device = device;
    bool mma = true;
    for (uint32_t s = 0; s < n; ++s)
      for (const auto* L : lay[s]) mma = mma && L->mrecs != nullptr;
    if (mma) {
      const int me = qwdev::plan_mma_chain(&C->mplan, d.data(), n, num_sms);
      if (me == (int)cudaErrorInvalidValue) return fail(QW_ERR_ARG, "chain: a step's layers differ in geometry");
      if (me) return cuda_fail((cudaError_t)me, "chain plan (mma)");
      *out = C.release();
      return (int)QW_OK;
    }
    for (uint32_t s = 0; s < n; ++s)
      for (uint32_t l = 0; l < steps[s].n; ++l)
        if (!steps[s].layers[l]->k2_ok)
          return fail(QW_ERR_UNSUPPORTED, "chain: a layer the SIMT kernel cannot take needs an all tensor-core chain");
    const int e = qwdev::plan_chain(&C->plan, d.data(), n, num_sms);
    if (e == (int)cudaErrorInvalidValue) return fail(QW_ERR_ARG, "chain: a step's layers differ in geometry");
    if (e == (int)cudaErrorNotSupported)
      return fail(QW_ERR_UNSUPPORTED, "chain: step geometry not covered (group2 % 4 != 0 or > 16384 columns)");
    if (e) return cuda_fail((cudaError_t)e, "chain plan");
    *out = C.release();
    return (int)QW_OK;
  });
}

int qw_chain_run(const qw_chain* c, void* stream) {
  if (!c) return fail(QW_ERR_ARG, "chain: null");
  int dev_now = -1;
  cudaGetDevice(&dev_now);
  if (dev_now != c->device) cudaSetDevice(c->device);
  const int e = c->mplan ? qwdev::launch_mma_chain(c->mplan, stream) : qwdev::launch_chain(c->plan, stream);
  return e ? cuda_fail((cudaError_t)e, "chain launch") : QW_OK;
}

int qw_debug_chain_timeline(const qw_chain* c, unsigned long long* out, uint64_t n) {
  if (!c || !c->mplan || !out) return fail(QW_ERR_ARG, "chain timeline: needs a tensor-core chain planned with QW_DEBUG_MMA_TL=1");
  const int e = qwdev::mma_chain_timeline(c->mplan, out, n);
  return e ? cuda_fail((cudaError_t)e, "chain timeline") : QW_OK;
}

int qw_debug_chain_watch(uint32_t* out, uint32_t n) {
  const unsigned* w = qwdev::chain_watch();
  if (!w || !out) return fail(QW_ERR_ARG, "chain watch: not enabled (QW_CHAIN_WATCH)");
  std::memcpy(out, w, (size_t)std::min<uint32_t>(n, 148 * 32 * 8 * 4) * 4);
  return QW_OK;
}

int qw_chain_free(qw_chain* c) {
  delete c;
  return QW_OK;
}

int qw_debug_group_timeline(const qw_group* g, const float* x, float* const* ys, unsigned long long* stamps,
                            uint32_t flags, void* stream) {
  if (!g || !x || !ys || !stamps) return fail(QW_ERR_ARG, "timeline: null argument");
  cudaSetDevice(g->device);
  const float* xs[qwdev::kMaxSeg];
  std::fill(xs, xs + qwdev::kMaxSeg, x);
  // K2m groups: %globaltimer stamps at the K2m events (qw_mma.cu)
  const int e = g->mma ? qwdev::launch_mma(g->mplan, g->layers.data(), (uint32_t)g->layers.size(), xs, ys, stream,
                                           flags & 1u, (flags & 4u) ? qwdev::kXIndependent : 0u, nullptr, stamps)
                       : qwdev::launch_gemv_group(g->plan, g->layers.data(), (uint32_t)g->layers.size(), xs, ys,
                                                  stream, flags & 1u, (flags & 4u) ? qwdev::kXIndependent : 0u,
                                                  stamps, 1, (flags & 2u) != 0);
  return e ? cuda_fail((cudaError_t)e, "group launch") : QW_OK;
}

int qw_debug_gemm_timeline(const qw_layer* L, const float* x, uint32_t batch, float* y,
                           unsigned long long* stamps, void* stream) {
  if (!L || !x || !y || !stamps) return fail(QW_ERR_ARG, "timeline: null argument");
  if (!L->dev.gemm.ok || batch < 2 || batch > 16) return fail(QW_ERR_UNSUPPORTED, "timeline: no batched path");
  cudaSetDevice(L->device);
  const int e = qwdev::launch_gemm(L->dev, x, batch, y, stream, stamps);
  return e ? cuda_fail((cudaError_t)e, "gemm launch") : QW_OK;
}

int qw_debug_timeline_events(void) { return (int)qwdev::kTimelineEvents; }

uint32_t qw_debug_knob(const char* name, uint32_t dflt) { return name ? qwdev::knob(name, dflt) : dflt; }

int qw_debug_gemm_shift(const qw_layer* L, int* shift) {
  if (!L || !shift) return fail(QW_ERR_ARG, "gemm shift: null argument");
  if (!L->dev.gemm.ok) return fail(QW_ERR_UNSUPPORTED, "gemm shift: layer has no batched tensor-core plan");
  *shift = L->dev.gemm.shift;
  return QW_OK;
}

int qw_launches_per_matvec(const qw_layer* L, uint32_t batch) {
  return qw_launches_per_matvec_ex(L, batch, 0u);
}

int qw_matvec_push(const qw_layer* L, const float* x, float* y, float* const* peer_y, uint32_t* const* peer_flag,
                   uint32_t npeer, void* stream, uint32_t flags) {
  if (!L || !x || !y || (npeer && (!peer_y || !peer_flag))) return fail(QW_ERR_ARG, "push: null argument");
  if (npeer > qwdev::kMaxPeer) return fail(QW_ERR_ARG, "push: at most 8 peers");
  if (L->dev.mrecs) return fail(QW_ERR_UNSUPPORTED, "push: the fused exchange runs on the SIMT kernel (upload with QW_UPLOAD_SIMT)");
  qwdev::PeerOut po{};
  for (uint32_t i = 0; i < npeer; ++i) {
    if (!peer_y[i] || !peer_flag[i]) return fail(QW_ERR_ARG, "push: null peer buffer");
    po.y[i] = peer_y[i], po.flag[i] = peer_flag[i];
  }
  po.n = npeer;
  int dev_now = -1;
  cudaGetDevice(&dev_now);
  if (dev_now != L->device) cudaSetDevice(L->device);
  const qwdev::DeviceLayer* one[1] = {&L->dev};
  const float* xs[1] = {x};
  float* ys[1] = {y};
  const uint32_t xflags = (flags & QW_LAUNCH_X_INDEPENDENT) ? qwdev::kXIndependent : 0u;
  const int e = qwdev::launch_gemv_group(L->dev.plan, one, 1, xs, ys, stream, (flags & QW_LAUNCH_PDL) != 0, xflags,
                                         nullptr, 1, false, &po);
  return e ? cuda_fail((cudaError_t)e, "push launch") : QW_OK;
}

int qw_push_arrivals(const qw_layer* L) {
  if (!L) return -fail(QW_ERR_ARG, "push arrivals: null layer");
  return (int)L->dev.plan.grid;
}

int qw_peer_wait(uint32_t* flag, uint32_t expected, void* stream) {
  if (!flag) return fail(QW_ERR_ARG, "peer wait: null counter");
  const int e = qwdev::launch_peer_wait(flag, expected, stream);
  return e ? cuda_fail((cudaError_t)e, "peer wait") : QW_OK;
}

int qw_peer_reduce(const float* staging, uint32_t world, uint32_t n, float* y, void* stream) {
  if (!staging || !y || world == 0) return fail(QW_ERR_ARG, "peer reduce: null argument");
  const int e = qwdev::launch_peer_reduce(staging, world, n, y, stream);
  return e ? cuda_fail((cudaError_t)e, "peer reduce") : QW_OK;
}

int qw_ipc_handle(const void* dev_ptr, uint8_t out[64]) {
  if (!dev_ptr || !out) return fail(QW_ERR_ARG, "ipc handle: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(out, &h, 64);
  return QW_OK;
}

int qw_ipc_open(const uint8_t handle[64], void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(QW_ERR_ARG, "ipc open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? QW_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

int qw_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(QW_ERR_ARG, "ipc close: null pointer");
  const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? QW_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

int qw_matvec_uses_gemm(const qw_layer* L, uint32_t batch, uint32_t flags) {
  if (!L) return -fail(QW_ERR_ARG, "uses_gemm: null layer");  // negative: 0 / 1 are answers
  return uses_gemm(L, batch, flags) ? 1 : 0;
}

int qw_launches_per_matvec_ex(const qw_layer* L, uint32_t batch, uint32_t flags) {
  if (L && uses_gemm(L, batch, flags)) return 2;  // x prologue (+ CSR), GEMM
  if (L && batch > 1 && column_groups()) return (int)qwdev::column_launches(L->dev, batch);
  return (int)batch;
}

}  // extern "C"
