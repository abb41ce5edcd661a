// qwb_gpu_producer.cpp -- quantize_layer (quantizer.cpp:132-146) with its
// data-parallel passes on the GPU (csrc/device/qw_quantize.cu): channel
// amplitudes, outlier scores (histogram + candidates), first-order group fits
// and codes, the 2-order pass.  The host keeps what needs a global order: the
// channel plan (plan_from_amplitudes, shared with the CPU producer), the final
// top-K ranking (score desc, row asc, col asc: outliers.cpp:20-26), the CSR
// split (outliers.cpp:99-129), the fp16 conversions and pack_layer.  Output is
// bit-identical to quantize_layer (tests/test_gpu_producer.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "qwb_host.hpp"

namespace qwdev {
int producer_amplitudes(const float* w, const float* h, uint32_t rows, uint32_t cols, double* amp);
int producer_scores(const float* w, const float* h, const uint32_t* perm, uint32_t rows, uint32_t cols,
                    uint32_t n2p, uint32_t mode, unsigned long long* hist, uint32_t floor_bucket, double* cs,
                    uint32_t* crow, uint32_t* ccol, unsigned long long* ncand, uint32_t* bad);
int producer_fits(const float* w, const uint32_t* perm, const uint32_t* row_ptr, const uint16_t* col_ind,
                  uint32_t* outmask, uint32_t rows, uint32_t cols, uint32_t n2p, uint32_t n4, uint32_t group2,
                  uint8_t* codes2, uint8_t* zeros2, float* scale1, uint8_t* codes4, float* s4, uint8_t* z4,
                  uint8_t* scodes, float* s2, uint8_t* zero2, uint32_t* bad);
}  // namespace qwdev

namespace qwb {

namespace {

// device buffers freed on scope exit
struct DevBufs {
  std::vector<void*> p;
  template <class T>
  T* alloc(size_t n) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) throw Error("gpu producer: out of memory");
    p.push_back(q);
    return static_cast<T*>(q);
  }
  ~DevBufs() {
    for (void* q : p) cudaFree(q);
  }
};

void cuda_check(int e, const char* what) {
  if (e != 0) throw Error(std::string("gpu producer: ") + what + ": " + cudaGetErrorString((cudaError_t)e));
}
template <class T>
void h2d(T* d, const T* h, size_t n) {
  cuda_check(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice), "copy to device");
}
template <class T>
void d2h(T* h, const T* d, size_t n) {
  cuda_check(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost), "copy to host");
}

struct Cand {
  double score;
  uint32_t row, col;
};
bool ranks_before(const Cand& a, const Cand& b) {  // outliers.cpp:20-26
  if (a.score != b.score) return a.score > b.score;
  if (a.row != b.row) return a.row < b.row;
  return a.col < b.col;
}

}  // namespace

PackedLayer quantize_layer_gpu(const float* w, uint32_t rows, uint32_t cols, std::span<const float> h,
                               const QuantizeParams& p, int device) {
  // the same argument checks, in the same order, as quantize_layer / build_plan_from
  if (!(p.alpha >= 0.0 && p.alpha <= 1.0)) throw Error("quantize: alpha must lie in [0, 1]");
  if (p.group2 == 0) throw Error("quantize: group2 must be positive");
  if (!(p.outlier_ratio >= 0.0 && p.outlier_ratio <= 1.0))
    throw Error("quantize: outlier ratio must lie in [0, 1]");
  if (!w || rows == 0 || cols == 0) throw Error("quantize: malformed weight matrix");
  if (cols < kG1 || cols % kG1 != 0) throw Error("quantize: cols must be a positive multiple of 16");
  if (h.size() != cols) throw Error("compute_amplitudes: calibration length != input channels");
  for (float v : h)
    if (!(v > 0.0f) || !std::isfinite(v)) throw Error("compute_amplitudes: calibration entries must be positive");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");

  DevBufs B;
  const size_t nw = (size_t)rows * cols;
  float* dw = B.alloc<float>(nw);
  float* dh = B.alloc<float>(cols);
  double* damp = B.alloc<double>(cols);
  uint32_t* dbad = B.alloc<uint32_t>(1);
  h2d(dw, w, nw);
  h2d(dh, h.data(), cols);
  cuda_check(cudaMemset(dbad, 0, 4), "memset");

  // ---- channel plan (plan.cpp:10-73): amplitudes on the device, ranking here
  cuda_check(qwdev::producer_amplitudes(dw, dh, rows, cols, damp), "amplitudes");
  std::vector<double> amp(cols);
  d2h(amp.data(), damp, cols);
  const ChannelPlan plan = plan_from_amplitudes(amp, cols, p.alpha);
  const uint32_t n2p = plan.n2_padded(), pc = plan.padded_channels(), n4 = plan.n4;
  uint32_t* dperm = B.alloc<uint32_t>(pc);
  h2d(dperm, plan.perm.data(), pc);

  // ---- outlier selection (outliers.cpp:61-97): top-k by (score desc, row asc, col asc)
  const uint64_t budget = (uint64_t)std::llround(p.outlier_ratio * (double)nw);
  std::vector<SlotRef> sel;
  uint32_t bad = 0;
  if (budget > 0) {
    constexpr size_t kBuckets = 1u << 16;
    unsigned long long* dhist = B.alloc<unsigned long long>(kBuckets);
    unsigned long long* dn = B.alloc<unsigned long long>(1);
    cuda_check(cudaMemset(dhist, 0, kBuckets * 8), "memset");
    cuda_check(qwdev::producer_scores(dw, dh, dperm, rows, cols, n2p, 0, dhist, 0, nullptr, nullptr, nullptr, dn,
                                      dbad),
               "scores");
    std::vector<unsigned long long> hist(kBuckets);
    d2h(hist.data(), dhist, kBuckets);
    d2h(&bad, dbad, 1);
    if (bad) throw Error("fit_scale_zero: non-finite value");
    uint64_t total = 0;
    for (auto c : hist) total += c;
    uint32_t floor_bucket = 0;
    if (total > budget) {
      uint64_t seen = 0;
      for (size_t b = kBuckets; b-- > 0;) {
        seen += hist[b];
        if (seen >= budget) {
          floor_bucket = (uint32_t)b;
          break;
        }
      }
    }
    uint64_t ncand = 0;
    for (size_t b = floor_bucket; b < kBuckets; ++b) ncand += hist[b];
    double* dcs = B.alloc<double>(ncand);
    uint32_t* dcr = B.alloc<uint32_t>(ncand);
    uint32_t* dcc = B.alloc<uint32_t>(ncand);
    cuda_check(cudaMemset(dn, 0, 8), "memset");
    cuda_check(qwdev::producer_scores(dw, dh, dperm, rows, cols, n2p, 1, dhist, floor_bucket, dcs, dcr, dcc, dn,
                                      dbad),
               "candidates");
    std::vector<double> cs(ncand);
    std::vector<uint32_t> cr(ncand), cc(ncand);
    d2h(cs.data(), dcs, ncand), d2h(cr.data(), dcr, ncand), d2h(cc.data(), dcc, ncand);
    std::vector<Cand> cands(ncand);
    for (size_t i = 0; i < ncand; ++i) cands[i] = {cs[i], cr[i], cc[i]};
    if (cands.size() > budget) {
      std::nth_element(cands.begin(), cands.begin() + (ptrdiff_t)budget, cands.end(), ranks_before);
      cands.resize(budget);
    }
    sel.resize(cands.size());
    for (size_t i = 0; i < cands.size(); ++i) sel[i] = {cands[i].row, cands[i].col};
    std::sort(sel.begin(), sel.end(),
              [](const SlotRef& a, const SlotRef& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
  }

  LayerConfig cfg;
  cfg.group2 = (uint16_t)p.group2;
  cfg.rows = rows;
  cfg.cols = cols;
  cfg.n4 = n4;
  cfg.pad2 = plan.pad2;
  cfg.outlier_count = (uint32_t)sel.size();
  cfg.alpha = (float)p.alpha;
  cfg.outlier_ratio = (float)p.outlier_ratio;

  // ---- split_dense_sparse (outliers.cpp:99-129)
  CsrOutliers csr;
  csr.row_ptr.assign((size_t)rows + 1, 0);
  csr.col_ind.reserve(sel.size());
  csr.values.reserve(sel.size());
  for (const SlotRef& s : sel) {
    if (s.col >= n2p || plan.perm[s.col] == kPad)
      throw Error("split_dense_sparse: selected slot outside 2-bit region");
    csr.row_ptr[s.row + 1]++;
    csr.col_ind.push_back((uint16_t)s.col);
    csr.values.push_back(f32_to_f16(w[(size_t)s.row * cols + plan.perm[s.col]]));
  }
  for (uint32_t r = 0; r < rows; ++r) csr.row_ptr[r + 1] += csr.row_ptr[r];

  // ---- group fits (quantizer.cpp:38-107) on the device
  const uint32_t gpr = cfg.groups_per_row(), T4 = cfg.blocks4(), rbs = cfg.row_blocks();
  uint32_t* drp = B.alloc<uint32_t>(rows + 1);
  uint16_t* dci = B.alloc<uint16_t>(csr.col_ind.size());
  uint32_t* dmask = B.alloc<uint32_t>((size_t)rows * ((pc + 31) / 32));
  uint8_t* dc2 = B.alloc<uint8_t>((size_t)rows * n2p);
  uint8_t* dz2 = B.alloc<uint8_t>((size_t)rows * gpr);
  float* ds1 = B.alloc<float>((size_t)rows * gpr);
  uint8_t* dc4 = B.alloc<uint8_t>((size_t)rows * n4);
  float* ds4 = B.alloc<float>((size_t)rows * T4);
  uint8_t* dz4 = B.alloc<uint8_t>((size_t)rows * T4);
  uint8_t* dsc = B.alloc<uint8_t>((size_t)rows * gpr);
  float* dsc2 = B.alloc<float>((size_t)rbs * gpr);
  uint8_t* dzo2 = B.alloc<uint8_t>((size_t)rbs * gpr);
  h2d(drp, csr.row_ptr.data(), rows + 1);
  if (!csr.col_ind.empty()) h2d(dci, csr.col_ind.data(), csr.col_ind.size());
  cuda_check(qwdev::producer_fits(dw, dperm, drp, dci, dmask, rows, cols, n2p, n4, p.group2, dc2, dz2, ds1, dc4,
                                  ds4, dz4, dsc, dsc2, dzo2, dbad),
             "fits");
  cuda_check(cudaDeviceSynchronize(), "fits");
  d2h(&bad, dbad, 1);
  if (bad & 1u) throw Error("fit_scale_zero: non-finite value");
  if (bad & 2u) throw Error("quantize_scales_2order: scales must be non-negative");

  LayerGroups g;
  g.codes2.resize((size_t)rows * n2p);
  g.zeros2.resize((size_t)rows * gpr);
  g.scodes.resize((size_t)rows * gpr);
  g.codes4.resize((size_t)rows * n4);
  g.sorder.resize((size_t)rbs * gpr);
  g.fourbit.resize((size_t)rows * T4);
  d2h(g.codes2.data(), dc2, g.codes2.size());
  d2h(g.zeros2.data(), dz2, g.zeros2.size());
  d2h(g.scodes.data(), dsc, g.scodes.size());
  d2h(g.codes4.data(), dc4, g.codes4.size());
  std::vector<float> s2((size_t)rbs * gpr), s4((size_t)rows * T4);
  std::vector<uint8_t> z2((size_t)rbs * gpr), z4((size_t)rows * T4);
  d2h(s2.data(), dsc2, s2.size()), d2h(z2.data(), dzo2, z2.size());
  d2h(s4.data(), ds4, s4.size()), d2h(z4.data(), dz4, z4.size());
  for (size_t i = 0; i < g.sorder.size(); ++i) g.sorder[i] = {z2[i], f32_to_f16(s2[i])};
  for (size_t i = 0; i < g.fourbit.size(); ++i) g.fourbit[i] = {f32_to_f16(s4[i]), z4[i]};
  return pack_layer(cfg, plan, g, std::move(csr));
}

}  // namespace qwb
