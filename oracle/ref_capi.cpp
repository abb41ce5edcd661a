// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.  extern "C" shim over the
// UNMODIFIED reference library (arXiv 2311.16442 artifact, namespace
// qweight), compiled by oracle/Makefile from the reference sources where they
// lie (/root/reference/proj/src/*.cpp) into oracle/_ref/libqweight_ref.so.
// Used by tests/ to pin the C oracle and the host producer, and by bench.py
// as the reference CPU arm.  It adds no arithmetic of its own: every value it
// returns comes from a reference function.
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "qweight/bitpack.hpp"
#include "qweight/container.hpp"
#include "qweight/engine.hpp"
#include "qweight/fp16.hpp"
#include "qweight/metrics.hpp"
#include "qweight/quant.hpp"
#include "qweight/quantizer.hpp"
#include "qweight/synth.hpp"

#include "../include/qweight_b200.h"

namespace {

thread_local std::string last;

struct RefLayer {
  qweight::PackedLayer L;
  std::vector<uint8_t> sz, fz;
  std::vector<uint16_t> ss, fs;
  void soa() {
    sz.clear(), ss.clear(), fz.clear(), fs.clear();
    for (auto& p : L.sorder) sz.push_back(p.zero2), ss.push_back(p.scale2);
    for (auto& p : L.fourbit) fz.push_back(p.zero), fs.push_back(p.scale);
  }
};

template <class F>
int wrap(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    last = e.what();
    return 1;
  }
}

template <class T>
std::vector<T> vec(const T* p, uint64_t n) {
  return n ? std::vector<T>(p, p + n) : std::vector<T>{};
}

}  // namespace

extern "C" {

const char* qwref_last_error(void) { return last.c_str(); }

// quantize_layer (quantizer.hpp:21-22)
int qwref_quantize(const float* w, uint32_t rows, uint32_t cols, const float* h, double alpha,
                   uint32_t group2, double ratio, void** out) {
  return wrap([&] {
    qweight::WeightMatrix W;
    W.rows = rows, W.cols = cols, W.data = vec(w, (uint64_t)rows * cols);
    qweight::CalibrationVector H;
    H.h = vec(h, cols);
    qweight::QuantizeParams p;
    p.alpha = alpha, p.group2 = group2, p.outlier_ratio = ratio;
    auto R = std::make_unique<RefLayer>();
    R->L = qweight::quantize_layer(W, H, p);
    R->soa();
    *out = R.release();
  });
}

int qwref_from_view(const qw_layer_view* v, void** out) {
  return wrap([&] {
    auto R = std::make_unique<RefLayer>();
    auto& L = R->L;
    auto& c = L.cfg;
    c.n = v->n, c.n2 = v->n2, c.group1 = v->group1, c.group2 = v->group2, c.tile = v->tile;
    c.rows = v->rows, c.cols = v->cols, c.n4 = v->n4, c.pad2 = v->pad2;
    c.outlier_count = v->outlier_count, c.alpha = v->alpha, c.outlier_ratio = v->outlier_ratio;
    L.plan.in_channels = v->cols, L.plan.n4 = v->n4, L.plan.pad2 = v->pad2;
    L.plan.bits = vec(v->plan_bits, v->plan_bits_len);
    L.plan.perm = vec(v->plan_perm, v->plan_perm_len);
    L.main = vec(v->main, v->main_len);
    L.tail2 = vec(v->tail2, v->tail2_len);
    L.tail4 = vec(v->tail4, v->tail4_len);
    L.secondary = vec(v->secondary, v->secondary_len);
    L.meta = vec(v->meta, v->meta_len);
    for (uint64_t i = 0; i < v->sorder_len; ++i) L.sorder.push_back({v->sorder_zero2[i], v->sorder_scale2[i]});
    for (uint64_t i = 0; i < v->fourbit_len; ++i) L.fourbit.push_back({v->fourbit_scale[i], v->fourbit_zero[i]});
    L.csr.row_ptr = vec(v->csr_row_ptr, v->csr_row_ptr_len);
    L.csr.col_ind = vec(v->csr_col_ind, v->csr_nnz);
    L.csr.values = vec(v->csr_values, v->csr_nnz);
    qweight::validate_layer(L);
    R->soa();
    *out = R.release();
  });
}

int qwref_view(void* h, qw_layer_view* v) {
  auto* R = (RefLayer*)h;
  const auto& L = R->L;
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
  v->sorder_zero2 = R->sz.data(), v->sorder_scale2 = R->ss.data(), v->sorder_len = L.sorder.size();
  v->fourbit_scale = R->fs.data(), v->fourbit_zero = R->fz.data(), v->fourbit_len = L.fourbit.size();
  v->csr_row_ptr = L.csr.row_ptr.data(), v->csr_row_ptr_len = L.csr.row_ptr.size();
  v->csr_col_ind = L.csr.col_ind.data(), v->csr_values = L.csr.values.data();
  v->csr_nnz = L.csr.col_ind.size();
  return 0;
}

void qwref_free(void* h) { delete (RefLayer*)h; }

// matvec_oracle / matvec_pipelined (engine.hpp:31-36); wall_ns as reported
int qwref_matvec_oracle(void* h, const float* x, uint64_t n, float* y, uint64_t* wall_ns) {
  return wrap([&] {
    auto r = qweight::matvec_oracle(((RefLayer*)h)->L, {x, n});
    std::memcpy(y, r.y.data(), r.y.size() * 4);
    if (wall_ns) *wall_ns = r.wall_ns;
  });
}

int qwref_matvec_pipelined(void* h, const float* x, uint64_t n, uint32_t workers, float* y,
                           uint64_t* wall_ns) {
  return wrap([&] {
    auto r = qweight::matvec_pipelined(((RefLayer*)h)->L, {x, n}, workers);
    std::memcpy(y, r.y.data(), r.y.size() * 4);
    if (wall_ns) *wall_ns = r.wall_ns;
  });
}

int qwref_matvec_f64(void* h, const float* x, uint64_t n, double* y) {
  return wrap([&] {
    auto r = qweight::matvec_reference_f64(((RefLayer*)h)->L, {x, n});
    std::memcpy(y, r.data(), r.size() * 8);
  });
}

int qwref_reconstruct(void* h, float* w) {
  return wrap([&] {
    auto r = qweight::reconstruct_dense(((RefLayer*)h)->L);
    std::memcpy(w, r.data.data(), r.data.size() * 4);
  });
}

int qwref_unpack(void* h, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes, uint8_t* codes4) {
  return wrap([&] {
    auto g = qweight::unpack_layer(((RefLayer*)h)->L);
    std::memcpy(codes2, g.codes2.data(), g.codes2.size());
    std::memcpy(zeros2, g.zeros2.data(), g.zeros2.size());
    std::memcpy(scodes, g.scodes.data(), g.scodes.size());
    if (!g.codes4.empty()) std::memcpy(codes4, g.codes4.data(), g.codes4.size());
  });
}

uint64_t qwref_payload_bytes(void* h) { return qweight::payload_bytes(((RefLayer*)h)->L); }

int qwref_write(void* h, const char* path) {
  return wrap([&] { qweight::write_packed_layer(((RefLayer*)h)->L, path); });
}

int qwref_read(const char* path, void** out) {
  return wrap([&] {
    auto R = std::make_unique<RefLayer>();
    R->L = qweight::read_packed_layer(path);
    R->soa();
    *out = R.release();
  });
}

int qwref_synth_gaussian(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  return wrap([&] {
    auto w = qweight::synth_gaussian(rows, cols, seed);
    std::memcpy(out, w.data.data(), w.data.size() * 4);
  });
}

int qwref_plant_outliers(float* w, uint32_t rows, uint32_t cols, double ratio, float scale,
                         uint64_t seed) {
  return wrap([&] {
    qweight::WeightMatrix W;
    W.rows = rows, W.cols = cols, W.data = vec(w, (uint64_t)rows * cols);
    qweight::plant_outliers(W, ratio, scale, seed);
    std::memcpy(w, W.data.data(), W.data.size() * 4);
  });
}

int qwref_synth_calibration(uint32_t cols, uint64_t seed, float* out) {
  return wrap([&] {
    auto h = qweight::synth_calibration(cols, seed);
    std::memcpy(out, h.h.data(), h.h.size() * 4);
  });
}

int qwref_synth_activation(uint32_t cols, uint64_t seed, float* out) {
  return wrap([&] {
    auto x = qweight::synth_activation(cols, seed);
    std::memcpy(out, x.data(), x.size() * 4);
  });
}

// pack_tile (bitpack.hpp:31-34) -> 22-byte wire image (helpers.hpp:27-33)
int qwref_pack_tile(const uint8_t* c2, const uint8_t* c4, const uint8_t* z, const uint8_t* s,
                    uint8_t* out22) {
  return wrap([&] {
    auto t = qweight::pack_tile({c2, 48}, {c4, 16}, {z, 3}, {s, 3});
    std::memcpy(out22, t.main.data(), 16);
    std::memcpy(out22 + 16, t.secondary.data(), 4);
    out22[20] = (uint8_t)(t.meta & 0xFF);
    out22[21] = (uint8_t)(t.meta >> 8);
  });
}

uint16_t qwref_f32_to_f16(float f) { return qweight::f32_to_f16(f); }
float qwref_f16_to_f32(uint16_t h) { return qweight::f16_to_f32(h); }

}  // extern "C"
