// qwb_producer.cpp -- offline producer of packed layers (host, C++).
//
// Reproduces the reference pipeline quantize_layer (quantizer.cpp:132-146):
// Eq. 8 amplitudes -> channel plan -> permutation -> outlier scoring ->
// global top-K -> dense/sparse split -> per-group fits -> 2-order pass ->
// pack.  Outputs are bit-identical to the reference; the implementation is
// organised for speed instead (row-parallel passes, no full score matrix, a
// histogram threshold instead of a global sort), which the selection order
// (score desc, row asc, col asc) makes safe because it is a strict total
// order.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <thread>

#include "qwb_host.hpp"

namespace qwb {

// ------------------------------------------------------------------ synth
// synth.cpp:11-21
WeightMatrix synth_gaussian(uint32_t rows, uint32_t cols, uint64_t seed) {
  WeightMatrix w;
  w.rows = rows;
  w.cols = cols;
  w.data.resize((size_t)rows * cols);
  std::mt19937_64 gen(seed);
  std::normal_distribution<float> nd(0.0f, 1.0f);
  for (float& v : w.data) v = nd(gen);
  return w;
}

// synth.cpp:23-37
void plant_outliers(std::span<float> w, double ratio, float scale, uint64_t seed) {
  if (!(ratio >= 0.0 && ratio <= 1.0))
    throw Error("plant_outliers: ratio must lie in [0, 1]");
  const size_t count = (size_t)std::llround(ratio * (double)w.size());
  if (count == 0) return;
  std::mt19937_64 gen(seed ^ 0x9E3779B97F4A7C15ull);
  std::vector<size_t> order(w.size());
  std::iota(order.begin(), order.end(), (size_t)0);
  std::shuffle(order.begin(), order.end(), gen);
  std::uniform_real_distribution<float> mag(scale, 2.0f * scale);
  std::bernoulli_distribution heads(0.5);
  for (size_t i = 0; i < count; ++i) {
    const bool pos = heads(gen);
    w[order[i]] = pos ? mag(gen) : -mag(gen);
  }
}

// synth.cpp:39-47
std::vector<float> synth_calibration(uint32_t cols, uint64_t seed) {
  std::mt19937_64 gen(seed ^ 0xD1B54A32D192ED03ull);
  std::normal_distribution<float> nd(1.0f, 0.25f);
  std::vector<float> h(cols);
  for (float& v : h) v = std::fabs(nd(gen)) + 0.05f;
  return h;
}

// synth.cpp:49-56
std::vector<float> synth_activation(uint32_t cols, uint64_t seed) {
  std::mt19937_64 gen(seed ^ 0xA0761D6478BD642Full);
  std::normal_distribution<float> nd(0.0f, 1.0f);
  std::vector<float> x(cols);
  for (float& v : x) v = nd(gen);
  return x;
}

// ------------------------------------------------------------------ plan
// compute_amplitudes (plan.cpp:10-30) fused with build_plan (plan.cpp:32-73).
ChannelPlan build_plan_from(const WeightMatrix& w, std::span<const float> h,
                            double alpha, unsigned threads) {
  if (!w.valid() || w.rows == 0 || w.cols == 0)
    throw Error("compute_amplitudes: malformed weight matrix");
  if (h.size() != w.cols)
    throw Error("compute_amplitudes: calibration length != input channels");
  for (float v : h)
    if (!(v > 0.0f) || !std::isfinite(v))
      throw Error("compute_amplitudes: calibration entries must be positive");
  const uint32_t ic = w.cols;
  if (ic % kG1 != 0)
    throw Error("build_plan: channel count must be a positive multiple of 16");
  if (!(alpha >= 0.0 && alpha <= 1.0))
    throw Error("build_plan: alpha must lie in [0, 1]");

  // Each column accumulates over rows in ascending order, as the reference.
  std::vector<double> amp(ic, 0.0);
  parallel_for(ic, threads, [&](uint64_t c0, uint64_t c1) {
    for (uint32_t r = 0; r < w.rows; ++r) {
      const float* row = w.data.data() + (size_t)r * ic;
      for (uint64_t c = c0; c < c1; ++c) {
        const double a = row[c];
        const double b = h[c];
        amp[c] += (a * a) / (b * b);
      }
    }
  });

  return plan_from_amplitudes(amp, ic, alpha);
}

// build_plan (plan.cpp:32-73) from the channel amplitudes: the top n4 by
// (amplitude desc, index asc) become 4-bit; layout [2-bit asc | pads | 4-bit asc].
ChannelPlan plan_from_amplitudes(const std::vector<double>& amp, uint32_t ic, double alpha) {
  uint32_t n4 = 16u * (uint32_t)std::floor(alpha * (double)ic / 16.0 + 0.5);
  n4 = std::min(n4, ic);
  std::vector<uint32_t> idx(ic);
  std::iota(idx.begin(), idx.end(), 0u);
  auto louder = [&](uint32_t a, uint32_t b) {
    return amp[a] != amp[b] ? amp[a] > amp[b] : a < b;
  };
  if (n4 > 0 && n4 < ic) std::nth_element(idx.begin(), idx.begin() + n4, idx.end(), louder);
  std::vector<uint32_t> four(idx.begin(), idx.begin() + n4);
  std::sort(four.begin(), four.end());

  ChannelPlan plan;
  plan.in_channels = ic;
  plan.n4 = n4;
  plan.bits.assign(ic, 2);
  for (uint32_t c : four) plan.bits[c] = 4;
  const uint32_t n2 = ic - n4;
  plan.pad2 = (kTile2 - n2 % kTile2) % kTile2;
  if ((uint64_t)n2 + plan.pad2 + n4 > kMaxSlots)
    throw Error("build_plan: padded channel count exceeds 65536");
  plan.perm.reserve(plan.padded_channels());
  for (uint32_t c = 0; c < ic; ++c)
    if (plan.bits[c] == 2) plan.perm.push_back(c);
  plan.perm.insert(plan.perm.end(), plan.pad2, kPad);
  plan.perm.insert(plan.perm.end(), four.begin(), four.end());
  return plan;
}

namespace {

// permute_matrix (plan.cpp:129-144) for one row.
void permute_row(const float* src, const ChannelPlan& plan, float* dst) {
  const uint32_t n = plan.padded_channels();
  for (uint32_t s = 0; s < n; ++s) dst[s] = plan.perm[s] == kPad ? 0.0f : src[plan.perm[s]];
}

// Residual score of the baseline 2-bit group fit (outliers.cpp:30-44,
// score_outliers 61-79), handed to `sink(col, score)` for real 2-bit slots.
template <class Sink>
void score_row(const float* wp, const ChannelPlan& plan, std::span<const float> h,
               Sink&& sink) {
  uint8_t codes[kG1];
  for (uint32_t base = 0; base < plan.n2_padded(); base += kG1) {
    std::span<const float> vals(wp + base, kG1);
    const ScaleZero sz = fit_scale_zero(vals, 2);
    quantize_values(vals, sz.scale, sz.zero, 2, codes);
    for (uint32_t k = 0; k < kG1; ++k) {
      const uint32_t orig = plan.perm[base + k];
      if (orig == kPad) continue;
      const double res = (double)dequantize_one(codes[k], sz.zero, sz.scale) - (double)vals[k];
      const double dh = h[orig];
      const double s = (res * res) / (dh * dh);
      if (s > 0.0) sink(base + k, s);
    }
  }
}

struct Cand {
  double score;
  uint32_t row, col;
};
inline bool ranks_before(const Cand& a, const Cand& b) {  // outliers.cpp:20-26
  if (a.score != b.score) return a.score > b.score;
  if (a.row != b.row) return a.row < b.row;
  return a.col < b.col;
}
inline uint32_t score_bucket(double s) {  // positive doubles order by bits
  uint64_t u;
  std::memcpy(&u, &s, sizeof u);
  return (uint32_t)(u >> 48);
}

// select_outliers (outliers.cpp:81-97): global top-k by (score desc, row asc,
// col asc), returned sorted by (row, col).  A first pass histograms the
// scores by their top 16 bits to find the bucket holding rank k; the second
// pass keeps only candidates at or above it.
std::vector<SlotRef> select_top(const WeightMatrix& w, const ChannelPlan& plan,
                                std::span<const float> h, uint64_t k, unsigned threads) {
  if (k == 0) return {};
  const uint32_t pc = plan.padded_channels();
  constexpr size_t kBuckets = 1u << 16;
  std::vector<std::vector<uint64_t>> hist_parts;
  const unsigned nt = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
  const uint64_t parts = std::min<uint64_t>(nt, w.rows);
  hist_parts.assign(parts, std::vector<uint64_t>(kBuckets, 0));
  parallel_for(parts, (unsigned)parts, [&](uint64_t p0, uint64_t p1) {
    for (uint64_t p = p0; p < p1; ++p) {
      std::vector<float> wp(pc);
      auto& hist = hist_parts[p];
      const uint32_t r0 = (uint32_t)(w.rows * p / parts), r1 = (uint32_t)(w.rows * (p + 1) / parts);
      for (uint32_t r = r0; r < r1; ++r) {
        permute_row(w.data.data() + (size_t)r * w.cols, plan, wp.data());
        score_row(wp.data(), plan, h, [&](uint32_t, double s) { hist[score_bucket(s)]++; });
      }
    }
  });
  std::vector<uint64_t> hist(kBuckets, 0);
  for (auto& hp : hist_parts)
    for (size_t b = 0; b < kBuckets; ++b) hist[b] += hp[b];
  uint64_t total = 0;
  for (uint64_t c : hist) total += c;
  uint32_t floor_bucket = 0;
  if (total > k) {
    uint64_t seen = 0;
    for (size_t b = kBuckets; b-- > 0;) {
      seen += hist[b];
      if (seen >= k) {
        floor_bucket = (uint32_t)b;
        break;
      }
    }
  }
  std::vector<std::vector<Cand>> keep_parts(parts);
  parallel_for(parts, (unsigned)parts, [&](uint64_t p0, uint64_t p1) {
    for (uint64_t p = p0; p < p1; ++p) {
      std::vector<float> wp(pc);
      auto& keep = keep_parts[p];
      const uint32_t r0 = (uint32_t)(w.rows * p / parts), r1 = (uint32_t)(w.rows * (p + 1) / parts);
      for (uint32_t r = r0; r < r1; ++r) {
        permute_row(w.data.data() + (size_t)r * w.cols, plan, wp.data());
        score_row(wp.data(), plan, h, [&](uint32_t c, double s) {
          if (score_bucket(s) >= floor_bucket) keep.push_back({s, r, c});
        });
      }
    }
  });
  std::vector<Cand> cands;
  for (auto& kp : keep_parts) cands.insert(cands.end(), kp.begin(), kp.end());
  if (cands.size() > k) {
    std::nth_element(cands.begin(), cands.begin() + (ptrdiff_t)k, cands.end(), ranks_before);
    cands.resize(k);
  }
  std::vector<SlotRef> sel(cands.size());
  for (size_t i = 0; i < cands.size(); ++i) sel[i] = {cands[i].row, cands[i].col};
  std::sort(sel.begin(), sel.end(), [](const SlotRef& a, const SlotRef& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  return sel;
}

// quantize_scales_2order (quant.cpp:87-107)
void scales_2order(std::span<const float> col, uint8_t* codes, SorderParam* out) {
  if (col.empty()) throw Error("quantize_scales_2order: empty scale column");
  float hi = 0.0f;
  for (float s : col) {
    if (!(s >= 0.0f) || !std::isfinite(s))
      throw Error("quantize_scales_2order: scales must be non-negative");
    hi = std::max(hi, s);
  }
  const float ends[2] = {0.0f, hi};
  const ScaleZero sz = fit_scale_zero(ends, 4);
  quantize_values(col, sz.scale, sz.zero, 4, codes);
  out->zero2 = sz.zero;
  out->scale2 = f32_to_f16(sz.scale);
}

}  // namespace

// quantize_layer (quantizer.cpp:132-146) = plan + selection +
// quantize_with_plan (111-130) + quantize_groups (38-109) + pack_layer.
PackedLayer quantize_layer(const WeightMatrix& w, std::span<const float> h,
                           const QuantizeParams& p, unsigned threads) {
  if (!(p.alpha >= 0.0 && p.alpha <= 1.0)) throw Error("quantize: alpha must lie in [0, 1]");
  if (p.group2 == 0) throw Error("quantize: group2 must be positive");
  if (!(p.outlier_ratio >= 0.0 && p.outlier_ratio <= 1.0))
    throw Error("quantize: outlier ratio must lie in [0, 1]");
  if (!w.valid() || w.rows == 0) throw Error("quantize: malformed weight matrix");
  if (w.cols < kG1 || w.cols % kG1 != 0)
    throw Error("quantize: cols must be a positive multiple of 16");

  const ChannelPlan plan = build_plan_from(w, h, p.alpha, threads);
  const uint64_t budget = (uint64_t)std::llround(p.outlier_ratio * (double)((uint64_t)w.rows * w.cols));
  const std::vector<SlotRef> sel = select_top(w, plan, h, budget, threads);

  LayerConfig cfg;
  cfg.group2 = (uint16_t)p.group2;
  cfg.rows = w.rows;
  cfg.cols = w.cols;
  cfg.n4 = plan.n4;
  cfg.pad2 = plan.pad2;
  cfg.outlier_count = (uint32_t)sel.size();
  cfg.alpha = (float)p.alpha;
  cfg.outlier_ratio = (float)p.outlier_ratio;

  // split_dense_sparse (outliers.cpp:99-129): CSR of the selected slots
  CsrOutliers csr;
  csr.row_ptr.assign((size_t)w.rows + 1, 0);
  csr.col_ind.reserve(sel.size());
  csr.values.reserve(sel.size());
  for (const SlotRef& s : sel) {
    if (s.col >= plan.n2_padded() || plan.perm[s.col] == kPad)
      throw Error("split_dense_sparse: selected slot outside 2-bit region");
    csr.row_ptr[s.row + 1]++;
    csr.col_ind.push_back((uint16_t)s.col);
    csr.values.push_back(f32_to_f16(w.at(s.row, plan.perm[s.col])));
  }
  for (uint32_t r = 0; r < w.rows; ++r) csr.row_ptr[r + 1] += csr.row_ptr[r];

  const uint32_t gpr = cfg.groups_per_row(), n2p = cfg.n2_padded(), pc = cfg.padded_cols();
  LayerGroups g;
  g.codes2.resize((size_t)cfg.rows * n2p);
  g.zeros2.resize((size_t)cfg.rows * gpr);
  g.scodes.assign((size_t)cfg.rows * gpr, 0);
  g.sorder.resize(cfg.sorder_count());
  g.codes4.resize((size_t)cfg.rows * cfg.n4);
  g.fourbit.resize(cfg.fourbit_count());
  std::vector<float> scale1((size_t)cfg.rows * gpr);

  // first-order fits; outlier slots hold 0 in the dense copy and are left
  // out of the 2-bit refit (quantizer.cpp:50-80)
  parallel_for(cfg.rows, threads, [&](uint64_t r0, uint64_t r1) {
    std::vector<float> wp(pc);
    std::vector<uint8_t> is_out(pc);
    float keep[kG1];
    for (uint64_t r = r0; r < r1; ++r) {
      permute_row(w.data.data() + (size_t)r * w.cols, plan, wp.data());
      std::fill(is_out.begin(), is_out.end(), 0);
      for (uint32_t i = csr.row_ptr[r]; i < csr.row_ptr[r + 1]; ++i) {
        is_out[csr.col_ind[i]] = 1;
        wp[csr.col_ind[i]] = 0.0f;
      }
      for (uint32_t j = 0; j < gpr; ++j) {
        const uint32_t base = j * kG1;
        size_t kept = 0;
        for (uint32_t k = 0; k < kG1; ++k)
          if (!is_out[base + k]) keep[kept++] = wp[base + k];
        if (kept == 0) keep[kept++] = 0.0f;
        const ScaleZero sz = fit_scale_zero({keep, kept}, cfg.n);
        scale1[r * gpr + j] = sz.scale;
        g.zeros2[r * gpr + j] = sz.zero;
        quantize_values({wp.data() + base, kG1}, sz.scale, sz.zero, cfg.n,
                        g.codes2.data() + r * n2p + base);
      }
      for (uint32_t b = 0; b < cfg.blocks4(); ++b) {
        std::span<const float> vals(wp.data() + n2p + b * kG1, kG1);
        const ScaleZero sz = fit_scale_zero(vals, cfg.n2);
        quantize_values(vals, sz.scale, sz.zero, cfg.n2,
                        g.codes4.data() + r * cfg.n4 + b * kG1);
        g.fourbit[r * cfg.blocks4() + b] = {f32_to_f16(sz.scale), sz.zero};
      }
    }
  });

  // second-order pass down each group column of a row block, 4/3/3 rule
  // (quantizer.cpp:82-107)
  parallel_for(cfg.row_blocks(), threads, [&](uint64_t b0, uint64_t b1) {
    std::vector<float> col(cfg.group2);
    std::vector<uint8_t> codes(cfg.group2);
    for (uint64_t rb = b0; rb < b1; ++rb) {
      const uint32_t r0 = (uint32_t)rb * cfg.group2;
      const uint32_t rn = std::min<uint32_t>(cfg.group2, cfg.rows - r0);
      for (uint32_t j = 0; j < gpr; ++j) {
        for (uint32_t i = 0; i < rn; ++i) col[i] = scale1[(size_t)(r0 + i) * gpr + j];
        scales_2order({col.data(), rn}, codes.data(), &g.sorder[rb * gpr + j]);
        for (uint32_t i = 0; i < rn; ++i)
          g.scodes[(size_t)(r0 + i) * gpr + j] = (j % 3 == 0) ? codes[i] : (uint8_t)(codes[i] >> 1);
      }
    }
  });

  return pack_layer(cfg, plan, g, std::move(csr));
}

}  // namespace qwb
